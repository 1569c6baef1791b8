"""Quick device-resident timing probe (not the bench): PLE of ctr matrices."""
import sys, time
import torch
import paper_1111_6549_b200 as G

sizes = [int(x) for x in sys.argv[1:]] or [4096, 16384, 65536]
for n in sizes:
    m = n
    a = G.DeviceMatrix(m, n)
    b = G.DeviceMatrix(m, n)
    b.fill_ctr(1)
    for it in range(3):
        a.copy_from(b)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = G.block_iterative_ple(a, G.PleConfig(time_kernels=(it == 2)))
        t1 = time.perf_counter()
        s = out.stats
        print(f"n={n} it={it} rank={out.rank} wall={1e3*(t1-t0):.2f} ms steps={s['steps']} "
              f"trail={s['trailing_ms']:.2f} panel={s['panel_ms']:.2f} apply={s['coef_ms']:.2f} ms "
              f"alg={s['alg_bytes']/1e9:.2f} GB -> {s['alg_bytes']/1e9/(1e-3*(t1-t0)):.0f} GB/s wall, "
              f"{(s['alg_bytes']/1e9/(1e-3*s['trailing_ms'])) if s['trailing_ms'] else 0:.0f} GB/s trailing", flush=True)
    print("checksum", hex(a.checksum()))
