import sys, time, torch
import paper_1111_6549_b200 as G
for n in [int(x) for x in sys.argv[1:]]:
    a = G.DeviceMatrix(n, n); b = G.DeviceMatrix(n, n); b.fill_ctr(1)
    for it in range(3):
        a.copy_from(b); torch.cuda.synchronize()
        t0 = time.perf_counter()
        o = G.block_iterative_ple(a, G.PleConfig(time_kernels=True))
        t1 = time.perf_counter()
        print(f"n={n} wall {1e3*(t1-t0):.3f} ms kernel {o.stats['kernel_ms']:.3f} ms steps {o.stats['steps']}")
