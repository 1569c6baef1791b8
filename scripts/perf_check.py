"""Kernel times of the default single-GPU driver (and optionally forced ones)
on ctr(seed 1) inputs, with device checksums so a speed change that breaks
the result shows. usage: python scripts/perf_check.py [reps] [driver]"""
import sys

import paper_1111_6549_b200 as G

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
drv = sys.argv[2] if len(sys.argv) > 2 else "default"
KNOWN = {(65536, 65536): 0x172719ccff15b03a, (32768, 32768): 0x91405a67a0125ea4}
cfgs = {"default": {}, "super": {"super_step": True}, "single": {"single_panel": True}}
for (m, n) in [(4096, 4096), (16384, 16384), (16384, 65536), (32768, 32768), (65536, 65536)]:
    dm = G.DeviceMatrix(m, n)
    ts = []
    for _ in range(reps):
        dm.fill_ctr(1)
        out = G.block_iterative_ple(dm, G.PleConfig(time_kernels=True, **cfgs[drv]))
        ts.append(out.stats["kernel_ms"])
    cs = dm.checksum()
    ok = "" if (m, n) not in KNOWN else ("  checksum ok" if cs == KNOWN[(m, n)] else "  CHECKSUM MISMATCH")
    print(f"{m}x{n} driver {out.stats['driver']}: min {min(ts):.3f} ms  med {sorted(ts)[len(ts)//2]:.3f} ms "
          f"rank {out.rank} {cs:#x}{ok}", flush=True)
    dm.close()
