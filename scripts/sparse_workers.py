"""Per-worker timeline of the two-panel driver on a sparse input (32768^2 fill_random(p)).
usage: PYTHONPATH=.:tests python scripts/sparse_workers.py [p]"""
import os, sys
import numpy as np
sys.path.insert(0, "tests")
import paper_1111_6549_b200 as G
p = float(sys.argv[1]) if len(sys.argv) > 1 else 1 / 256
m = n = 32768
a = G.BitMatrix(m, n)
G.fill_random(a, p, 1)
d = G.DeviceMatrix(m, n)
out = "gpurun_out/workers_sparse.bin"
for it in range(3):
    d.upload(a.words)
    if it == 2:
        os.environ["GF2CU_DUMP_WORKERS"] = out
    o = G.block_iterative_ple(d, G.PleConfig(time_kernels=True, super_step=True))
print("kernel_ms", o.stats["kernel_ms"], "panel_ms", o.stats["panel_ms"])
os.system(f"python scripts/super_workers.py 0x0 {out} | tail -14")
