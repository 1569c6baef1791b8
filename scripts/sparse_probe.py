"""32768^2 fill_random(p) (BASELINE config 3: window misses) with both persistent drivers: wall time and kernel time.
usage: PYTHONPATH=.:tests python scripts/sparse_probe.py [p]"""
import sys, time, json
import numpy as np
sys.path.insert(0, "tests")
import paper_1111_6549_b200 as G
m = n = 32768
a = G.BitMatrix(m, n)
G.fill_random(a, float(sys.argv[1]) if len(sys.argv) > 1 else 1/256, 1)
src = a.words.copy()
d = G.DeviceMatrix(m, n)
import torch
for label, cfg in (("default", G.PleConfig()), ("timed", G.PleConfig(time_kernels=True)), ("single", G.PleConfig(single_panel=True)), ("single timed", G.PleConfig(single_panel=True, time_kernels=True))):
    ts = []
    for it in range(3):
        d.upload(src)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = G.block_iterative_ple(d, cfg)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    print(label, [round(t, 2) for t in ts], "kernel_ms", out.stats["kernel_ms"], "rank", out.rank, flush=True)
