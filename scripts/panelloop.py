"""Median panel pivot-loop time (device stamps 6/7) of the single-panel driver."""
import os
import sys

import numpy as np

import paper_1111_6549_b200 as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a, b = G.DeviceMatrix(n, n), G.DeviceMatrix(n, n)
b.fill_ctr(1)
path = "gpurun_out/ploop.txt"
for it in range(2):
    a.copy_from(b)
    if it == 1:
        os.environ["GF2CU_DUMP_PHASES"] = path
    o = G.block_iterative_ple(a, G.PleConfig(time_kernels=True, single_panel=True))
d = np.loadtxt(path, skiprows=1, comments="#")
loop = (d[:, 10] - d[:, 9]) / 1e3
tot = (d[:, 4] - d[:, 3]) / 1e3
ok = loop > 0
print(f"n={n} kernel {o.stats['kernel_ms']:.3f} ms; pivot loop median {np.median(loop[ok][5:-5]):.2f} us, "
      f"panel median {np.median(tot[ok][5:-5]):.2f} us")
