"""Per-step device timeline of the persistent driver (GF2CU_DUMP_PHASES)."""
import os, sys
import numpy as np
import paper_1111_6549_b200 as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/phases.txt"
a = G.DeviceMatrix(n, n); b = G.DeviceMatrix(n, n); b.fill_ctr(1)
for it in range(2):
    a.copy_from(b)
    if it == 1: os.environ["GF2CU_DUMP_PHASES"] = out
    o = G.block_iterative_ple(a, G.PleConfig(time_kernels=True))
print(o.stats)
