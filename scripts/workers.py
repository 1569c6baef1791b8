"""Dump per-worker rest-sweep stamps of one persistent PLE (diagnostics).
usage: GF2CU_DUMP_WORKERS=<out.bin> python scripts/workers.py N"""
import sys

import paper_1111_6549_b200 as G

n = int(sys.argv[1])
dm = G.DeviceMatrix(n, n)
for _ in range(2):
    dm.fill_ctr(1)
    out = G.block_iterative_ple(dm, G.PleConfig(time_kernels=True))
print("rank", out.rank, "kernel_ms", out.stats["kernel_ms"])
