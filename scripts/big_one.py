"""Kernel time of the default driver on one n x n ctr(seed 1) matrix."""
import sys

import paper_1111_6549_b200 as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
d = G.DeviceMatrix(n, n)
ts = []
for _ in range(2):
    d.fill_ctr(1)
    o = G.block_iterative_ple(d, G.PleConfig(time_kernels=True))
    ts.append(o.stats["kernel_ms"])
print(f"{n}^2: {min(ts):.1f} ms, rank {o.rank}, driver {o.stats['driver']}, "
      f"{o.stats['alg_bytes'] / min(ts) / 1e9:.0f} GB/s effective")
