"""One multi-kernel-driver PLE (so panel_factor is its own launch) for ncu."""
import sys
import paper_1111_6549_b200 as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a = G.DeviceMatrix(n, n)
a.fill_ctr(1)
out = G.block_iterative_ple(a, G.PleConfig(multi_kernel=True))
print("rank", out.rank)
