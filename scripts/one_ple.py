"""One device-resident PLE of the n x n ctr(seed 1) matrix (profiling target)."""
import sys

import paper_1111_6549_b200 as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
dm = G.DeviceMatrix(n, n)
dm.fill_ctr(1)
out = G.block_iterative_ple(dm)
print("rank", out.rank, "driver", out.stats["driver"], "alg_bytes(k64)", out.stats["alg_bytes"],
      "sweep_bytes", out.stats["sweep_bytes"])
