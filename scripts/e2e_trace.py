"""Timeline of one drop-in call (gf2cu_ple on a pinned host buffer): host
timestamps and stream events, GF2CU_TRACE=1 (gf2cu.cu, Trace).
usage: PYTHONPATH=. python scripts/e2e_trace.py [n] [pageable]"""
import os
import sys

import numpy as np
import torch

import paper_1111_6549_b200 as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
W = n // 64
if len(sys.argv) > 2:
    buf = np.empty((n, W), dtype=np.uint64)
else:
    buf = torch.empty((n, W), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
d = G.DeviceMatrix(n, n)
d.fill_ctr(1)
src = np.empty((n, W), dtype=np.uint64)
d.download(src)
v = G.MatrixView(buf, W, 0, n, n)
for it in range(3):
    buf[:] = src
    torch.cuda.synchronize()
    if it == 2:
        os.environ["GF2CU_TRACE"] = "1"
    o = G.block_iterative_ple(v)
print("rank", o.rank, o.stats)
