"""e2e of the drop-in gf2cu_ple on a pinned host view (65536^2 ctr): wall time
per call, H2D + PLE + streamed D2H (as bench.py's e2e)."""
import time

import numpy as np
import torch

import paper_1111_6549_b200 as G

n = 65536
Wd = n // 64
d = G.DeviceMatrix(n, n)
d.fill_ctr(1)
host = torch.empty((n, Wd), dtype=torch.int64, pin_memory=True)
h = host.numpy().view(np.uint64)
d.download(h)
src = h.copy()
view = G.MatrixView(h, Wd, 0, n, n)
ts = []
for it in range(4):
    np.copyto(h, src)
    t0 = time.perf_counter()
    o = G.block_iterative_ple(view, G.PleConfig())
    ts.append(time.perf_counter() - t0)
print("e2e ms per call:", " ".join(f"{1e3 * t:.2f}" for t in ts[1:]), "rank", o.rank)
