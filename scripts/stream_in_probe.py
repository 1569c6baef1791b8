"""The drop-in call (gf2cu_ple on host buffers) with and without streamed
input: end-to-end wall time per call, pinned and pageable host memory, for a
few first-block shares. usage: PYTHONPATH=. python scripts/stream_in_probe.py [n] [fracs...]"""
import os
import sys
import time

import numpy as np
import torch

import paper_1111_6549_b200 as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
# each setting: a GF2CU_STREAM_IN_BLOCKS list, optionally "@T1,T2,.." = GF2CU_STREAM_IN_STEPS
fracs = sys.argv[2:] or ["0.27", "0.0625,0.1875,0.4375", "0.125,0.375", "0.03125,0.09375,0.21875,0.46875"]
W = n // 64
pin = torch.empty((n, W), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
d = G.DeviceMatrix(n, n)
d.fill_ctr(1)
src = np.empty((n, W), dtype=np.uint64)
d.download(src)
want = None


def run(buf, label, reps=4):
    global want
    v = G.MatrixView(buf, W, 0, n, n)
    ts = []
    for it in range(reps):
        buf[:] = src
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        o = G.block_iterative_ple(v)
        ts.append(time.perf_counter() - t0)
    h = G.host_checksum(buf, n)
    if want is None:
        want = (h, o.rank)
    ok = (h, o.rank) == want
    print(f"{label}: {[round(1e3 * t, 2) for t in ts]} ms  rank {o.rank} first block {o.stats['input_first_rows']} rows / "
          f"{o.stats['input_first_steps']} super-steps / {o.stats['input_blocks']} blocks  same result: {ok}", flush=True)


for name, buf in (("pinned", pin), ("pageable", np.empty((n, W), dtype=np.uint64))):
    os.environ["GF2CU_STREAM_IN"] = "0"
    run(buf, f"{name} whole upload")
    os.environ.pop("GF2CU_STREAM_IN", None)  # the default rule: the time model picks the super-steps
    for f in fracs:
        b, _, t = f.partition("@")
        os.environ["GF2CU_STREAM_IN_BLOCKS"] = b
        os.environ.pop("GF2CU_STREAM_IN_STEPS", None)
        if t:
            os.environ["GF2CU_STREAM_IN_STEPS"] = t
        run(buf, f"{name} streamed blocks={f}")
