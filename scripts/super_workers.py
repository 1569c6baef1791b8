"""Per-worker timeline of the super-step driver (GF2CU_DUMP_WORKERS): where the
workers' time goes per super-step -- pre-work, barrier wait, rest sweep, and
the end-of-step spread (max rest end - each worker's rest end) that work
stealing could recover.
usage: python scripts/super_workers.py [n] [dumpfile]"""
import os
import sys

import numpy as np

import paper_1111_6549_b200 as G

arg = sys.argv[1] if len(sys.argv) > 1 else "65536"
m, n = (int(x) for x in arg.split("x")) if "x" in arg else (int(arg), int(arg))
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/workers_super.bin"
if n > 0:
    a = G.DeviceMatrix(m, n)
    b = G.DeviceMatrix(m, n)
    b.fill_ctr(1)
    for it in range(3):
        a.copy_from(b)
        if it == 2:
            os.environ["GF2CU_DUMP_WORKERS"] = out
        o = G.block_iterative_ple(a, G.PleConfig(time_kernels=True, super_step=True))
    print("stats", o.stats)

raw = np.fromfile(out, dtype=np.uint64)
W, nw, per = int(raw[0]), int(raw[1]), int(raw[2])
d = raw[3:].reshape(W + 1, nw, per).astype(np.int64)
ok = (d[:, :, 0] > 0).all(axis=1) & (d[:, :, 3] > 0).all(axis=1)
d = d[ok]
t0 = d[0, :, 0].min()
d = d - t0
wake, pre, rs, re = d[:, :, 0], d[:, :, 1], d[:, :, 2], d[:, :, 3]
ns = len(d)
endmax = re.max(axis=1)
prev_end = np.concatenate([[0], endmax[:-1]])
tot = endmax[-1] / 1e6
print(f"{ns} super-steps, {nw} workers, total {tot:.2f} ms (first wake -> last rest end)")
comp = {
    "wait for panel (prev max end -> wake)": (wake - prev_end[:, None]).clip(0).mean(axis=1),
    "pre-work": (pre - wake).mean(axis=1),
    "barrier wait (pre-work end -> rest start)": (rs - pre).mean(axis=1),
    "rest sweep": (re - rs).mean(axis=1),
    "end spread (max end - own end)": (endmax[:, None] - re).mean(axis=1),
}
for k, v in comp.items():
    print(f"  {k:45s} {v.sum() / 1e6:8.2f} ms")
edges = [0, 32, 64, 128, 256, 384, 448, 480, 512, ns]
for lo, hi in zip(edges[:-1], edges[1:]):
    if lo >= ns:
        break
    hi = min(hi, ns)
    sel = slice(lo, hi)
    per_step = (endmax[sel] - prev_end[sel]).mean() / 1e3
    print(f"  S {lo:4d}-{hi:4d}: step {per_step:7.1f} us | " + " | ".join(
        f"{v[sel].mean() / 1e3:6.1f}" for v in comp.values()))
