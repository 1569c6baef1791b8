"""Summarize a GF2CU_DUMP_PHASES file of the super-step driver: per range of
super-steps, the step period, the panel CTA's span and the worker-0 rest sweep.
usage: python scripts/timeline_stats.py gpurun_out/phases65536.txt"""
import sys

import numpy as np

rows = [l.split() for l in open(sys.argv[1]) if l[:1].isdigit()]
a = np.array([[int(x) for x in r] for r in rows], dtype=np.int64)
s = a[a[:, 3] > 0]
t0 = s[0, 3]
p0, p1, r0, r1 = s[:, 3] - t0, s[:, 4] - t0, s[:, 6] - t0, s[:, 8] - t0
dur = np.diff(np.concatenate([[0], r1])) / 1e6
panel = (p1 - p0) / 1e6
rest = (r1 - r0) / 1e6
n = len(s)
edges = [0, 64, 128, 256, 384, 448, 480, n]
for lo, hi in zip(edges[:-1], edges[1:]):
    sel = slice(lo, min(hi, n))
    if lo >= n:
        break
    print(f"S {lo:4d}-{hi:4d}: {dur[sel].sum():7.2f} ms, rest sweep {rest[sel].sum():6.2f} ms, "
          f"avg step {dur[sel].mean() * 1e3:6.1f} us, avg panel span {panel[sel].mean() * 1e3:5.1f} us")
print(f"total {dur.sum():.2f} ms over {n} super-steps")
