"""Per-step breakdown from a GF2CU_DUMP_WORKERS file: mean rest, end spread, gap."""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64)
W, nw = int(raw[0]), int(raw[1])
d = raw[2:].reshape(W + 1, nw, 2).astype(np.int64)
st, en = d[:W, :, 0], d[:W, :, 1]
valid = (st[:, 0] > 0) & (en[:, 0] > 0)
st, en = st[valid], en[valid]
period = np.diff(en.max(axis=1)) / 1e3
mean_rest = ((en - st).mean(axis=1) / 1e3)[1:]
spread = ((en.max(axis=1) - en.mean(axis=1)) / 1e3)[1:]
gap = (st.min(axis=1)[1:] - en.max(axis=1)[:-1]) / 1e3
gapm = (st.mean(axis=1)[1:] - en.max(axis=1)[:-1]) / 1e3
print("total %.2f ms; mean rest %.2f; spread %.2f; gap(min start) %.2f; gap(mean start) %.2f"
      % (period.sum() / 1e3, mean_rest.sum() / 1e3, spread.sum() / 1e3, gap.sum() / 1e3, gapm.sum() / 1e3))
for w in [10, 100, 300, 600, 900, 1000]:
    if w - 1 < len(period):
        print(f" step {w}: period {period[w-1]:.1f} mean rest {mean_rest[w-1]:.1f} spread {spread[w-1]:.1f} "
              f"gap {gap[w-1]:.1f} gapmean {gapm[w-1]:.1f}")
