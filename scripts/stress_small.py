"""Repeat the small-matrix suite against the oracle and report mismatches
(race hunting); argv[1] = repetitions, argv[2] = driver (single|multi|super)."""
import sys

import numpy as np

sys.path.insert(0, "tests")
import oracle as O  # noqa: E402
import suite as S  # noqa: E402
import paper_1111_6549_b200 as G  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
drv = sys.argv[2] if len(sys.argv) > 2 else "single"
cfg = {"single": G.PleConfig(single_panel=True), "multi": G.PleConfig(multi_kernel=True),
       "super": G.PleConfig(super_step=True)}[drv]
specs = S.suite_specs(260)
cache = {}
bad = []
for rep in range(reps):
    for sp in specs:
        m, n, kind, seed = sp
        if sp not in cache:
            a = S.build(m, n, kind, seed)
            ref = a.copy()
            want = O.ple(ref, m, n)
            cache[sp] = (a, ref, want.rank)
        a, ref, rk = cache[sp]
        bm = G.BitMatrix(m, n, a.copy())
        out = G.block_iterative_ple(bm, cfg)
        if out.rank != rk or not np.array_equal(bm.words, ref):
            bad.append((rep, m, n, kind, seed, out.rank, rk))
print(drv, "reps", reps, "cases", reps * len(specs), "failures", len(bad), bad[:8])
