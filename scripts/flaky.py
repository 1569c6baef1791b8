"""Repeat small PLEs against the oracle and count mismatches (race hunting)."""
import sys

import numpy as np

sys.path.insert(0, "tests")
import oracle as O  # noqa: E402
import paper_1111_6549_b200 as G  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
bad = {}
shapes = [(128, 128), (127, 129), (129, 127), (150, 300), (64, 64), (257, 193), (1000, 200)]
for rep in range(reps):
    for (m, n) in shapes:
        seed = m * 1000 + n
        a = O.fill_random(m, n, 0.5, seed)
        rng = np.random.default_rng(seed)
        for _ in range(4):
            d, s = rng.integers(0, m, 2)
            a[d] = a[s]
        ref = a.copy()
        want = O.ple(ref, m, n)
        bm = G.BitMatrix(m, n, a.copy())
        got = G.block_iterative_ple(bm)
        ok = got.rank == want.rank and np.array_equal(bm.words, ref) and np.array_equal(got.q, want.q.astype(np.uint64))
        if not ok:
            bad[(m, n)] = bad.get((m, n), 0) + 1
print("reps", reps, "failures", bad)
