import sys
import numpy as np
sys.path.insert(0, "tests")
import oracle as O
import suite as S
import paper_1111_6549_b200 as G
for (r, n) in [(65, 1), (65, 2), (65, 64), (66, 1), (128, 1), (129, 1), (130, 65)]:
    rng = np.random.default_rng(r * 31 + n)
    u = S.pack(rng.integers(0, 2, size=(r, r), dtype=np.uint8), r)
    b = O.fill_random(r, n, 0.5, r + n)
    want = b.copy()
    O.trsm_upper(u, r, want, n)
    ub, bb = G.BitMatrix(r, r, u.copy()), G.BitMatrix(r, n, b.copy())
    G.trsm_upper_left_unit(ub, bb)
    bad = np.nonzero((bb.words != want).any(axis=1))[0]
    print(r, n, "bad rows", bad[:10], len(bad))
