"""Print where the device PLE differs from the oracle for one small shape."""
import sys

import numpy as np

sys.path.insert(0, "tests")
import oracle as O  # noqa: E402
import paper_1111_6549_b200 as G  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
a = O.fill_random(m, n, 0.5, 7)
ref = a.copy()
want = O.ple(ref, m, n)
bm = G.BitMatrix(m, n, a.copy())
got = G.block_iterative_ple(bm)
print("rank", got.rank, want.rank, "q same", np.array_equal(got.q, want.q.astype(np.uint64)),
      "swaps same", np.array_equal(got.p.swaps, want.swaps.astype(np.uint64)))
bad = np.argwhere(bm.words != ref)
print("differing words:", len(bad))
rows = sorted(set(int(i) for i, _ in bad))
print("rows:", rows[:40])
cols = sorted(set(int(x) for _, x in bad))
print("word cols:", cols[:20])
for i, x in bad[:6]:
    print(i, x, hex(int(bm.words[i, x])), hex(int(ref[i, x])))
