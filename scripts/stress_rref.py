"""Mimic tests/test_rref_gpu.py::test_rref_from_ple_suite repeatedly (PLE then
rref_from_ple on the same cached device matrix) and log every mismatch."""
import sys

import numpy as np

sys.path.insert(0, "tests")
import oracle as O  # noqa: E402
import suite as S  # noqa: E402
import paper_1111_6549_b200 as G  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
specs = S.suite_specs(260)
cache = {}
bad = []
for rep in range(reps):
    for full in (True, False):
        for sp in specs:
            m, n, kind, seed = sp
            key = (sp, full)
            if key not in cache:
                a = S.build(m, n, kind, seed)
                want = a.copy()
                r = O.echelonize(want, m, n, full)
                ref = a.copy()
                O.ple(ref, m, n)
                cache[key] = (a, want, r, ref)
            a, want, r, ref = cache[key]
            bm = G.BitMatrix(m, n, a.copy())
            out = G.block_iterative_ple(bm)
            ple_ok = out.rank == r and np.array_equal(bm.words, ref)
            G.rref_from_ple(bm, out, full)
            rref_ok = np.array_equal(bm.words, want)
            if not (ple_ok and rref_ok):
                bad.append((rep, full, m, n, kind, seed, out.rank, r, ple_ok, rref_ok))
print("reps", reps, "failures", len(bad))
for b in bad[:20]:
    print(b)
