"""CPU: the echelon-form row of SURVEY.md 8(f) #1 before the device runs it.

1. Pin the oracle restatements (orc_echelonize = naive_echelonize,
   orc_trsm_upper = trsm_upper_left_unit) against the compiled reference
   (ref_echelonize for every strategy, ref_trsm_upper_left_unit).
2. Check the two facts the device design rests on,
   with a numpy model of the kernels, against the reference's own
   rref_from_ple on reference PLE outputs:
   - the closed form of undo_column_swaps + zero_below_pivots on a genuine
     PLE state (rows < rank: columns <= q_i cleared, bit q_i set; rows below
     zero);
   - the reduced form computed in pivot-first column coordinates
     (X = U^-1 N, R_i = e_{q_i} + X_i on the non-pivot columns).
3. The reference's known answers: full-rank square -> identity
   (test_ple.cpp:265-277), rank zero (:279-285).
"""
import numpy as np
import pytest

import oracle as O
import suite as S

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def cases():
    out = []
    for i, (m, n, kind, seed) in enumerate(S.suite_specs(120)):
        out.append((m, n, kind, seed))
    out += [(64, 80, 2, 7), (200, 500, 3, 8), (500, 200, 2, 9), (130, 130, 4, 10)]
    return out


@pytest.mark.parametrize("full", [True, False])
def test_echelonize_oracle_matches_reference(full):
    for (m, n, kind, seed) in cases():
        a = S.build(m, n, kind, seed)
        want = a.copy()
        r_ref = O.ref_echelonize(want, m, n, "naive", full)
        for strat in ("ple_iterative", "m4ri"):
            b = a.copy()
            assert O.ref_echelonize(b, m, n, strat, full) == r_ref
            if full:  # the reduced form is unique
                assert np.array_equal(b, want), (m, n, kind, strat)
        got = a.copy()
        assert O.echelonize(got, m, n, full) == r_ref
        assert np.array_equal(got, want), (m, n, kind, full)


def random_upper(r, seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, size=(r, r), dtype=np.uint8)
    return S.pack(bits, r)


def test_trsm_oracle_matches_reference():
    for (r, n, seed) in [(1, 5, 1), (2, 64, 2), (63, 70, 3), (64, 64, 4), (65, 1, 5), (129, 200, 6),
                         (200, 129, 7), (300, 33, 8)]:
        u = random_upper(r, seed)
        b = O.fill_random(r, n, 0.5, seed + 100)
        want = b.copy()
        O.ref_trsm_upper_left_unit(u, r, want, n)
        got = b.copy()
        O.trsm_upper(u, r, got, n)
        assert np.array_equal(got, want), (r, n)


# ---------------------------------------------------------------- host model
def closed_form_echelon(a, m, n, q):
    """The device's rref_echelon_kernel, in numpy."""
    bits = S.unpack(a, n)
    r = len(q)
    out = np.zeros_like(bits)
    for i in range(r):
        row = bits[i].copy()
        row[: q[i] + 1] = 0
        row[q[i]] = 1
        out[i] = row
    return S.pack(out, n)


def pivot_coordinate_rref(a, m, n, q):
    """The device's gather -> blocked back-substitution -> scatter, in numpy."""
    bits = S.unpack(a, n)
    r = len(q)
    piv = np.array(q, dtype=np.int64)
    nonp = np.array([c for c in range(n) if c not in set(q)], dtype=np.int64)
    E = np.zeros((r, n), dtype=np.uint8)
    for i in range(r):
        E[i] = bits[i]
        E[i, : q[i] + 1] = 0
        E[i, q[i]] = 1
    U = E[:, piv] if r else np.zeros((0, 0), np.uint8)
    N = E[:, nonp].copy() if r else np.zeros((0, len(nonp)), np.uint8)
    X = N.copy()
    # bottom-up 64-row blocks: in-block solve, then update the rows above
    R = (r + 63) // 64 * 64
    for J in range(R // 64 - 1, -1, -1):
        lo, hi = 64 * J, min(64 * J + 64, r)
        for t in range(hi - 1, lo - 1, -1):
            for j in range(t + 1, hi):
                if U[t, j]:
                    X[t] ^= X[j]
        for i in range(lo):
            for j in range(lo, hi):
                if U[i, j]:
                    X[i] ^= X[j]
    out = np.zeros((m, n), dtype=np.uint8)
    for i in range(r):
        out[i, q[i]] = 1
        out[i, nonp] = X[i]
    return S.pack(out, n)


def test_closed_forms_match_reference_rref_from_ple():
    for (m, n, kind, seed) in cases()[:80] + [(150, 300, 3, 11), (300, 150, 5, 12)]:
        a = S.build(m, n, kind, seed)
        dec = a.copy()
        out, _ = O.ref_ple(dec, m, n)
        q = [int(x) for x in out.q]
        for full in (False, True):
            want = dec.copy()
            O.ref_rref_from_ple(want, m, n, out, full)
            got = closed_form_echelon(dec, m, n, q) if not full else pivot_coordinate_rref(dec, m, n, q)
            assert np.array_equal(got, want), (m, n, kind, full)
            # the oracle the GPU tests use: naive_echelonize on the original
            orc = a.copy()
            assert O.echelonize(orc, m, n, full) == out.rank
            assert np.array_equal(orc, want), (m, n, kind, full)


def test_known_answers():
    # full-rank square -> identity (test_ple.cpp:265-277)
    tested = 0
    for seed in range(64):
        a = O.fill_random(50, 50, 0.5, seed)
        if O.ref_echelonize(a.copy(), 50, 50, "naive", True) != 50:
            continue
        got = a.copy()
        assert O.echelonize(got, 50, 50, True) == 50
        assert np.array_equal(got, S.pack(np.eye(50, dtype=np.uint8), 50))
        tested += 1
        if tested == 5:
            break
    assert tested == 5
    # rank zero (test_ple.cpp:279-285)
    z = np.zeros((6, 1), dtype=np.uint64)
    assert O.echelonize(z, 6, 9, True) == 0 and not z.any()


def test_strategy_equivalences_pinned():
    """What lets one device path serve recursive_ple and every echelonize
    strategy: recursive_ple's in-place result, rank, q and p.swaps equal
    block_iterative_ple's for any recursion cut-off, and the non-reduced
    forms of naive / m4ri / ple_iterative / ple_recursive coincide."""
    for (m, n, kind, seed) in cases()[:100] + [(500, 500, 2, 1), (300, 900, 3, 2), (900, 300, 2, 3)]:
        a = S.build(m, n, kind, seed)
        x = a.copy()
        o1, _ = O.ref_ple(x, m, n)
        for bb, bn in [(0, 0), (512, 32), (8 << 10, 0)]:
            y = a.copy()
            o2 = O.ref_recursive_ple(y, m, n, base_bytes=bb, base_ncols=bn)
            assert np.array_equal(x, y) and o1.rank == o2.rank, (m, n, kind)
            assert np.array_equal(o1.q, o2.q) and np.array_equal(o1.swaps, o2.swaps), (m, n, kind)
        forms = []
        for strat in ("naive", "m4ri", "ple_iterative", "ple_recursive"):
            u = a.copy()
            O.ref_echelonize(u, m, n, strat, False)
            forms.append(u)
        assert all(np.array_equal(forms[0], f) for f in forms[1:]), (m, n, kind)


def test_mul_oracle_matches_reference():
    for (m, l, n, seed) in [(1, 1, 1, 1), (3, 70, 5, 2), (64, 64, 64, 3), (65, 129, 63, 4),
                            (200, 300, 100, 5), (130, 1, 70, 6)]:
        a = O.fill_random(m, l, 0.5, seed)
        b = O.fill_random(l, n, 0.5, seed + 1)
        assert np.array_equal(O.mul(a, l, b, n), O.ref_mul(a, l, b, n)), (m, l, n)
