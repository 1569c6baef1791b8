"""CPU: pin the oracle (oracle/ple_oracle.c) before trusting it.

1. against the golden fixtures produced by the compiled reference
   (tests/golden/*.json, script tests/golden/make_golden.py);
2. against the compiled reference itself (oracle/_ref) on fresh random cases,
   across the reference's stripe widths k and table counts (its output is
   k-independent);
3. the reference's own known answers for this path (test_ple.cpp:74-95,
   208-222; acceptance_main.cpp:376-397).
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import suite as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def words_from_hex(rows):
    return np.array([[int(x, 16) for x in r.split()] for r in rows], dtype=np.uint64)


def test_generators_match_reference():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for (m, n, d, seed) in [(5, 70, 0.5, 1), (33, 129, 0.08, 99), (64, 64, 1 / 256, 5), (7, 3, 1.0, 2),
                            (9, 200, 0.0, 3)]:
        assert np.array_equal(O.fill_random(m, n, d, seed), O.ref_fill_random(m, n, d, seed))
    for (m, n, nnz, seed) in [(10, 100, 3, 1), (10, 100, 80, 2), (20, 65, 65, 3), (4, 1, 1, 4)]:
        assert np.array_equal(O.fill_random_rows(m, n, nnz, seed), O.ref_fill_random_rows(m, n, nnz, seed))


def test_small_golden_fixtures():
    for c in load("small.json")["cases"]:
        m, n = c["m"], c["n"]
        a = words_from_hex(c["input"])
        out = O.ple(a, m, n)
        assert np.array_equal(a, words_from_hex(c["output"])), c["name"]
        assert out.rank == c["rank"], c["name"]
        assert list(out.swaps) == c["swaps"] and list(out.q) == c["q"], c["name"]


def test_small_golden_known_answers():
    cases = {c["name"]: c for c in load("small.json")["cases"]}
    # identity stays put, rank n, trivial P and Q, no column swaps (test_ple.cpp:84-95)
    c = cases["identity_33"]
    assert c["rank"] == 33 and c["swaps"] == list(range(33)) and c["q"] == list(range(33))
    assert c["output"] == c["input"] and c["ref_col_swaps"] == []
    # zero matrix: rank 0, untouched (test_ple.cpp:74-82)
    c = cases["zero_6x9"]
    assert c["rank"] == 0 and c["output"] == c["input"]
    # section 3.2 worked example: the row [1 0 1 ...] gets multipliers [1 0 0]
    # w.r.t. the three pivot rows (acceptance_main.cpp:376-397)
    c = cases["sec32_multipliers"]
    out = words_from_hex(c["output"])
    row3 = [(int(out[3, 0]) >> j) & 1 for j in range(3)]
    assert row3 == [1, 0, 0]


def test_suite_golden_hashes():
    for e in load("suite.json")["cases"]:
        a = S.build(e["m"], e["n"], e["kind"], e["seed"])
        out = O.ple(a, e["m"], e["n"])
        assert out.rank == e["rank"], e
        assert S.outcome_hash(a, e["n"], out.rank, out.swaps, out.q) == e["sha256"], e


@pytest.mark.parametrize("seed", range(6))
def test_oracle_vs_reference_random(seed):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(1000 + seed)
    for _ in range(25):
        m, n = int(rng.integers(1, 260)), int(rng.integers(1, 260))
        kind = int(rng.integers(0, 7))
        a = S.build(m, n, kind, int(rng.integers(0, 2**62)))
        b = a.copy()
        oa = O.ple(a, m, n)
        ob, _ = O.ref_ple(b, m, n, k=int(rng.integers(0, 17)), table_count=int(rng.choice([1, 2, 4, 8])))
        assert np.array_equal(a, b)
        assert oa.rank == ob.rank and np.array_equal(oa.swaps, ob.swaps) and np.array_equal(oa.q, ob.q)


def test_canonical_col_swaps_accepted_by_reference():
    """extract_e / rref_from_ple give identical results with the canonical
    compression list {j, q[j], j} and with the reference's own k-dependent list."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    for _ in range(40):
        m, n = int(rng.integers(2, 200)), int(rng.integers(2, 200))
        a = S.build(m, n, int(rng.integers(2, 7)), int(rng.integers(0, 2**62)))
        b = a.copy()
        ob, _ = O.ref_ple(b, m, n, k=int(rng.integers(1, 17)))
        canon = O.Outcome(ob.rank, ob.swaps, ob.q, O.canonical_col_swaps(ob.q))
        assert np.array_equal(O.ref_extract_e(b, m, n, ob), O.ref_extract_e(b, m, n, canon))
        r1, r2 = b.copy(), b.copy()
        O.ref_rref_from_ple(r1, m, n, ob)
        O.ref_rref_from_ple(r2, m, n, canon)
        assert np.array_equal(r1, r2)
        assert O.ref_reconstructs(a, b, m, n, canon)


def test_oracle_properties_medium():
    """P*L*E == A and the rank/q agree with the reference at a medium size."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    m = n = 1500
    a = O.fill_ctr(m, n, 5)
    b = a.copy()
    oa = O.ple(b, m, n)
    assert O.ref_reconstructs(a, b, m, n, oa)


def partial_processed_rule(m, n, rank, swaps, q):
    """The rule gf2cu_partial_ple applies (csrc/gf2cu.cu partial_processed):
    processed < m only when rank < m and the pivot columns run consecutively
    from q[0] to column n-1 (empty columns before q[0] do not count)."""
    if rank == 0:
        return 0
    q = [int(x) for x in q]
    if rank >= m or q[-1] != n - 1 or q[-1] - q[0] != rank - 1:
        return m
    return max(rank, int(max(swaps)) + 1)


def _partial_cases():
    rng = np.random.default_rng(2026)
    for i in range(600):
        m, n = int(rng.integers(1, 140)), int(rng.integers(1, 140))
        if i % 3 == 0:  # tall: full column rank is likely, so the lazy pass stops early
            n = int(rng.integers(1, 40))
            m = n + int(rng.integers(1, 100))
        kind = i % 7
        a = S.build(m, n, kind, int(rng.integers(0, 2**62)))
        if i % 5 == 1 and n > 2:  # empty leading columns (read while r = 0)
            lead = int(rng.integers(1, n))
            for c in range(lead):
                a[:, c >> 6] &= ~np.uint64(1 << (c & 63))
        yield m, n, a


def test_partial_ple_tiny_exhaustive():
    """Every 2x3, 3x2 and 3x3 matrix (and the reference's
    ColumnRankProfile sizes): restatement == compiled reference."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for (m, n) in [(2, 3), (3, 2), (3, 3), (4, 2)]:
        for bits in range(1 << (m * n)):
            a = np.zeros((m, 1), dtype=np.uint64)
            for i in range(m):
                for j in range(n):
                    if (bits >> (i * n + j)) & 1:
                        a[i, 0] |= np.uint64(1 << j)
            x, y = a.copy(), a.copy()
            got, gp = O.partial_ple(x, m, n)
            want, wp = O.ref_partial_ple(y, m, n)
            assert (got.rank, gp) == (want.rank, wp) and np.array_equal(x, y), (m, n, bits)
            assert partial_processed_rule(m, n, want.rank, want.swaps, want.q) == wp, (m, n, bits)


def test_partial_ple_restatement_vs_reference():
    """orc_partial_ple (the watermark restatement) == the compiled reference's
    partial_ple: words, rank, swaps, q, processed; and the processed rule the
    device path uses reproduces the reference's watermark."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    early = 0
    for m, n, a in _partial_cases():
        x, y = a.copy(), a.copy()
        got, gp = O.partial_ple(x, m, n)
        want, wp = O.ref_partial_ple(y, m, n)
        assert (got.rank, gp) == (want.rank, wp), (m, n)
        assert np.array_equal(got.swaps, want.swaps) and np.array_equal(got.q, want.q), (m, n)
        assert np.array_equal(x, y), (m, n)
        assert partial_processed_rule(m, n, want.rank, want.swaps, want.q) == wp, (m, n)
        if wp < m:
            early += 1
            # rows past the watermark are untouched apart from the recorded
            # column swaps (acceptance_main.cpp:127-139)
            tail = a[wp:].copy()
            cs = want.col_swaps.astype(np.uintp).reshape(-1, 3)[::-1].copy()
            cs[:, 2] = 0  # (every swap starts above the tail)
            O.undo_col_swaps(tail, m - wp, cs)  # reversed list, replayed backwards = forward
            assert np.array_equal(y[wp:], tail)
        # rank / q / swaps are the complete decomposition's
        z = a.copy()
        full = O.ple(z, m, n)
        assert full.rank == want.rank and np.array_equal(full.q, want.q)
        assert np.array_equal(full.swaps, want.swaps)
        assert np.array_equal(z[:wp], y[:wp])
    assert early > 20  # the lazy early stop is exercised
