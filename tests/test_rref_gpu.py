"""GPU parity of the echelon-form row through the C ABI:
rref_from_ple (ple.hpp:318-329), extract_e (:344-352),
echelonize(ple_iterative) (m4ri.hpp:95-98) and trsm_upper_left_unit
(multiply.hpp:314-335) vs the oracle restatements (orc_echelonize,
orc_trsm_upper; pinned to the compiled reference in tests/test_rref_host.py).
Bit-exact: the reduced form is unique and the echelon form is the PLE's E."""
import numpy as np
import pytest

import oracle as O
import paper_1111_6549_b200 as G
import suite as S

pytestmark = pytest.mark.gpu


def oracle_echelon(a, m, n, full):
    want = a.copy()
    r = O.echelonize(want, m, n, full)
    return want, r


@pytest.mark.parametrize("full", [True, False])
def test_rref_from_ple_suite(full):
    for (m, n, kind, seed) in S.suite_specs(260):
        a = S.build(m, n, kind, seed)
        want, r = oracle_echelon(a, m, n, full)
        bm = G.BitMatrix(m, n, a.copy())
        out = G.block_iterative_ple(bm)
        assert out.rank == r
        G.rref_from_ple(bm, out, full)
        assert np.array_equal(bm.words, want), (m, n, kind, seed, full)


@pytest.mark.parametrize("m,n,kind", [(1, 1, "dense"), (64, 80, "dense"), (65, 65, "thin"),
                                      (200, 1000, "dense"), (1000, 200, "dense"),
                                      (1024, 1024, "dense"), (1500, 2500, "sparse64"),
                                      (2048, 2048, "sparse256"), (2048, 6000, "ctr"),
                                      (4096, 4096, "ctr"), (3000, 3000, "deficient")])
@pytest.mark.parametrize("full", [True, False])
def test_echelonize(m, n, kind, full):
    seed = m + 7 * n
    if kind == "dense":
        a = O.fill_random(m, n, 0.5, seed)
    elif kind == "thin":
        a = O.fill_random(m, n, 0.08, seed)
    elif kind == "sparse64":
        a = O.fill_random(m, n, 1 / 64, seed)
    elif kind == "sparse256":
        a = O.fill_random(m, n, 1 / 256, seed)
    elif kind == "ctr":
        a = O.fill_ctr(m, n, seed)
    else:  # rank-deficient: duplicated rows and a zero column band
        a = O.fill_ctr(m, n, seed)
        a[m // 2:] = a[: m - m // 2]
        a[:, 5] = 0
    want, r = oracle_echelon(a, m, n, full)
    bm = G.BitMatrix(m, n, a.copy())
    assert G.echelonize(bm, full) == r
    assert np.array_equal(bm.words, want), (m, n, kind, full)


def test_device_resident_rref():
    m = n = 4096
    dm = G.DeviceMatrix(m, n)
    dm.fill_ctr(3)
    a = O.fill_ctr(m, n, 3)
    want, r = oracle_echelon(a, m, n, True)
    out = G.block_iterative_ple(dm)
    assert out.rank == r
    G.rref_from_ple(dm, out, True)
    assert np.array_equal(dm.download(), want)
    dm.fill_ctr(3)
    assert G.echelonize(dm, True) == r
    assert np.array_equal(dm.download(), want)


def test_unaligned_view():
    parent = O.fill_random(300, 384, 0.5, 5)  # 6 words per row
    m, n, off = 300, 250, 37
    view_bits = S.unpack(parent, 384)[:, off:off + n]
    a = S.pack(view_bits, n)
    want, r = oracle_echelon(a, m, n, True)
    work = parent.copy()
    v = G.MatrixView(work, 6, off, m, n)
    assert G.echelonize(v, True) == r
    got_bits = S.unpack(work, 384)
    assert np.array_equal(S.pack(got_bits[:, off:off + n], n), want)
    before = S.unpack(parent, 384)
    assert np.array_equal(got_bits[:, :off], before[:, :off])
    assert np.array_equal(got_bits[:, off + n:], before[:, off + n:])


def test_extract_e():
    for (m, n, seed) in [(100, 300, 1), (300, 100, 2), (257, 193, 3), (1200, 1100, 4)]:
        a = O.fill_random(m, n, 0.5, seed)
        want, r = oracle_echelon(a, m, n, False)
        bm = G.BitMatrix(m, n, a.copy())
        out = G.block_iterative_ple(bm)
        before = bm.words.copy()
        e = G.extract_e(bm, out)
        assert np.array_equal(bm.words, before)  # input untouched
        assert e.nrows() == r and np.array_equal(e.words, want[:r])


def test_known_answers():
    # full-rank square -> identity (test_ple.cpp:265-277)
    tested = 0
    for seed in range(64):
        a = O.fill_random(50, 50, 0.5, seed)
        bm = G.BitMatrix(50, 50, a)
        out = G.block_iterative_ple(bm)
        if out.rank != 50:
            continue
        G.rref_from_ple(bm, out, True)
        assert bm == G.BitMatrix.identity(50)
        tested += 1
        if tested == 5:
            break
    assert tested == 5
    # rank zero (test_ple.cpp:279-285)
    z = G.BitMatrix(6, 9)
    out = G.block_iterative_ple(z)
    G.rref_from_ple(z, out, True)
    assert out.rank == 0 and not z.words.any()
    # identity (test_ple.cpp:347): rank 33
    i33 = G.BitMatrix.identity(33)
    assert G.echelonize(i33, True) == 33 and i33 == G.BitMatrix.identity(33)


def test_rejects_corrupt_outcome():
    # check_pivots (ple.hpp:299-307; test_ple.cpp:305-314)
    bm = G.BitMatrix(10, 10, O.fill_random(10, 10, 0.5, 5))
    out = G.block_iterative_ple(bm)
    assert out.rank >= 2
    out.q = out.q.copy()
    out.q[[0, 1]] = out.q[[1, 0]]
    with pytest.raises(ValueError):
        G.rref_from_ple(bm, out, True)


@pytest.mark.parametrize("r,n", [(1, 5), (2, 64), (63, 70), (64, 64), (65, 1), (129, 200), (200, 129),
                                 (300, 33), (1000, 1000), (4096, 130), (2000, 5000)])
def test_trsm_upper_left_unit(r, n):
    rng = np.random.default_rng(r * 31 + n)
    u = S.pack(rng.integers(0, 2, size=(r, r), dtype=np.uint8), r)
    b = O.fill_random(r, n, 0.5, r + n)
    want = b.copy()
    O.trsm_upper(u, r, want, n)
    ub, bb = G.BitMatrix(r, r, u.copy()), G.BitMatrix(r, n, b.copy())
    G.trsm_upper_left_unit(ub, bb)
    assert np.array_equal(bb.words, want), (r, n)
    assert np.array_equal(ub.words, u)


def test_trsm_dimension_mismatch():
    with pytest.raises(ValueError):
        G.trsm_upper_left_unit(G.BitMatrix(3, 4), G.BitMatrix(3, 5))
    with pytest.raises(ValueError):
        G.trsm_upper_left_unit(G.BitMatrix(3, 3), G.BitMatrix(4, 5))


def rowspace_check(a, r_words, m, n, q, trials=4, seed=0):
    """rowspace(A) within rowspace(R) on random combinations (R in RREF with
    pivots q), plus R's pivot columns form the identity on its top rows."""
    rng = np.random.default_rng(seed)
    rank = len(q)
    qa = np.asarray(q, dtype=np.int64)
    pw, pb = qa >> 6, (qa & 63).astype(np.uint64)
    top = r_words[:rank]
    bits = (top[:, pw] >> pb[None, :]) & np.uint64(1)
    assert np.array_equal(bits, np.eye(rank, dtype=np.uint64))
    assert not r_words[rank:].any()
    for _ in range(trials):
        sel = rng.integers(0, 2, size=m).astype(bool)
        v = np.bitwise_xor.reduce(a[sel], axis=0) if sel.any() else np.zeros(a.shape[1], np.uint64)
        coef = ((v[pw] >> pb) & np.uint64(1)).astype(bool)
        red = v ^ (np.bitwise_xor.reduce(top[coef], axis=0) if coef.any() else 0)
        assert not np.any(red), "a row combination of A is not in the row space of R"


@pytest.mark.slow
def test_large_rowspace_property():
    m = n = 16384
    a = O.fill_ctr(m, n, 1)
    bm = G.BitMatrix(m, n, a.copy())
    out = G.block_iterative_ple(bm)
    G.rref_from_ple(bm, out, True)
    rowspace_check(a, bm.words, m, n, [int(x) for x in out.q])
