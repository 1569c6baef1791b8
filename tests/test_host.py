"""CPU: host-side logic of the mirror interface and the bench accounting."""
import numpy as np

import paper_1111_6549_b200 as G


def test_row_permutation_lapack_vector():
    # P = [0 2 2 4 4] applied to I yields rows e0 e2 e1 e4 e3 (test_bit_matrix.cpp:195-205)
    p = G.RowPermutation(np.array([0, 2, 2, 4, 4], dtype=np.uint64))
    a = np.eye(5, dtype=np.uint8)
    p.apply(a)
    assert [int(np.argmax(r)) for r in a] == [0, 2, 1, 4, 3]
    p.apply_inverse(a)
    assert np.array_equal(a, np.eye(5, dtype=np.uint8))


def test_row_permutation_validate():
    import pytest
    with pytest.raises(ValueError):
        G.RowPermutation(np.array([1, 0], dtype=np.uint64)).validate(2)


def test_bitmatrix_roundtrip():
    rows = ["10010111", "01011110", "00100111"]
    a = G.BitMatrix.from_rows(rows)
    assert [a.row_string(i) for i in range(3)] == rows
    assert a.view().sub(1, 2, 2, 3).get(0, 0) == a.get(1, 2)
    b = G.BitMatrix.identity(70)
    assert b.get(69, 69) and not b.get(0, 69)


def test_host_checksum_matches_definition():
    a = np.arange(12, dtype=np.uint64).reshape(3, 4)
    h = G.host_checksum(a, 200)
    # recompute by the definition
    P = 0x100000001B3
    M = (1 << 64) - 1
    acc = 0xCBF29CE484222325
    for row in a:
        r = 0xCBF29CE484222325
        for x in row[:4]:
            r = ((r ^ int(x)) * P) & M
        acc = ((acc ^ r) * P) & M
    assert h == acc


def test_bench_alg_bytes_definition():
    import bench
    # m = n = 128: W = 2; step 0 finds 64 pivots, step 1 is the last panel (no tail)
    assert bench.alg_bytes_from_history(128, 128, [0, 64], [64, 64]) == 16 * (128 - 64) * 1


def _plan(m, W, pageable=False):
    import ctypes as C
    from paper_1111_6549_b200 import _lib
    lib = _lib.load()
    rows = (C.c_size_t * 8)()
    steps = (C.c_uint * 8)()
    n = C.c_size_t(0)
    _lib.check(lib.gf2cu_stream_in_plan(m, W, int(pageable), rows, steps, C.byref(n)))
    return list(rows[: n.value]), list(steps[: n.value])


def test_stream_in_plan_invariants(monkeypatch):
    """The row-block plan of the streamed input (run on the host, no device):
    blocks grow, end at m, every phase keeps a full window and a full next
    window among its rows, super-steps never decrease; the knobs are obeyed and
    shapes that cannot profit get no plan."""
    for v in ("GF2CU_STREAM_IN", "GF2CU_STREAM_IN_BLOCKS", "GF2CU_STREAM_IN_FRAC", "GF2CU_STREAM_IN_STEPS"):
        monkeypatch.delenv(v, raising=False)

    def check(m, W, rows, steps):
        nss = (W + 1) // 2
        assert rows[-1] == m and steps[0] == 0 and len(rows) == len(steps) <= 8
        assert all(a < b for a, b in zip(rows, rows[1:])) and all(a <= b for a, b in zip(steps, steps[1:]))
        assert all(r % 256 == 0 for r in rows[:-1]) and rows[0] >= 512
        for k in range(1, len(rows)):
            assert steps[k] <= (rows[k - 1] - 256) // 128 and steps[k] <= nss - 1

    # BASELINE config 5, default rule: four geometric blocks, a few dozen super-steps
    for pageable in (False, True):
        rows, steps = _plan(65536, 1024, pageable)
        assert rows == [4096, 12288, 28672, 65536], rows
        check(65536, 1024, rows, steps)
        assert 8 <= steps[-1] <= 120
    rows, steps = _plan(131072, 2048)
    check(131072, 2048, rows, steps)
    # small matrices and shapes without room for a block: uploaded whole
    assert _plan(2048, 32) == ([], [])
    assert _plan(0, 0) == ([], [])
    assert _plan(300, 100000) == ([], [])
    # forced on (tests): as many super-steps per block as its rows allow
    monkeypatch.setenv("GF2CU_STREAM_IN", "1")
    rows, steps = _plan(4096, 64)
    check(4096, 64, rows, steps)
    assert steps[1] == (rows[0] - 256) // 128
    monkeypatch.setenv("GF2CU_STREAM_IN_BLOCKS", "0.5,0.2,0.9,7,abc")  # unsorted, out of range, junk
    rows, steps = _plan(8192, 128)
    check(8192, 128, rows, steps)
    monkeypatch.setenv("GF2CU_STREAM_IN_BLOCKS", "0.125,0.375,0.625")
    monkeypatch.setenv("GF2CU_STREAM_IN_STEPS", "2,1,100000")  # decreasing and too large: clamped
    rows, steps = _plan(8192, 128)
    check(8192, 128, rows, steps)
    assert steps[1] == 2 and steps[2] == 2
    monkeypatch.setenv("GF2CU_STREAM_IN", "0")
    assert _plan(65536, 1024) == ([], [])
