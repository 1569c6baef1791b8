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
