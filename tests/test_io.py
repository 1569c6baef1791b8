"""CPU: gf2b / ASCII files (io.hpp:14-124) against the
reference's own save/load (oracle/_ref), byte for byte, including every
rejection the reference makes; the CLI's usage / I/O exit codes; the host
fill_random_rows against the reference's."""
import io
import os

import numpy as np
import pytest

import oracle as O
import paper_1111_6549_b200 as G
from paper_1111_6549_b200 import io as gio
from paper_1111_6549_b200 import tool

ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
SHAPES = [(0, 0), (0, 5), (5, 0), (1, 1), (3, 63), (4, 64), (5, 65), (7, 129), (33, 200)]


def bm(m, n, seed):
    a = G.BitMatrix(m, n)
    if m and n:
        G.fill_random(a, 0.5, seed)
    return a


@ref
@pytest.mark.parametrize("m,n", SHAPES)
def test_save_matches_reference_bytes(m, n):
    a = bm(m, n, m * 100 + n)
    for ascii in (False, True):
        buf = io.BytesIO()
        (gio.save_ascii if ascii else gio.save_gf2b)(buf, a)
        assert buf.getvalue() == O.ref_save_matrix(a.words, m, n, ascii), (m, n, ascii)


@ref
@pytest.mark.parametrize("m,n", SHAPES)
def test_load_round_trip_and_reference(m, n):
    a = bm(m, n, m * 7 + n)
    for ascii in (False, True):
        data = O.ref_save_matrix(a.words, m, n, ascii)
        got = gio.load_matrix(io.BytesIO(data))
        assert got.nrows() == m and got.ncols() == n
        assert np.array_equal(got.words, a.words)
        rm, rn, rw = O.ref_load_matrix(data)
        assert (rm, rn) == (m, n)
        if m and n:
            assert np.array_equal(rw, a.words)


def _gf2b(m, n, words):
    return gio.MAGIC + np.array([m, n], dtype="<u8").tobytes() + np.asarray(words, "<u8").tobytes()


REJECTS = {
    "bad magic": b"GF2C\x01" + bytes(16),
    "truncated header": gio.MAGIC + bytes(10),
    "truncated data": _gf2b(2, 64, [1]),
    "dirty padding": _gf2b(1, 3, [0b1000]),
    "trailing bytes": _gf2b(1, 3, [0b101]) + b"x",
    "huge dims": gio.MAGIC + np.array([1 << 33, 1], dtype="<u8").tobytes(),
    "ascii bad header": b"x 3\n",
    "ascii truncated": b"2 3\n101\n",
    "ascii short row": b"2 3\n101\n10\n",
    "ascii bad char": b"1 3\n1x1\n",
}


@ref
@pytest.mark.parametrize("name", sorted(REJECTS))
def test_rejections_match_reference(name):
    data = REJECTS[name]
    want = O.ref_load_matrix(data)
    assert want[0] == "io_error", (name, want)
    with pytest.raises(gio.IoError) as e:
        gio.load_matrix(io.BytesIO(data))
    assert str(e.value) == want[1], (name, str(e.value), want[1])


@ref
def test_ascii_quirks_match_reference():
    # CRLF line ends, header split over lines, no final newline
    for data in (b"2 3\r\n101\r\n011\r\n", b"2\n3\n101\n011\n", b"2 3\n101\n011", b"0 0\n"):
        want = O.ref_load_matrix(data)
        got = gio.load_matrix(io.BytesIO(data))
        assert (got.nrows(), got.ncols()) == want[:2]
        if got.nrows():
            assert np.array_equal(got.words, want[2])


@ref
def test_fill_random_rows_matches_reference():
    for (m, n, nnz, seed) in [(10, 100, 3, 1), (10, 100, 80, 2), (20, 65, 65, 3), (4, 1, 1, 4), (3, 0, 0, 5)]:
        a = G.BitMatrix(m, n)
        G.fill_random_rows(a, nnz, seed)
        if n:
            assert np.array_equal(a.words, O.ref_fill_random_rows(m, n, nnz, seed)), (m, n, nnz)
    with pytest.raises(ValueError):
        G.fill_random_rows(G.BitMatrix(2, 5), 6, 1)


def test_tool_gen_and_usage(tmp_path):
    out = str(tmp_path / "a.gf2b")
    assert tool.main(["gen", "--rows", "40", "--cols", "70", "--seed", "3", "--out", out]) == 0
    a = gio.load_gf2b(out)
    want = G.BitMatrix(40, 70)
    G.fill_random(want, 0.5, 3)
    assert a == want
    txt = str(tmp_path / "b.txt")
    assert tool.main(["gen", "--rows", "5", "--cols", "9", "--nnz-per-row", "2", "--out", txt,
                      "--format", "ascii"]) == 0
    b = gio.load_matrix(txt)
    assert b.nrows() == 5 and all(bin(int(w)).count("1") == 2 for w in b.words[:, 0])
    # usage errors (exit 1), missing input (exit 2) -- test_io_cli.cpp:200-214
    assert tool.main(["echelonize", "nosuch.gf2b", "--strategy", "warp"]) == 1
    assert tool.main(["echelonize", "nosuch.gf2b", "--k", "0"]) == 1
    assert tool.main(["echelonize", str(tmp_path / "does_not_exist.gf2b")]) == 2
    assert tool.main(["--help"]) == 0
