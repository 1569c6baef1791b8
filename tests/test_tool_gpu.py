"""GPU: the CLI glue (paper_1111_6549_b200/tool.py) end to end on files:
outputs against the oracle, --verify passing, --inject-fault caught with
exit 3 (the reference's CLI contract, test_io_cli.cpp:255-282)."""
import numpy as np
import pytest

import oracle as O
from paper_1111_6549_b200 import io as gio
from paper_1111_6549_b200 import tool

pytestmark = pytest.mark.gpu


def gen(tmp_path, name, m, n, seed, density=0.5):
    path = str(tmp_path / name)
    assert tool.main(["gen", "--rows", str(m), "--cols", str(n), "--seed", str(seed),
                      "--density", str(density), "--out", path]) == 0
    return path


@pytest.mark.parametrize("m,n,density", [(300, 200, 0.5), (200, 300, 0.05), (1000, 1000, 0.5)])
def test_ple_and_echelonize(tmp_path, m, n, density):
    a_path = gen(tmp_path, "a.gf2b", m, n, 7, density)
    a = gio.load_gf2b(a_path).words
    e_path = str(tmp_path / "e.gf2b")
    assert tool.main(["ple", a_path, "--verify", "--out", e_path]) == 0
    want_e = a.copy()
    r = O.echelonize(want_e, m, n, False)
    e = gio.load_gf2b(e_path)
    assert e.nrows() == r and np.array_equal(e.words, want_e[:r])
    for full in (True, False):
        out = str(tmp_path / f"r{int(full)}.txt")
        args = ["echelonize", a_path, "--verify", "--out", out, "--format", "ascii"]
        assert tool.main(args + ([] if full else ["--ref"])) == 0
        want = a.copy()
        O.echelonize(want, m, n, full)
        assert np.array_equal(gio.load_matrix(out).words, want)
    assert tool.main(["ple", a_path, "--verify", "--inject-fault"]) == 3
    assert tool.main(["echelonize", a_path, "--verify", "--inject-fault"]) == 3


def test_multiply(tmp_path):
    a_path = gen(tmp_path, "a.gf2b", 300, 200, 1)
    b_path = gen(tmp_path, "b.gf2b", 200, 250, 2)
    c_path = str(tmp_path / "c.gf2b")
    assert tool.main(["multiply", a_path, b_path, "--out", c_path, "--verify"]) == 0
    a, b = gio.load_gf2b(a_path).words, gio.load_gf2b(b_path).words
    assert np.array_equal(gio.load_gf2b(c_path).words, O.mul(a, 200, b, 250))
    assert tool.main(["multiply", a_path, b_path, "--out", c_path, "--verify", "--inject-fault"]) == 3
    assert tool.main(["multiply", a_path, a_path, "--out", c_path]) == 1  # dimension mismatch
