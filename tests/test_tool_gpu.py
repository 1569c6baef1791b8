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


def _csv(text):
    return [line.split(",") for line in text.strip().splitlines()]


def test_bench_suites_emit_the_reference_csv(tmp_path, capsys):
    """gf2tool bench (gf2tool.cpp:260-423), as the reference's own CLI tests
    drive it (test_io_cli.cpp:330-374): the 11-column CSV, one row per cell,
    medians on stderr; --device-metrics appends the device columns."""
    csv = str(tmp_path / "bench.csv")
    assert tool.main(["bench", "--suite", "table2", "--sizes", "64", "--seeds", "1", "2", "3",
                      "--out", csv]) == 0
    rows = _csv(open(csv).read())
    assert rows[0] == tool.BENCH_COLUMNS
    assert all(len(r) == 11 and r[1] == "64" and float(r[8]) > 0 and int(r[10]) <= 64 for r in rows[1:])
    assert sum(r[0] == "m4ri" for r in rows) == 3 and sum(r[0] == "ple-recursive" for r in rows) == 3
    capsys.readouterr()
    assert tool.main(["bench", "--suite", "table1", "--sizes", "48", "--seeds", "1"]) == 0
    out = capsys.readouterr()
    rows = _csv(out.out)
    assert len(rows) == 3 and rows[1][0] == "ple-recursive-striped-base"
    assert rows[2][0] == "ple-recursive-cubic-base" and "median algorithm=" in out.err
    assert tool.main(["bench", "--suite", "fig3", "--sizes", "48", "--seeds", "1"]) == 0
    rows = _csv(capsys.readouterr().out)
    assert sum(r[3].startswith("nnz:") for r in rows[1:]) == 40
    assert sum(r[3] == "uniform:0.5" for r in rows[1:]) == 1
    # ranks agree with the oracle
    a = O.fill_random(1024, 1024, 0.5, 3)
    want = O.echelonize(a.copy(), 1024, 1024, False)
    assert tool.main(["bench", "--suite", "table1", "--sizes", "1024", "--seeds", "3",
                      "--device-metrics"]) == 0
    rows = _csv(capsys.readouterr().out)
    assert rows[0] == tool.BENCH_COLUMNS + tool.DEVICE_COLUMNS
    for r in rows[1:]:
        assert int(r[10]) == want and int(r[11]) == 1 and int(r[12]) == 64
        assert float(r[13]) > 0 and float(r[15]) > 0 and 0 < float(r[16]) < 1.5
