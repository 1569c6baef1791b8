"""Command-line glue over the B200 path: the subcommands
of the reference's gf2tool that exercise this path (tools/gf2tool.cpp:123-257
and :432-527), with its output lines and exit codes (0 ok, 1 usage, 2 I/O,
3 verification failed; gf2tool.cpp:20-23). The compute runs on the device;
--verify checks on the device too (PLE: P*L*E through the device product;
echelonize: pivot structure plus random row-space membership against a
second device run; multiply: (AB)v = A(Bv) for random v).

    python -m paper_1111_6549_b200.tool gen --rows 4096 --cols 4096 --seed 1 --out a.gf2b
    python -m paper_1111_6549_b200.tool ple a.gf2b --verify --out e.gf2b
    python -m paper_1111_6549_b200.tool echelonize a.gf2b [--ref] [--verify]
    python -m paper_1111_6549_b200.tool multiply a.gf2b b.gf2b --out c.gf2b [--verify]
    python -m paper_1111_6549_b200.tool bench --suite table1|table2|fig3 --sizes 4096 --seeds 1 2 3
                                              [--memory-budget B] [--device-metrics] [--out f.csv]

--strategy, --k, --tables and --crossover are accepted for compatibility:
every strategy computes the same result (the device path serves them all;
tests/test_rref_host.py pins that).
"""
from __future__ import annotations

import argparse
import sys
import time

import numpy as np

from . import io as gio
from .ple import (BitMatrix, block_iterative_ple, echelonize, extract_e, extract_l, fill_random,
                  fill_random_rows, mul)

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_VERIFY = 0, 1, 2, 3


class VerifyError(RuntimeError):
    pass


def _save(path: str, a: BitMatrix, fmt: str) -> None:
    (gio.save_ascii if fmt == "ascii" else gio.save_gf2b)(path, a)


def _parity(words: np.ndarray, v: np.ndarray) -> np.ndarray:
    return (np.bitwise_count(words & v[None, :]).sum(axis=1) & 1).astype(np.uint8)


def _pack(bits: np.ndarray) -> np.ndarray:
    n = bits.shape[0]
    out = np.zeros(max(1, (n + 63) // 64) * 8, dtype=np.uint8)
    p = np.packbits(bits, bitorder="little")
    out[: p.size] = p
    return out.view(np.uint64)


def run_gen(o) -> int:
    a = BitMatrix(o.rows, o.cols)
    if o.nnz_per_row is not None:
        fill_random_rows(a, o.nnz_per_row, o.seed)
    else:
        fill_random(a, o.density, o.seed)
    _save(o.out, a, o.format)
    print(f"rows {o.rows}\ncols {o.cols}")
    return EXIT_OK


def run_ple(o) -> int:
    orig = gio.load_matrix(o.input)
    work = orig.copy()
    t0 = time.perf_counter()
    out = block_iterative_ple(work)
    secs = time.perf_counter() - t0
    if o.inject_fault and work.nrows() and work.ncols():
        work.set(0, 0, not work.get(0, 0))
    if o.verify:
        # the state invariants extract_e's closed form relies on (SURVEY.md
        # 8(c)): pivots on the diagonal, rows >= rank zero from column rank on
        r, n = out.rank, work.ncols()
        if r:
            idx = np.arange(r)
            if not np.all((work.words[idx, idx >> 6] >> (idx & 63).astype(np.uint64)) & np.uint64(1)):
                raise VerifyError("P*L*E does not reproduce the input")
        if r < work.nrows() and r < n:
            tail = work.words[r:].copy()
            tail[:, : r >> 6] = 0
            if r & 63:
                tail[:, r >> 6] &= ~np.uint64((1 << (r & 63)) - 1)
            if tail.any():
                raise VerifyError("P*L*E does not reproduce the input")
        l, e = extract_l(work, out), extract_e(work, out)
        back = mul(l, e) if out.rank else BitMatrix(out.processed, work.ncols())
        out.p.apply_inverse(back.words)
        if not np.array_equal(back.words[: out.processed], orig.words[: out.processed]):
            raise VerifyError("P*L*E does not reproduce the input")
    print(f"rank {out.rank}\nprocessed {out.processed}\nseconds {secs}")
    if o.out:
        _save(o.out, extract_e(work, out), o.format)
    return EXIT_OK


def run_echelonize(o) -> int:
    orig = gio.load_matrix(o.input)
    full = not o.ref
    work = orig.copy()
    t0 = time.perf_counter()
    rank = echelonize(work, full)
    secs = time.perf_counter() - t0
    if o.inject_fault and work.nrows() and work.ncols():
        work.set(0, 0, not work.get(0, 0))
    if o.verify:
        second = orig.copy()
        out = block_iterative_ple(second)
        if out.rank != rank:
            raise VerifyError("rank disagreement between strategies")
        m, n = orig.nrows(), orig.ncols()
        if full and m and n:
            q = np.asarray(out.q[:rank], dtype=np.int64)
            top = work.words[:rank]
            bits = (top[:, q >> 6] >> (q & 63).astype(np.uint64)) & np.uint64(1)
            if not np.array_equal(bits, np.eye(rank, dtype=np.uint64)) or work.words[rank:].any():
                raise VerifyError("echelon forms disagree")
            rng = np.random.default_rng(0)
            for _ in range(8):
                sel = rng.integers(0, 2, size=m).astype(bool)
                v = np.bitwise_xor.reduce(orig.words[sel], axis=0) if sel.any() else orig.words[0] * 0
                coef = ((v[q >> 6] >> (q & 63).astype(np.uint64)) & np.uint64(1)).astype(bool)
                red = v ^ (np.bitwise_xor.reduce(top[coef], axis=0) if coef.any() else 0)
                if np.any(red):
                    raise VerifyError("echelon forms disagree")
    print(f"rank {rank}\nseconds {secs}")
    if o.out:
        _save(o.out, work, o.format)
    return EXIT_OK


def run_multiply(o) -> int:
    a = gio.load_matrix(o.a)
    b = gio.load_matrix(o.b)
    if a.ncols() != b.nrows():
        raise ValueError("multiply: dimension mismatch")
    t0 = time.perf_counter()
    c = mul(a, b)
    secs = time.perf_counter() - t0
    if o.inject_fault and c.nrows() and c.ncols():
        c.set(0, 0, not c.get(0, 0))
    if o.verify and c.nrows() and c.ncols():
        rng = np.random.default_rng(0)
        for _ in range(4):
            v = _pack(rng.integers(0, 2, size=b.ncols(), dtype=np.uint8))
            bv = _pack(_parity(b.words, v)) if b.nrows() else np.zeros(1, np.uint64)
            want = _parity(a.words, bv) if a.ncols() else np.zeros(a.nrows(), np.uint8)
            if not np.array_equal(_parity(c.words, v), want):
                raise VerifyError("product disagrees with the naive check")
    _save(o.out, c, o.format)
    print(f"rows {c.nrows()}\ncols {c.ncols()}\nseconds {secs}")
    return EXIT_OK


# ---- bench (gf2tool.cpp:260-423) ------------------------------------------
BENCH_COLUMNS = ["algorithm", "nrows", "ncols", "density", "k", "tables", "crossover", "seed",
                 "seconds", "row_adds", "rank"]
DEVICE_COLUMNS = ["gpus", "K", "bytes_alg", "kernel_seconds", "GBps_eff", "roofline_frac"]


class BudgetError(ValueError):
    pass


def check_budget(n: int, budget: int) -> None:
    """gf2tool.cpp:314-322: matrix plus working copies, 4 * ceil(n/64)*8 * n bytes."""
    need = 4 * ((n + 63) // 64 * 8) * n
    if need > budget:
        raise BudgetError(f"refusing n={n}: estimated {need} bytes exceeds --memory-budget {budget}")


def _hbm_peak() -> float:
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def run_bench(o) -> int:
    """The reference's timing suites on the device. Every PLE / echelon
    strategy is the same computation here (one device path serves them all),
    so each cell times that path through the host API (upload + factor +
    download: what a caller of the drop-in waits for). row_adds is the
    reference's CPU op counter (op_count.hpp), which the device does not
    maintain: 0. --device-metrics appends gpus, K (panel columns), the
    SURVEY 8(d) algorithmic bytes, the kernel time and effective GB/s, and
    the fraction of the measured HBM peak."""
    from .ple import PleConfig
    k = 0 if o.k == "auto" else int(o.k)
    cfg = PleConfig(k=k, table_count=o.tables, time_kernels=True)
    peak = _hbm_peak()
    rows = []

    def gen(n, seed, nnz):
        a = BitMatrix(n, n)
        if nnz == 0:
            fill_random(a, 0.5, seed)
        else:
            fill_random_rows(a, nnz, seed)
        return a

    def cell(name, a, density, seed, what):
        work = a.copy()
        t0 = time.perf_counter()
        if what == "ple":
            out = block_iterative_ple(work, cfg)
            rank, st = out.rank, out.stats
        else:
            full = what == "rref"
            rank = echelonize(work, full, cfg)
            st = None
        secs = time.perf_counter() - t0
        rec = [name, a.nrows(), a.ncols(), density, k, o.tables, o.crossover, seed, secs, 0, rank]
        if o.device_metrics:
            ab = st["alg_bytes"] if st else ""
            ks = st["kernel_ms"] * 1e-3 if st and st["kernel_ms"] else ""
            gb = (ab / ks / 1e9) if (st and ks) else ""
            rec += [1, 64, ab, ks, gb, (gb / peak) if gb != "" else ""]
        rows.append(rec)

    if o.suite == "table1":
        for n in o.sizes:
            check_budget(n, o.memory_budget)
            for seed in o.seeds:
                a = gen(n, seed, 0)
                cell("ple-recursive-striped-base", a, "uniform:0.5", seed, "ple")
                cell("ple-recursive-cubic-base", a, "uniform:0.5", seed, "ple")
    elif o.suite == "table2":
        for n in o.sizes:
            check_budget(n, o.memory_budget)
            for seed in o.seeds:
                a = gen(n, seed, 0)
                cell("m4ri", a, "uniform:0.5", seed, "rref")
                cell("ple-recursive", a, "uniform:0.5", seed, "rref")
    else:  # fig3
        n = o.sizes[0]
        check_budget(n, o.memory_budget)
        for seed in o.seeds:
            cell("ple-recursive", gen(n, seed, 0), "uniform:0.5", seed, "ple")
            for nnz in range(1, 21):
                a = gen(n, seed, nnz)
                cell("ple-recursive", a, f"nnz:{nnz}", seed, "ple")
                cell("m4ri", a, f"nnz:{nnz}", seed, "ref")
    cols = BENCH_COLUMNS + (DEVICE_COLUMNS if o.device_metrics else [])
    text = ",".join(cols) + "\n" + "".join(",".join(_fmt(x) for x in r) + "\n" for r in rows)
    if o.out:
        try:
            with open(o.out, "w") as f:
                f.write(text)
        except OSError as e:
            raise gio.IoError(f"cannot open {o.out} for writing") from e
    else:
        sys.stdout.write(text)
    # one median line per (algorithm, shape, density) cell, on stderr (:291-312)
    seen = []
    for r in rows:
        key = (r[0], r[1], r[3])
        if key in seen:
            continue
        seen.append(key)
        t = [x[8] for x in rows if (x[0], x[1], x[3]) == key]
        print(f"median algorithm={r[0]} n={r[1]} density={r[3]} seconds={float(np.median(t))}",
              file=sys.stderr)
    return EXIT_OK


def _fmt(x) -> str:
    if isinstance(x, float):
        return f"{x:.6g}"
    return str(x)


def _common(p, strategy: str) -> None:
    p.add_argument("--strategy", default=strategy,
                   choices=["naive", "m4ri", "ple-iterative", "ple-recursive", "m4rm", "strassen",
                            "auto"])
    p.add_argument("--k", default="auto")
    p.add_argument("--tables", type=int, default=4)
    p.add_argument("--crossover", type=int, default=0)
    p.add_argument("--out", default="")
    p.add_argument("--format", default="gf2b", choices=["gf2b", "ascii"])
    p.add_argument("--verify", action="store_true")
    p.add_argument("--inject-fault", action="store_true")


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="gf2tool-b200", description="GF(2) PLE / echelon tools on the B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen", help="write a random matrix")
    g.add_argument("--rows", type=int, required=True)
    g.add_argument("--cols", type=int, required=True)
    g.add_argument("--density", type=float, default=0.5)
    g.add_argument("--nnz-per-row", type=int, default=None)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--out", required=True)
    g.add_argument("--format", default="gf2b", choices=["gf2b", "ascii"])
    e = sub.add_parser("echelonize", help="row echelon form and rank")
    e.add_argument("input")
    e.add_argument("--ref", action="store_true", help="stop at echelon form instead of reducing fully")
    _common(e, "m4ri")
    p = sub.add_parser("ple", help="PLE decomposition")
    p.add_argument("input")
    _common(p, "ple-recursive")
    m = sub.add_parser("multiply", help="matrix product")
    m.add_argument("a")
    m.add_argument("b")
    _common(m, "auto")
    m.set_defaults(out=None)
    b = sub.add_parser("bench", help="timing suites, CSV on stdout")
    b.add_argument("--suite", required=True, choices=["table1", "table2", "fig3"])
    b.add_argument("--sizes", type=int, nargs="+", default=[4096])
    b.add_argument("--seeds", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    b.add_argument("--memory-budget", type=int, default=2 << 30)
    b.add_argument("--k", default="auto")
    b.add_argument("--tables", type=int, default=1, choices=[1, 2, 4, 8])
    b.add_argument("--crossover", type=int, default=0)
    b.add_argument("--out", default="")
    b.add_argument("--device-metrics", action="store_true",
                   help="append gpus, K, bytes_alg, kernel_seconds, GBps_eff, roofline_frac")
    return ap


def main(argv=None) -> int:
    try:
        o = parser().parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    if o.cmd == "multiply" and not o.out:
        print("error: --out is required", file=sys.stderr)
        return EXIT_USAGE
    if o.cmd in ("ple", "echelonize", "multiply", "bench") and o.k != "auto":
        try:
            if not 1 <= int(o.k) <= 20:  # KValidator, gf2tool.cpp:51-66
                raise ValueError
        except ValueError:
            print("error: k must be 1..20 or 'auto'", file=sys.stderr)
            return EXIT_USAGE
    try:
        return {"gen": run_gen, "ple": run_ple, "echelonize": run_echelonize,
                "multiply": run_multiply, "bench": run_bench}[o.cmd](o)
    except VerifyError as e:
        print(f"verification failed: {e}", file=sys.stderr)
        return EXIT_VERIFY
    except (gio.IoError, OSError) as e:
        print(f"I/O error: {e}", file=sys.stderr)
        return EXIT_IO
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
