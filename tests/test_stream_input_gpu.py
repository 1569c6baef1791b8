"""Streamed input of the drop-in gf2cu_ple (run_ple / SuperRange): the
factorization starts on the first row block while the later ones are uploaded,
each late block replays the super-steps so far from the panel history, and the
rest runs on all rows. Bit-exact against the oracle like every other path; a column
without a pivot among the first block's rows must fall back to the ordinary
path (sparse, rank-deficient and zero inputs)."""
import numpy as np
import pytest

import oracle as O
import paper_1111_6549_b200 as G
from test_ple_gpu import assert_same, run_both

pytestmark = pytest.mark.gpu


@pytest.fixture
def stream_in(monkeypatch):
    monkeypatch.setenv("GF2CU_STREAM_IN", "1")
    return monkeypatch


def make(kind, m, n, seed):
    if kind == "dense":
        return O.fill_random(m, n, 0.5, seed)
    if kind == "ctr":
        return O.fill_ctr(m, n, seed)
    if kind == "p64":
        return O.fill_random(m, n, 1 / 64, seed)
    if kind == "p256":
        return O.fill_random(m, n, 1 / 256, seed)
    if kind == "dup":  # duplicated rows: rank deficiency, window misses late
        a = O.fill_random(m, n, 0.5, seed)
        rng = np.random.default_rng(seed)
        for _ in range(40):
            d, s = rng.integers(0, m, 2)
            a[d] = a[s]
        return a
    if kind == "dupcols":  # an early column without any pivot: the first phase gives up
        a = O.fill_random(m, n, 0.5, seed)
        a[:, 0] &= ~np.uint64(1 << 5)
        return a
    if kind == "zero":
        return np.zeros((m, (n + 63) // 64), dtype=np.uint64)
    if kind == "late":  # column 3 is set in one of the last rows only
        a = O.fill_random(m, n, 0.5, seed)
        a[:, 0] &= ~np.uint64(1 << 3)
        a[m - 2, 0] |= np.uint64(1 << 3)
        return a
    raise ValueError(kind)


SHAPES = [(2048, 2048), (4096, 4096), (3000, 4096), (4096, 2048), (2048, 8192), (5000, 3008)]


@pytest.mark.parametrize("m,n", SHAPES)
@pytest.mark.parametrize("kind", ["dense", "ctr", "dup"])
def test_streamed_input_matches_oracle(stream_in, m, n, kind):
    a = make(kind, m, n, m + 3 * n)
    ref, want, bm, got = run_both(a, m, n, G.PleConfig(super_step=True))
    assert_same(ref, want, bm, got, what=f"{kind} {m}x{n}")
    # the first phase ran (and did not give up) on these inputs
    assert got.stats["input_first_rows"] >= 512 and got.stats["input_first_steps"] >= 1


@pytest.mark.parametrize("frac", ["0.1", "0.27", "0.5", "0.8"])
def test_streamed_input_block_sizes(stream_in, frac):
    stream_in.setenv("GF2CU_STREAM_IN_FRAC", frac)
    m, n = 4096, 4096
    a = make("dense", m, n, 17)
    ref, want, bm, got = run_both(a, m, n, G.PleConfig(super_step=True))
    assert_same(ref, want, bm, got, what=f"frac {frac}")
    assert got.stats["input_first_rows"] > 0


@pytest.mark.parametrize("blocks,steps", [
    ("0.125,0.25,0.5", None),             # as many super-steps per block as its rows allow
    ("0.2,0.6", "3,9"),
    ("0.125,0.375,0.625,0.875", "2,2,10,12"),  # a block that joins without new super-steps
    ("0.3,0.5", "0,5"),                   # nothing runs on the first block alone
    ("0.0625,0.1875,0.4375", None),       # the default shares
])
@pytest.mark.parametrize("m,n,kind", [(4096, 4096, "dense"), (8192, 4096, "dup"), (5000, 8192, "ctr")])
def test_streamed_input_multi_block(stream_in, blocks, steps, m, n, kind):
    stream_in.setenv("GF2CU_STREAM_IN_BLOCKS", blocks)
    if steps:
        stream_in.setenv("GF2CU_STREAM_IN_STEPS", steps)
    a = make(kind, m, n, m + n)
    ref, want, bm, got = run_both(a, m, n, G.PleConfig(super_step=True))
    assert_same(ref, want, bm, got, what=f"blocks {blocks} steps {steps} {kind} {m}x{n}")
    assert got.stats["input_blocks"] >= 3 and got.stats["input_first_steps"] >= 1


@pytest.mark.parametrize("kind", ["p64", "p256", "dupcols", "zero", "late"])
def test_streamed_input_gives_up_cleanly(stream_in, kind):
    """Columns without a pivot among the first block's rows: the first phase
    sets its verdict, the later launches do nothing, and the ordinary path
    factors the (by then complete) upload."""
    m, n = 4096, 4096
    a = make(kind, m, n, 5)
    ref, want, bm, got = run_both(a, m, n, G.PleConfig(super_step=True))
    assert_same(ref, want, bm, got, what=kind)


def test_streamed_input_check_mode(stream_in):
    m, n = 4096, 4096
    a = make("dup", m, n, 23)
    ref, want, bm, got = run_both(a, m, n, G.PleConfig(super_step=True, check=True))
    assert_same(ref, want, bm, got, what="check mode")


def test_streamed_input_large_pageable_and_repeat(stream_in):
    """8192^2 = 8 MiB: the pageable staging path of both row blocks, twice on
    the same cached matrix (counters and history are reset per call)."""
    m, n = 8192, 8192
    for seed in (1, 2):
        a = make("ctr", m, n, seed)
        ref, want, bm, got = run_both(a, m, n, G.PleConfig(super_step=True))
        assert_same(ref, want, bm, got, what=f"8192 seed {seed}")
        assert got.stats["input_first_rows"] > 0


def test_default_rule_small_matrices_upload_whole():
    m, n = 2048, 2048
    a = make("dense", m, n, 3)
    ref, want, bm, got = run_both(a, m, n, G.PleConfig(super_step=True))
    assert_same(ref, want, bm, got)
    assert got.stats["input_first_rows"] == 0
