"""GPU parity against the golden fixtures made by the compiled reference
(tests/golden/make_golden.py): the 520-case edge/fill-kind suite, the small
full-content fixtures, and the BASELINE.json configs 1-5 at FULL size
(bit-exact via sha256 of the in-place words + rank + q + p.swaps)."""
import json
import os

import numpy as np
import pytest

import paper_1111_6549_b200 as G
import suite as S

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    p = os.path.join(GOLD, name)
    if not os.path.exists(p):
        pytest.skip(f"{name} not generated")
    with open(p) as f:
        return json.load(f)


SUITE_CFGS = {"single": G.PleConfig(single_panel=True), "super": G.PleConfig(super_step=True),
              "peer2": G.PleConfig(peer_ranks=2), "peer5": G.PleConfig(peer_ranks=5),
              "peer3s": G.PleConfig(peer_ranks=3, super_step=True)}


@pytest.mark.parametrize("driver", sorted(SUITE_CFGS))
def test_suite_golden_gpu(driver):
    bad = []
    cfg = SUITE_CFGS[driver]
    for e in load("suite.json")["cases"]:
        m, n = e["m"], e["n"]
        a = G.BitMatrix(m, n, S.build(m, n, e["kind"], e["seed"]))
        out = G.block_iterative_ple(a, cfg)
        h = S.outcome_hash(a.words, n, out.rank, out.p.swaps, out.q)
        if out.rank != e["rank"] or h != e["sha256"]:
            bad.append((m, n, e["kind"], e["seed"]))
    assert not bad, bad[:10]


def test_small_golden_gpu():
    for c in load("small.json")["cases"]:
        m, n = c["m"], c["n"]
        words = np.array([[int(x, 16) for x in r.split()] for r in c["input"]], dtype=np.uint64)
        a = G.BitMatrix(m, n, words)
        out = G.block_iterative_ple(a, G.PleConfig(k=c["k"]))
        want = np.array([[int(x, 16) for x in r.split()] for r in c["output"]], dtype=np.uint64)
        assert np.array_equal(a.words, want), c["name"]
        assert out.rank == c["rank"] and list(out.q) == c["q"] and list(out.p.swaps) == c["swaps"]


def full_input(cfg):
    m, n, gen = cfg["m"], cfg["n"], cfg["generator"]
    a = G.BitMatrix(m, n)
    if gen == "fill_random":
        G.fill_random(a, cfg["param"], cfg["seed"])
    elif gen == "ctr":
        G.fill_ctr(a, cfg["seed"])
    elif gen == "xy":
        import oracle as O
        if not O.ref_available():
            pytest.skip("X*Y needs oracle/_ref for the product")
        l = cfg["param"]
        x = O.fill_ctr(m, l, cfg["seed"][0])
        y = O.fill_ctr(l, n, cfg["seed"][1])
        a.words[:] = O.ref_mul(x, l, y, n)
    return a


@pytest.mark.parametrize("name", ["c1_4096_dense", "c2_16384_dense", "c2_16384x65536_dense",
                                  "c3_32768_p64", "c3_32768_p256", "c4_32768_xy", "c5_65536_ctr",
                                  "c5_131072_ctr"])
def test_full_config_bit_exact(name):
    cfgs = {c["name"]: c for c in load("full_configs.json")["configs"]}
    if name not in cfgs:
        pytest.skip(f"{name} not in full_configs.json yet")
    cfg = cfgs[name]
    m, n = cfg["m"], cfg["n"]
    a = full_input(cfg)
    assert S.outcome_hash(a.words, n, 0, [], []) == cfg["input_sha256"], "input generator mismatch"
    d = G.DeviceMatrix(m, n)
    d.upload(a.words)
    out = G.block_iterative_ple(d)
    d.download(a.words)
    assert out.rank == cfg["rank"]
    assert S.outcome_hash(a.words, n, out.rank, out.p.swaps, out.q) == cfg["sha256"]


@pytest.mark.parametrize("name,ranks", [("c2_16384x65536_dense", 4), ("c3_32768_p256", 4),
                                        ("c3_32768_p64", 2), ("c4_32768_xy", 3), ("c5_65536_ctr", 8),
                                        ("c5_131072_ctr", 8)])
def test_full_config_peer_ranks(name, ranks):
    """The row-sharded peer-memory driver (ple_peer.cuh) with `ranks` ranks
    emulated on the one GPU, bit-exact on full-size BASELINE configs: sparse
    (window misses), rank-deficient, wide, and config 5 over 8 ranks."""
    cfgs = {c["name"]: c for c in load("full_configs.json")["configs"]}
    if name not in cfgs:
        pytest.skip(f"{name} not in full_configs.json yet")
    cfg = cfgs[name]
    m, n = cfg["m"], cfg["n"]
    a = full_input(cfg)
    d = G.DeviceMatrix(m, n)
    d.upload(a.words)
    out = G.block_iterative_ple(d, G.PleConfig(peer_ranks=ranks))
    assert out.stats["driver"] == 4  # two panels per sweep at these sizes
    d.download(a.words)
    assert out.rank == cfg["rank"]
    assert S.outcome_hash(a.words, n, out.rank, out.p.swaps, out.q) == cfg["sha256"]
