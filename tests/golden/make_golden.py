#!/usr/bin/env python3
"""Generates the golden fixtures under tests/golden/ by running the REFERENCE
itself (oracle/_ref/libgf2ref.so = the unmodified gf2elim headers compiled
with -O3 -DNDEBUG). Run here, where /root/reference exists:

    python tests/golden/make_golden.py            # suite + small fixtures
    python tests/golden/make_golden.py --full     # + full-size BASELINE configs (slow)

Outputs
  suite.json        520 specs (m, n, kind, seed) -> reference rank + sha256
                    (tests/suite.py builds the inputs, hashes the outcome)
  small.json        full in-place results (hex words) of small cases + KATs
  full_configs.json BASELINE.json configs 1-5 at full size -> rank, sha256,
                    reference seconds
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle as O  # noqa: E402
import suite as S  # noqa: E402


def hexrows(a):
    return [" ".join(f"{int(x):016x}" for x in row) for row in a]


def ref_run(a, m, n, k=0):
    b = a.copy()
    out, secs = O.ref_ple(b, m, n, k=k)
    return b, out, secs


def make_suite():
    entries = []
    for (m, n, kind, seed) in S.suite_specs():
        a = S.build(m, n, kind, seed)
        b, out, _ = ref_run(a, m, n)
        entries.append({"m": m, "n": n, "kind": kind, "seed": seed, "rank": out.rank,
                        "sha256": S.outcome_hash(b, n, out.rank, out.swaps, out.q)})
    with open(os.path.join(HERE, "suite.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference: oracle/_ref)",
                   "hash": "tests/suite.py:outcome_hash", "cases": entries}, f, indent=0)
    print("suite.json:", len(entries), "cases")


def make_small():
    cases = []

    def add(name, a, m, n, k=0):
        b, out, _ = ref_run(a, m, n, k)
        cases.append({"name": name, "m": m, "n": n, "k": k, "input": hexrows(a), "output": hexrows(b),
                      "rank": out.rank, "swaps": [int(x) for x in out.swaps], "q": [int(x) for x in out.q],
                      "ref_col_swaps": [[int(v) for v in cs] for cs in out.col_swaps]})

    # Fig. 2 of the paper (PAPER.md; acceptance_main.cpp:321-372 / test_m4ri.cpp:109-134)
    fig2 = ["10010111", "01011110", "00100111", "00011010", "11001011", "01001001", "11011101"]
    add("paper_fig2", S.pack(np.array([[int(c) for c in r] for r in fig2], dtype=np.uint8), 8), 7, 8)
    # section 3.2 worked example as a PLE: three source rows + [1 0 1 ...] -> multipliers [1 0 0]
    ex = ["10110010", "01101100", "00111010", "10100111"]
    add("sec32_multipliers", S.pack(np.array([[int(c) for c in r] for r in ex], dtype=np.uint8), 8), 4, 8)
    add("identity_33", S.pack(np.eye(33, dtype=np.uint8), 33), 33, 33)
    add("zero_6x9", np.zeros((6, 1), dtype=np.uint64), 6, 9)
    rng = np.random.default_rng(7)
    for i in range(16):
        m, n = int(rng.integers(1, 71)), int(rng.integers(1, 131))
        kind = i % 7
        a = S.build(m, n, kind, int(rng.integers(0, 2**62)))
        add(f"small_{i}_{S.KINDS[kind]}", a, m, n, k=int(rng.integers(0, 17)))
    with open(os.path.join(HERE, "small.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference: oracle/_ref)", "cases": cases},
                  f, indent=1)
    print("small.json:", len(cases), "cases")


FULL = [
    # (name, m, n, generator, param, seed)
    ("c1_4096_dense", 4096, 4096, "fill_random", 0.5, 1),
    ("c2_16384_dense", 16384, 16384, "fill_random", 0.5, 1),
    ("c2_16384x65536_dense", 16384, 65536, "fill_random", 0.5, 1),
    ("c3_32768_p64", 32768, 32768, "fill_random", 1 / 64, 1),
    ("c3_32768_p256", 32768, 32768, "fill_random", 1 / 256, 1),
    ("c4_32768_xy", 32768, 32768, "xy", 24576, (11, 12)),
    ("c5_65536_ctr", 65536, 65536, "ctr", None, 1),
    ("c5_131072_ctr", 131072, 131072, "ctr", None, 1),
    # the sizes around the driver switch (tests/test_ple_gpu.py
    # test_default_driver_size_rule: ctr seed 9) and the streamed-output
    # cases (ctr seed 3 with rows m/3 .. m/3+200 copied from rows 10..210)
    ("m_8192x65536_ctr9", 8192, 65536, "ctr", None, 9),
    ("m_20480_ctr9", 20480, 20480, "ctr", None, 9),
    ("m_16384x24576_ctr9", 16384, 24576, "ctr", None, 9),
    ("m_16384_ctr9", 16384, 16384, "ctr", None, 9),
    ("m_12288_ctr9", 12288, 12288, "ctr", None, 9),
    ("s_16384_dup3", 16384, 16384, "ctr_dup", None, 3),
    ("s_12000x20000_dup3", 12000, 20000, "ctr_dup", None, 3),
    ("s_20000x9000_dup3", 20000, 9000, "ctr_dup", None, 3),
]


def full_input(gen, m, n, param, seed):
    if gen == "fill_random":
        return O.fill_random(m, n, param, seed)
    if gen == "ctr":
        return O.fill_ctr(m, n, seed)
    if gen == "ctr_dup":
        a = O.fill_ctr(m, n, seed)
        a[m // 3: m // 3 + 200] = a[10:210]
        return a
    if gen == "xy":
        l = param
        x = O.fill_ctr(m, l, seed[0])
        y = O.fill_ctr(l, n, seed[1])
        return O.ref_mul(x, l, y, n)
    raise ValueError(gen)


def make_full(only=None):
    path = os.path.join(HERE, "full_configs.json")
    old = {}
    if os.path.exists(path):
        with open(path) as f:
            old = {c["name"]: c for c in json.load(f)["configs"]}
    out = dict(old)
    for (name, m, n, gen, param, seed) in FULL:
        if only and name not in only:
            continue
        t0 = time.time()
        a = full_input(gen, m, n, param, seed)
        tg = time.time() - t0
        in_sha = S.outcome_hash(a, n, 0, [], [])
        b, o, secs = ref_run(a, m, n)
        out[name] = {"name": name, "m": m, "n": n, "generator": gen, "param": param, "seed": seed,
                     "input_sha256": in_sha, "rank": o.rank,
                     "sha256": S.outcome_hash(b, n, o.rank, o.swaps, o.q),
                     "ref_seconds": round(secs, 3), "gen_seconds": round(tg, 2)}
        print(name, "rank", o.rank, "ref", round(secs, 2), "s", flush=True)
        with open(path, "w") as f:
            json.dump({"generator": "tests/golden/make_golden.py --full (reference: oracle/_ref, 1 thread)",
                       "hash": "tests/suite.py:outcome_hash", "configs": list(out.values())}, f, indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--only", nargs="*")
    args = ap.parse_args()
    if args.full:
        make_full(args.only)
    else:
        make_suite()
        make_small()
