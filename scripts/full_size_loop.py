"""Determinism at full size: every BASELINE config factored repeatedly
(device-resident and through the drop-in call), each result's outcome hash
against the reference's (tests/golden/full_configs.json).
usage: PYTHONPATH=.:tests python scripts/full_size_loop.py [reps at 65536^2]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
import suite as S  # noqa: E402
import paper_1111_6549_b200 as G  # noqa: E402
from test_golden_gpu import full_input  # noqa: E402

reps65 = int(sys.argv[1]) if len(sys.argv) > 1 else 100
with open("tests/golden/full_configs.json") as f:
    cfgs = [c for c in json.load(f)["configs"] if c["name"].startswith("c")]
bad = 0
t0 = time.time()
for cfg in cfgs:
    m, n = cfg["m"], cfg["n"]
    reps = max(3, int(reps65 * (65536.0 / max(m, n)) ** 2.5)) if max(m, n) > 4096 else 4 * reps65
    reps = min(reps, 2000)
    a = full_input(cfg)
    src = a.words.copy()
    d = G.DeviceMatrix(m, n)
    d.upload(src)
    first = G.block_iterative_ple(d)
    d.download(a.words)
    ok = first.rank == cfg["rank"] and S.outcome_hash(a.words, n, first.rank, first.p.swaps, first.q) == cfg["sha256"]
    want = d.checksum()
    nbad = 0 if ok else 1
    for it in range(reps):
        d.upload(src)
        o = G.block_iterative_ple(d)
        if o.rank != first.rank or d.checksum() != want or not np.array_equal(o.q, first.q):
            nbad += 1
    hreps = max(2, reps // 10)
    for it in range(hreps):
        a.words[:] = src
        o = G.block_iterative_ple(a)
        if o.rank != first.rank or G.host_checksum(a.words, n) != want or not np.array_equal(o.p.swaps, first.p.swaps):
            nbad += 1
    bad += nbad
    print(f"{cfg['name']}: first run vs reference {'ok' if ok else 'MISMATCH'}; {reps} device + {hreps} drop-in "
          f"repeats, {nbad} deviations ({time.time() - t0:.0f} s)", flush=True)
    d.close()
print("total deviations", bad)
