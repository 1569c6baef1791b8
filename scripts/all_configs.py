"""Every BASELINE.json config at full size on the device: kernel time (CUDA
events around the persistent launch, device-resident input), the drop-in
gf2cu_ple call on pageable host memory (H2D + PLE + D2H), the outcome hash
against the reference's (tests/golden/full_configs.json), and the reference's
own single-core time from that file. Writes gpurun_out/all_configs.json.
usage: PYTHONPATH=.:tests python scripts/all_configs.py [name ...]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
import suite as S  # noqa: E402
import paper_1111_6549_b200 as G  # noqa: E402
from test_golden_gpu import full_input  # noqa: E402

with open("tests/golden/full_configs.json") as f:
    cfgs = json.load(f)["configs"]
want = set(sys.argv[1:])
rows = []
for cfg in cfgs:
    if want and cfg["name"] not in want:
        continue
    if cfg["generator"] not in ("fill_random", "ctr", "xy"):
        continue  # (the streamed-output cases have their own generator in tests/test_ple_gpu.py)
    m, n = cfg["m"], cfg["n"]
    try:
        a = full_input(cfg)
    except BaseException as e:  # noqa: BLE001  (pytest.skip when oracle/_ref is absent)
        print(cfg["name"], "skipped:", e)
        continue
    src = a.words.copy()
    d = G.DeviceMatrix(m, n)
    ks = []
    for it in range(4):
        d.upload(src)
        out = G.block_iterative_ple(d, G.PleConfig(time_kernels=True))
        if it:
            ks.append(out.stats["kernel_ms"])
    d.download(a.words)
    ok = out.rank == cfg["rank"] and S.outcome_hash(a.words, n, out.rank, out.p.swaps, out.q) == cfg["sha256"]
    d.close()
    e2e = []
    for it in range(3):
        a.words[:] = src
        t0 = time.perf_counter()
        o2 = G.block_iterative_ple(a)
        e2e.append(1e3 * (time.perf_counter() - t0))
    ok2 = o2.rank == cfg["rank"] and S.outcome_hash(a.words, n, o2.rank, o2.p.swaps, o2.q) == cfg["sha256"]
    row = {"name": cfg["name"], "m": m, "n": n, "rank": int(out.rank), "driver": int(out.stats["driver"]),
           "kernel_ms": round(float(np.median(ks)), 3), "e2e_pageable_ms": round(min(e2e[1:]), 3),
           "alg_GB": round(out.stats["alg_bytes"] / 1e9, 3),
           "eff_GBps": round(out.stats["alg_bytes"] / (np.median(ks) * 1e-3) / 1e9, 1),
           "reference_s": cfg.get("ref_seconds"),
           "speedup_e2e": round(cfg["ref_seconds"] * 1e3 / min(e2e[1:]), 1) if cfg.get("ref_seconds") else None,
           "bit_exact_device": bool(ok), "bit_exact_dropin": bool(ok2)}
    rows.append(row)
    print(json.dumps(row), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/all_configs.json", "w") as f:
    json.dump({"note": "scripts/all_configs.py on one B200; reference_s = the compiled reference, 1 core, "
                       "in the build container (tests/golden/full_configs.json)", "configs": rows}, f, indent=1)
