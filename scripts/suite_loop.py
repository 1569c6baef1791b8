"""Loop the 520-case golden suite (tests/golden/suite.json) on one driver
configuration and report every mismatch (race hunting).
usage: PYTHONPATH=.:tests python scripts/suite_loop.py <driver> <passes>
drivers: peer2 peer3 peer5 peer8 peer3s single super multi"""
import json
import sys
import time

import paper_1111_6549_b200 as G
import suite as S

CFG = {"peer2": dict(peer_ranks=2), "peer3": dict(peer_ranks=3), "peer5": dict(peer_ranks=5),
       "peer8": dict(peer_ranks=8), "peer3s": dict(peer_ranks=3, super_step=True),
       "single": dict(single_panel=True), "super": dict(super_step=True), "multi": dict(multi_kernel=True)}
drv, passes = sys.argv[1], int(sys.argv[2])
check = len(sys.argv) > 3 and sys.argv[3] == "check"
cfg = G.PleConfig(check=check, **CFG[drv])
cases = json.load(open("tests/golden/suite.json"))["cases"]
inputs = [(e, S.build(e["m"], e["n"], e["kind"], e["seed"])) for e in cases]
bad, t0 = 0, time.time()
for p in range(passes):
    for e, a in inputs:
        m, n = e["m"], e["n"]
        bm = G.BitMatrix(m, n, a.copy())
        try:
            out = G.block_iterative_ple(bm, cfg)
            ok = out.rank == e["rank"] and S.outcome_hash(bm.words, n, out.rank, out.p.swaps, out.q) == e["sha256"]
            why = f"rank {out.rank} vs {e['rank']}"
        except Exception as ex:  # noqa: BLE001
            ok, why = False, f"{type(ex).__name__}: {ex}"
        if not ok:
            bad += 1
            print(f"MISMATCH pass {p} case {m}x{n} kind {e['kind']} seed {e['seed']}: {why}", flush=True)
print(f"suite_loop {drv}{' check' if check else ''}: {passes} x {len(cases)} cases, {bad} mismatches, "
      f"{time.time() - t0:.1f} s", flush=True)
