"""Re-run one suite case many times on several drivers against the oracle.
usage: PYTHONPATH=.:tests python scripts/repro_case.py m n kind seed [reps]"""
import sys

import numpy as np

import oracle as O
import paper_1111_6549_b200 as G
import suite as S

m, n, kind, seed = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 200
a = S.build(m, n, kind, seed)
ref = a.copy()
want = O.ple(ref, m, n)
cfgs = {"peer5": G.PleConfig(peer_ranks=5), "peer5c": G.PleConfig(peer_ranks=5, check=True),
        "peer2": G.PleConfig(peer_ranks=2), "peer3": G.PleConfig(peer_ranks=3),
        "single": G.PleConfig(single_panel=True), "super": G.PleConfig(super_step=True)}
for name, cfg in cfgs.items():
    bad = 0
    first = None
    for it in range(reps):
        bm = G.BitMatrix(m, n, a.copy())
        try:
            got = G.block_iterative_ple(bm, cfg)
            ok = got.rank == want.rank and np.array_equal(bm.words, ref) and np.array_equal(got.q, want.q)
        except Exception as e:  # noqa: BLE001
            ok, got = False, e
        if not ok:
            bad += 1
            if first is None:
                first = (it, got if isinstance(got, Exception) else
                         (got.rank, int(np.count_nonzero(bm.words != ref)), np.argwhere(bm.words != ref)[:4].tolist()))
    print(f"{name}: {bad}/{reps} bad, first {first}", flush=True)
