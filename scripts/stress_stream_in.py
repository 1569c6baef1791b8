"""Streamed input soak: the drop-in gf2cu_ple on host matrices with random
row-block plans (GF2CU_STREAM_IN_BLOCKS / _STEPS), random shapes and input
kinds (incl. sparse / rank-deficient ones whose first phase gives up), every
result compared with the oracle.

usage: PYTHONPATH=.:tests python scripts/stress_stream_in.py [iterations] [seed]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
import oracle as O  # noqa: E402
import suite as S  # noqa: E402
import paper_1111_6549_b200 as G  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
os.environ["GF2CU_STREAM_IN"] = "1"
bad = 0
t0 = time.time()
used = 0
for it in range(iters):
    m = int(rng.integers(600, 4200))
    n = int(rng.integers(1, 5)) * 1024 if rng.random() < 0.6 else int(rng.integers(64, 4200))
    kind = int(rng.integers(0, 7))
    seed = int(rng.integers(0, 2**62))
    nb = int(rng.integers(1, 6))
    fr = np.sort(rng.random(nb) * 0.85 + 0.02)
    os.environ["GF2CU_STREAM_IN_BLOCKS"] = ",".join(f"{f:.4f}" for f in fr)
    if rng.random() < 0.5:
        st = np.sort(rng.integers(0, 1 + m // 128, nb))
        os.environ["GF2CU_STREAM_IN_STEPS"] = ",".join(str(int(s)) for s in st)
    else:
        os.environ.pop("GF2CU_STREAM_IN_STEPS", None)
    if rng.random() < 0.5:
        # dense, with a few duplicated rows (late window misses; the block plan survives)
        kind = 7
        a = O.fill_random(m, n, 0.5, seed)
        for _ in range(int(rng.integers(0, 30))):
            d, s2 = rng.integers(0, m, 2)
            a[d] = a[s2]
    else:
        a = S.build(m, n, kind, seed)
    ref = a.copy()
    want = O.ple(ref, m, n)
    bm = G.BitMatrix(m, n, a.copy())
    got = G.block_iterative_ple(bm, G.PleConfig(super_step=True, check=bool(rng.random() < 0.3)))
    ok = (got.rank == want.rank and np.array_equal(bm.words, ref)
          and np.array_equal(got.q, want.q.astype(np.uint64))
          and np.array_equal(got.p.swaps, want.swaps.astype(np.uint64)))
    used += got.stats["input_blocks"] > 0
    if not ok:
        bad += 1
        print(f"MISMATCH it {it}: {m}x{n} kind {kind} seed {seed} blocks {os.environ['GF2CU_STREAM_IN_BLOCKS']} "
              f"steps {os.environ.get('GF2CU_STREAM_IN_STEPS')} rank {got.rank} vs {want.rank} stats {got.stats}", flush=True)
print(f"{iters} calls, {used} with a block plan, {bad} mismatches, {time.time() - t0:.0f} s")
