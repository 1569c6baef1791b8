"""Race hunting: a random interleaving of the device entry points (PLE with all
three drivers, rref_from_ple full / echelon, trsm, mul / addmul) on random
small shapes, each checked against the oracle. Unlike stress_small.py the
shape and the operation change on every call, so cached device buffers are
re-created and re-used with stale contents, as inside pytest.

usage: python scripts/stress_mixed.py [iterations] [seed]
"""
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
import oracle as O  # noqa: E402
import suite as S  # noqa: E402
import paper_1111_6549_b200 as G  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
CFGS = {"single": G.PleConfig(single_panel=True), "multi": G.PleConfig(multi_kernel=True),
        "super": G.PleConfig(super_step=True), "peer2": G.PleConfig(peer_ranks=2),
        "peer3s": G.PleConfig(peer_ranks=3, super_step=True)}


def rand_shape():
    big = rng.random() < 0.15
    hi = 1500 if big else 320
    return int(rng.integers(1, hi)), int(rng.integers(1, hi))


def one(it):
    op = rng.choice(["ple", "ple", "ple", "rref", "echelon", "trsm", "mul", "addmul"])
    m, n = rand_shape()
    kind = int(rng.integers(0, 7))
    seed = int(rng.integers(0, 2**62))
    a = S.build(m, n, kind, seed)
    if op == "ple":
        drv = str(rng.choice(list(CFGS)))
        ref = a.copy()
        want = O.ple(ref, m, n)
        bm = G.BitMatrix(m, n, a.copy())
        got = G.block_iterative_ple(bm, CFGS[drv])
        ok = (got.rank == want.rank and np.array_equal(bm.words, ref)
              and np.array_equal(got.q, want.q.astype(np.uint64))
              and np.array_equal(got.p.swaps, want.swaps.astype(np.uint64)))
        return ok, f"ple/{drv} {m}x{n} kind {kind} seed {seed} rank {got.rank} vs {want.rank}"
    if op in ("rref", "echelon"):
        full = op == "rref"
        ref = a.copy()
        r = O.echelonize(ref, m, n, full)
        bm = G.BitMatrix(m, n, a.copy())
        got = G.echelonize(bm, full)
        return got == r and np.array_equal(bm.words, ref), f"{op} {m}x{n} kind {kind} seed {seed}"
    if op == "trsm":
        r = m
        u = S.build(r, r, 2, seed ^ 1)
        bits = S.unpack(u, r)
        np.fill_diagonal(bits, 1)
        u = S.pack(np.triu(bits), r)
        want = a.copy()
        O.trsm_upper(u, r, want, n)
        bb = G.BitMatrix(r, n, a.copy())
        G.trsm_upper_left_unit(G.BitMatrix(r, r, u), bb)
        return np.array_equal(bb.words, want), f"trsm {r}x{n} seed {seed}"
    L = int(rng.integers(1, 400))
    b = S.build(L, n, 2, seed ^ 2)
    x = S.build(m, L, kind, seed ^ 3)
    want = O.mul(x, L, b, n)
    if op == "mul":
        got = G.mul(G.BitMatrix(m, L, x), G.BitMatrix(L, n, b)).words
        return np.array_equal(got, want), f"mul {m}x{L}x{n} seed {seed}"
    c = a.copy()
    G.addmul(cm := G.BitMatrix(m, n, c), G.BitMatrix(m, L, x), G.BitMatrix(L, n, b))
    return np.array_equal(cm.words, want ^ a), f"addmul {m}x{L}x{n} seed {seed}"


t0 = time.time()
bad = []
for it in range(iters):
    try:
        ok, what = one(it)
    except Exception as e:  # noqa: BLE001 (check mode: Gf2cuCheckError names the step)
        ok, what = False, f"{type(e).__name__}: {e}"
    if not ok:
        bad.append((it, what))
        print("MISMATCH", it, what, flush=True)
print(f"stress_mixed: {iters} calls, {len(bad)} mismatches, {time.time() - t0:.1f} s", flush=True)
sys.exit(1 if bad else 0)
