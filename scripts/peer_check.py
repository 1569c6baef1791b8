"""The row-sharded peer-memory driver (ple_peer.cuh) with G ranks emulated on
one GPU: bit-exact vs the oracle on small shapes, vs the single-GPU driver
on medium ones (device checksums), then kernel times at the given sizes.
usage: python scripts/peer_check.py [sizes...]"""
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
import oracle as O  # noqa: E402
import suite as S  # noqa: E402
import paper_1111_6549_b200 as G  # noqa: E402

bad = 0
t0 = time.time()
for Gr, sup in ((1, False), (2, False), (3, False), (8, False), (1, True), (2, True), (3, True), (8, True)):
    cfg = G.PleConfig(peer_ranks=Gr, super_step=sup)
    for sp in S.suite_specs(120)[::3] + [(700, 900, 2, 5), (600, 600, 3, 6), (1000, 200, 5, 7),
                                          (200, 1000, 6, 8)]:
        m, n, kind, seed = sp
        a = S.build(m, n, kind, seed)
        ref = a.copy()
        want = O.ple(ref, m, n)
        bm = G.BitMatrix(m, n, a.copy())
        try:
            got = G.block_iterative_ple(bm, cfg)
        except Exception as e:  # noqa: BLE001
            print("ERROR", Gr, sp, e, flush=True)
            bad += 1
            if "watchdog" in str(e):
                sys.exit(1)
            continue
        ok = (got.rank == want.rank and np.array_equal(bm.words, ref)
              and np.array_equal(got.q, want.q.astype(np.uint64))
              and np.array_equal(got.p.swaps, want.swaps.astype(np.uint64)))
        if not ok:
            bad += 1
            print("MISMATCH", Gr, sup, sp, got.rank, want.rank, flush=True)
    print(f"G={Gr} super={sup}: small suite done, {bad} bad so far ({time.time() - t0:.1f} s)", flush=True)

for n in (4096, 16384):
    base = G.DeviceMatrix(n, n)
    base.fill_ctr(1)
    ref = G.block_iterative_ple(base)
    want = base.checksum()
    for Gr, sup in ((1, False), (2, False), (8, False), (1, True), (2, True), (8, True)):
        dm = G.DeviceMatrix(n, n)
        dm.fill_ctr(1)
        got = G.block_iterative_ple(dm, G.PleConfig(peer_ranks=Gr, super_step=sup))
        ok = got.rank == ref.rank and dm.checksum() == want and np.array_equal(got.q, ref.q)
        bad += 0 if ok else 1
        print(f"{n}^2 G={Gr} super={sup}: {'ok' if ok else 'MISMATCH'} rank {got.rank} "
              f"driver {got.stats['driver']}", flush=True)
        dm.close()
    base.close()

for n in [int(x) for x in sys.argv[1:]]:
    dm = G.DeviceMatrix(n, n)
    for Gr in (0, 1, 2, 4, 8):
        ts = []
        for _ in range(2):
            dm.fill_ctr(1)
            cfg = G.PleConfig(time_kernels=True, peer_ranks=Gr) if Gr else G.PleConfig(time_kernels=True)
            out = G.block_iterative_ple(dm, cfg)
            ts.append(out.stats["kernel_ms"])
        print(f"{n}^2 G={Gr} (0 = single-GPU driver): kernel {min(ts):.2f} ms, rank {out.rank}, "
              f"checksum {dm.checksum():#x}", flush=True)
    dm.close()
print("peer_check:", "FAIL" if bad else "ok", bad, flush=True)
sys.exit(1 if bad else 0)
