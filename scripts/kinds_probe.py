"""Timing anomalies across input structures: one size, many kinds (dense,
sparse densities, fixed row weight, permutation, low rank, duplicated rows,
zero blocks), device-resident PLE time next to the dense time, each result
against the oracle.
usage: PYTHONPATH=.:tests python scripts/kinds_probe.py [n]"""
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
import oracle as O  # noqa: E402
import paper_1111_6549_b200 as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
W = n // 64
rng = np.random.default_rng(5)


def perm_matrix():
    a = np.zeros((n, W), dtype=np.uint64)
    p = rng.permutation(n)
    a[np.arange(n), p >> 6] = np.uint64(1) << (p & 63).astype(np.uint64)
    return a


def low_rank(k):
    x = O.fill_random(n, k, 0.5, 3)
    y = O.fill_random(k, n, 0.5, 4)
    return O.mul(x, k, y, n)


def zero_block():
    a = O.fill_random(n, n, 0.5, 9)
    a[:, : W // 2] = 0  # the left half of the columns is empty
    return a


def late_rows():
    a = O.fill_random(n, n, 0.5, 10)
    a[: n // 2, :] = 0  # the first half of the rows is empty: every window misses at first
    return a


kinds = {
    "dense": lambda: O.fill_random(n, n, 0.5, 1),
    "p=1/64": lambda: O.fill_random(n, n, 1 / 64, 1),
    "p=1/256": lambda: O.fill_random(n, n, 1 / 256, 1),
    "p=1/1024": lambda: O.fill_random(n, n, 1 / 1024, 1),
    "p=1/4096": lambda: O.fill_random(n, n, 1 / 4096, 1),
    "rows nnz=3": lambda: O.fill_random_rows(n, n, 3, 1),
    "rows nnz=16": lambda: O.fill_random_rows(n, n, 16, 1),
    "permutation": perm_matrix,
    "rank 64": lambda: low_rank(64),
    "rank 1000": lambda: low_rank(1000),
    "zero left half": zero_block,
    "zero top half": late_rows,
    "all ones": lambda: O.fill_random(n, n, 1.0, 1),
}
d = G.DeviceMatrix(n, n)
only = set(sys.argv[2:])
for name, make in kinds.items():
    if only and name not in only:
        continue
    a = make()
    ref = a.copy()
    t0 = time.perf_counter()
    want = O.ple(ref, n, n)
    t_or = time.perf_counter() - t0
    line = f"{name:16s} rank {want.rank:6d} oracle {t_or:6.2f} s |"
    for label, cfg in (("default", G.PleConfig(time_kernels=True)), ("super", G.PleConfig(time_kernels=True, super_step=True)),
                       ("peer2", G.PleConfig(time_kernels=True, peer_ranks=2))):
        ks = []
        for it in range(3):
            d.upload(a)
            out = G.block_iterative_ple(d, cfg)
            ks.append(out.stats["kernel_ms"])
        got = np.empty_like(a)
        d.download(got)
        ok = out.rank == want.rank and np.array_equal(got, ref) and np.array_equal(out.q, want.q.astype(np.uint64))
        line += f" {label} {min(ks):8.3f} ms {'ok' if ok else 'MISMATCH'} |"
    print(line, flush=True)
