"""Shared input builders for the parity suites (test infrastructure).

The edge-dimension x fill-kind grid mirrors the reference's acceptance suite
coverage (acceptance_main.cpp:40-88: edge dims {1,2,3,31,...,300}, kinds zero,
all-ones, dense, thin, fixed nnz/row, and two with duplicated rows/columns),
with this repo's own deterministic seeding: inputs are regenerated from
(m, n, kind, seed) by the oracle's generators, so the golden files only need
to store specs and expected hashes.
"""
from __future__ import annotations

import hashlib

import numpy as np

import oracle as O

EDGE_DIMS = [1, 2, 3, 31, 32, 33, 63, 64, 65, 96, 127, 128, 129, 150, 191, 192, 193, 257, 300]
KINDS = ["zero", "ones", "dense", "thin", "nnz_rows", "dense_dup", "nnz_dup"]


def suite_specs(count: int = 520, master_seed: int = 20261020):
    rng = np.random.default_rng(master_seed)
    specs = []
    ne = len(EDGE_DIMS)
    for i in range(ne):
        for kind in range(len(KINDS)):
            specs.append((EDGE_DIMS[i], EDGE_DIMS[(i * 3 + kind) % ne], kind, int(rng.integers(0, 2**62))))
    while len(specs) < count:
        m, n = int(rng.integers(1, 301)), int(rng.integers(1, 301))
        specs.append((m, n, int(rng.integers(0, 7)), int(rng.integers(0, 2**62))))
    return specs


def build(m: int, n: int, kind: int, seed: int) -> np.ndarray:
    W = max(1, (n + 63) // 64)
    rng = np.random.default_rng(seed)
    if kind == 0:
        return np.zeros((m, W), dtype=np.uint64)
    if kind == 1:
        return O.fill_random(m, n, 1.0, seed)
    if kind == 2:
        return O.fill_random(m, n, 0.5, seed)
    if kind == 3:
        return O.fill_random(m, n, 0.08, seed)
    nnz = min(n, 1 + int(rng.integers(0, 20)))
    if kind == 4:
        return O.fill_random_rows(m, n, nnz, seed)
    a = O.fill_random(m, n, 0.5, seed) if kind == 5 else O.fill_random_rows(m, n, nnz, seed)
    bits = unpack(a, n)
    for _ in range(4):
        d, s = int(rng.integers(0, m)), int(rng.integers(0, m))
        bits[d] = bits[s]
    for _ in range(3):
        d, s = int(rng.integers(0, n)), int(rng.integers(0, n))
        bits[:, d] = bits[:, s]
    return pack(bits, n)


def unpack(a: np.ndarray, n: int) -> np.ndarray:
    """uint64 words -> (m, n) uint8 bit matrix (LSB-first within each word)."""
    b = np.unpackbits(a.view(np.uint8), axis=1, bitorder="little")
    return b[:, :n].copy()


def pack(bits: np.ndarray, n: int) -> np.ndarray:
    m = bits.shape[0]
    W = max(1, (n + 63) // 64)
    full = np.zeros((m, W * 64), dtype=np.uint8)
    full[:, :n] = bits
    return np.packbits(full, axis=1, bitorder="little").view(np.uint64).reshape(m, W).copy()


def outcome_hash(words: np.ndarray, n: int, rank: int, swaps, q) -> str:
    """sha256 over the logical words (W per row, LE), rank, q and p.swaps."""
    W = max(1, (n + 63) // 64)
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(words[:, :W], dtype="<u8").tobytes())
    h.update(np.uint64(rank).tobytes())
    h.update(np.asarray(q, dtype="<u8").tobytes())
    h.update(np.asarray(swaps, dtype="<u8").tobytes())
    return h.hexdigest()
