"""Row-sharded multi-GPU block_iterative_ple driven on the device
(kernel csrc/ple_peer.cuh).

One process per GPU. Rows are distributed block-cyclically exactly as in
shard.py (global row g on rank (g // block) % nranks), but there is no host
loop and no collective per step: every rank launches ONE persistent kernel
for the whole factorization, and the ranks exchange the panel column and the
pivot-row tails by storing into each other's exchange buffers over NVLink
(CUDA IPC mappings) and signalling system-scope counters. The host does only:

1. create this rank's engine and export the IPC handle of its exchange
   buffers;
2. all-gather the handles (torch.distributed) and map the peers (connect);
3. per factorization: reset this rank's counters, barrier (every rank reset
   before any rank runs), run, read the replicated outcome.

The same kernel runs all ranks in one cooperative launch on a single GPU
(PleConfig(peer_ranks=G) on the single-matrix API), which is how the
protocol is tested on one device.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, gf2cu_stats
from .shard import ShardResult, assemble, local_rows


class PeerEngine:
    """One rank's rows and exchange buffers (C ABI gf2cu_peer_*)."""

    def __init__(self, m: int, n: int, rank: int, nranks: int, block: int = 256, device: int = 0,
                 stream: Optional[int] = None):
        L = _lib.load()
        self.stream = stream  # cudaStream_t as an int (None: the library's own stream)
        self.L = L
        self.m, self.n, self.rank, self.nranks, self.block = m, n, rank, nranks, block
        self.W = (n + 63) // 64
        self.device = device
        h = C.c_void_p()
        check(L.gf2cu_peer_create(m, n, rank, nranks, block, device, C.byref(h)))
        self.h = h
        ml = C.c_size_t()
        check(L.gf2cu_peer_info(h, C.byref(ml)))
        self.m_local = ml.value
        self.last_stats = {}

    def _s(self):
        return C.c_void_p(self.stream) if self.stream else None

    def close(self):
        if getattr(self, "h", None):
            self.L.gf2cu_peer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self) -> bytes:
        buf = (C.c_ubyte * _lib.PEER_HANDLE_BYTES)()
        check(self.L.gf2cu_peer_export(self.h, buf))
        return bytes(buf)

    def connect(self, handles) -> None:
        assert len(handles) == self.nranks
        blob = b"".join(handles)
        assert len(blob) == self.nranks * _lib.PEER_HANDLE_BYTES
        buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        check(self.L.gf2cu_peer_connect(self.h, buf))

    def upload(self, words: np.ndarray) -> None:
        words = np.ascontiguousarray(words, dtype=np.uint64)
        check(self.L.gf2cu_peer_upload(self.h, words.ctypes.data_as(C.POINTER(C.c_uint64)),
                                       words.shape[1] if words.ndim == 2 else 1, self._s()))

    def fill_ctr(self, seed: int) -> None:
        check(self.L.gf2cu_peer_fill_ctr(self.h, C.c_uint64(seed), self._s()))

    def ping(self, value: int) -> list:
        """Store `value` into every rank's marker word for this rank through
        the peer mappings (value 0: only read); returns this rank's markers."""
        seen = (C.c_uint32 * self.nranks)()
        check(self.L.gf2cu_peer_ping(self.h, C.c_uint32(value), seen))
        return list(seen)

    def reset(self) -> None:
        check(self.L.gf2cu_peer_reset(self.h, self._s()))

    def run(self) -> dict:
        st = gf2cu_stats()
        check(self.L.gf2cu_peer_run(self.h, self._s(), C.byref(st)))
        self.last_stats = {f: getattr(st, f) for f, _ in gf2cu_stats._fields_}
        return self.last_stats

    def download(self, out: np.ndarray) -> None:
        """This rank's rows (local order) into `out` (m_local x >= W words)."""
        check(self.L.gf2cu_peer_download(self.h, out.ctypes.data_as(C.POINTER(C.c_uint64)), out.shape[1],
                                         self._s()))

    def finish(self) -> ShardResult:
        cap = max(1, min(self.m, self.n))
        swaps = np.empty(cap, dtype=np.uintp)
        q = np.empty(cap, dtype=np.uintp)
        perm = np.empty(max(1, self.m), dtype=np.uint32)
        rank = C.c_size_t()
        szp = C.POINTER(C.c_size_t)
        check(self.L.gf2cu_peer_finish(self.h, swaps.ctypes.data_as(szp), q.ctypes.data_as(szp),
                                       C.byref(rank), perm.ctypes.data_as(C.POINTER(C.c_uint32)), self._s()))
        Wd = max(1, self.W)
        loc = np.zeros((max(1, self.m_local), Wd), dtype=np.uint64)
        check(self.L.gf2cu_peer_download(self.h, loc.ctypes.data_as(C.POINTER(C.c_uint64)), Wd, self._s()))
        r = int(rank.value)
        return ShardResult(r, swaps[:r].astype(np.uint64), q[:r].astype(np.uint64),
                           perm[: self.m].astype(np.int64), loc[: self.m_local])


def exchange_handles(engine, dist, group=None) -> list:
    """All-gather every rank's exchange-buffer handle in rank order and map
    the peers' buffers (engine.connect). Returns the handles."""
    import torch
    mine = engine.export()
    n = dist.get_world_size(group)
    if n == 1:
        handles = [mine]
    else:
        gloo = dist.get_backend(group) == "gloo"
        dev = torch.device("cpu") if gloo else torch.device("cuda", engine.device)
        t = torch.tensor(list(mine), dtype=torch.uint8, device=dev)
        parts = [torch.zeros_like(t) for _ in range(n)]
        dist.all_gather(parts, t, group=group)
        handles = [bytes(p.cpu().numpy().tobytes()) for p in parts]
    engine.connect(handles)
    return handles


def run_peer(engine, dist, group=None) -> ShardResult:
    """One factorization: reset this rank's counters, wait until every rank
    has (no rank may signal into a peer's counters before that peer reset
    them), then the persistent kernel, then the replicated outcome."""
    engine.reset()
    dist.barrier(group=group)
    engine.run()
    # On its last step every rank still signals into every peer's counters
    # and no rank waits for those signals; a rank that reset for its next run
    # before a slow peer's late signal landed would start one count ahead.
    # run() returns once this rank's kernel has completed, so after this
    # barrier every kernel (and every store it issued) is done.
    dist.barrier(group=group)
    return engine.finish()


def peer_block_iterative_ple(words: np.ndarray, m: int, n: int, block: int = 256, group=None,
                             device: Optional[int] = None):
    """block_iterative_ple of the m x n host matrix `words` (every rank passes
    the same input) row-sharded over the torch.distributed group, one GPU per
    rank. Returns (this rank's ShardResult, assembled L\\E on every rank)."""
    import torch
    import torch.distributed as dist
    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device() if device is None else device
    eng = PeerEngine(m, n, rank, nranks, block=block, device=dev)
    try:
        exchange_handles(eng, dist, group)
        eng.upload(words[local_rows(m, rank, nranks, block)])
        res = run_peer(eng, dist, group)
        # every rank gathers every rank's rows (padded to the largest share)
        gloo = dist.get_backend(group) == "gloo"
        gdev = torch.device("cpu") if gloo else torch.device("cuda", dev)
        mloc = torch.tensor([res.local_words.shape[0]], device=gdev)
        sizes = [torch.zeros_like(mloc) for _ in range(nranks)]
        dist.all_gather(sizes, mloc, group=group)
        mx = int(max(int(s.item()) for s in sizes))
        pad = np.zeros((mx, res.local_words.shape[1]), dtype=np.uint64)
        pad[: res.local_words.shape[0]] = res.local_words
        t = torch.from_numpy(pad.view(np.int64)).to(gdev)
        parts = [torch.zeros_like(t) for _ in range(nranks)]
        dist.all_gather(parts, t, group=group)
        results = [ShardResult(res.rank, res.swaps, res.q, res.perm,
                               parts[o].cpu().numpy().view(np.uint64)[: int(sizes[o].item())])
                   for o in range(nranks)]
        return res, assemble(results, m, n, nranks, block)
    finally:
        eng.close()
