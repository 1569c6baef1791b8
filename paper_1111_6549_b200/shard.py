"""Row-sharded multi-GPU block_iterative_ple.

One process per GPU (torch.distributed, NCCL over NVLink on GPUs). Global row
g lives on rank (g // block) % nranks (block-cyclic, so every rank keeps a
near-equal share of the active rows as pivots retire). Rows never move:
positions (the reference's row order after its swaps) are a replicated
permutation that every rank updates identically by running the same panel
factorization. Per 64-column panel step w:

1. sum all-reduce of the active panel column (every rank contributes its
   own rows' panel words at their positions, 8 bytes per row);
2. every rank factors the panel from it (identical decisions everywhere);
3. every rank packs the raw tails of the pivot rows it owns straight into
   the tile-major stage (zeros elsewhere); sum all-reduce of the stage (the
   contributions are disjoint) -> the Gray-table sources on every rank;
4. every rank applies the step to its own rows (multipliers, compression,
   the d combinations) and runs the trailing update on them.

No step needs a host decision (no status read-back, no owner-dependent
broadcasts), so the host enqueues the whole loop asynchronously; it only
stops early from a lagged "all rows hold pivots" check.

The collectives use torch.distributed (NCCL on CUDA tensors, gloo on CPU
tensors), so the orchestration is also exercised by world_size-2/4 gloo tests
on CPU with a test engine (tests/test_shard_gloo.py). The device engine is
`GpuShardEngine` (C ABI gf2cu_shard_*, include/gf2cu.h).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check

WINDOW = 128


def owner_of(g, nranks: int, block: int):
    return (np.asarray(g) // block) % nranks


def local_of(g, nranks: int, block: int):
    g = np.asarray(g)
    return (g // (block * nranks)) * block + g % block


def local_rows(m: int, rank: int, nranks: int, block: int) -> np.ndarray:
    """Global ids of rank's rows, in local order."""
    g = np.arange(m)
    return g[owner_of(g, nranks, block) == rank]


@dataclass
class PanelStatus:
    miss: bool
    rb: int
    r: int
    owners: np.ndarray  # uint64 bitmask of pivots t per rank

    @staticmethod
    def from_words(words: np.ndarray, nranks: int) -> "PanelStatus":
        w = np.asarray(words, dtype=np.uint64)
        own = w[8:8 + 2 * nranks:2] | (w[9:9 + 2 * nranks:2] << np.uint64(32))
        return PanelStatus(bool(w[0]), int(w[1]), int(w[2]), own)


@dataclass
class ShardResult:
    rank: int
    swaps: np.ndarray
    q: np.ndarray
    perm: np.ndarray         # global row id at each final position
    local_words: np.ndarray  # this rank's rows (local order), L\E in place


class _HostStaged:
    """gloo has no reliable CUDA-tensor collectives: stage device tensors
    through host memory (NCCL is used as is)."""

    def __init__(self, dist, group):
        self.dist, self.group = dist, group

    def all_reduce(self, t, group=None):
        if t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, group=self.group)

    def broadcast(self, t, src, group=None):
        if t.is_cuda:
            h = t.cpu()
            self.dist.broadcast(h, src=src, group=self.group)
            t.copy_(h)
        else:
            self.dist.broadcast(t, src=src, group=self.group)


def run_sharded(engine, dist, group=None) -> ShardResult:
    """The per-step orchestration (the host logic that is tested with gloo)."""
    if dist.get_backend(group) == "gloo":
        dist, group = _HostStaged(dist, group), None
    with engine.stream_ctx():
        return _run_steps(engine, dist, group)


def _run_steps(engine, dist, group, check_every: int = 16) -> ShardResult:
    """Per 64-column panel step, with no host decision inside the step (so
    the whole loop is enqueued asynchronously on the device stream):

    1. every rank writes its active rows' panel words at their positions into
       a zeroed column; sum all-reduce -> the whole active column everywhere;
    2. every rank factors the panel from it (full scans on window misses, so
       the step never aborts; identical decisions on every rank);
    3. every rank packs the raw tails of the pivot rows it owns straight into
       the stage layout (zeros elsewhere); sum all-reduce -> all pivot tails
       everywhere (the contributions are disjoint);
    4. every rank applies the step to its rows and sweeps them.

    The host only stops early (all rows hold pivots) from a lagged check
    every `check_every` steps."""
    m, W = engine.m, engine.W
    solo = engine.nranks == 1  # the collectives are identities
    engine.begin()
    for w in range(W):
        if w and w % check_every == 0 and engine.pivots() >= m:
            break
        col = engine.step_gather(w)
        if not solo:
            dist.all_reduce(col, group=group)
        stage = engine.step_panel(w)
        if stage is not None and not solo:
            dist.all_reduce(stage, group=group)
        engine.step_update(w)
    return engine.finish()


def assemble(results, m: int, n: int, nranks: int, block: int) -> np.ndarray:
    """Rows of all ranks in final position order (the in-place L\\E)."""
    perm = results[0].perm
    Wd = (n + 63) // 64
    out = np.zeros((m, max(1, Wd)), dtype=np.uint64)
    own = owner_of(perm, nranks, block)
    loc = local_of(perm, nranks, block)
    for o in range(nranks):
        sel = own == o
        out[sel] = results[o].local_words[loc[sel]]
    return out


# ------------------------------------------------------------------ device
class GpuShardEngine:
    """Per-rank engine over the C ABI (gf2cu_shard_*); buffers are torch CUDA
    tensors so torch.distributed (NCCL) moves them directly."""

    def __init__(self, m: int, n: int, rank: int, nranks: int, block: int = 256,
                 device: int = 0, stream: Optional[int] = None):
        import torch
        self.torch = torch
        L = _lib.load()
        self.L = L
        self.m, self.n, self.rank, self.nranks, self.block = m, n, rank, nranks, block
        self.W = (n + 63) // 64
        self.Wpad8 = max(8, (self.W + 7) // 8 * 8)
        self.device = device
        h = C.c_void_p()
        check(L.gf2cu_shard_create(m, n, rank, nranks, block, device, C.byref(h)))
        self.h = h
        ml, pw = C.c_size_t(), C.c_size_t()
        check(L.gf2cu_shard_info(h, C.byref(ml), C.byref(pw)))
        self.m_local = ml.value
        dev = torch.device("cuda", device)
        self.pos_words = torch.zeros(m, dtype=torch.int64, device=dev)
        self.pack = torch.zeros(pw.value, dtype=torch.int64, device=dev)
        self.recv = torch.zeros(pw.value, dtype=torch.int64, device=dev)
        self.status = np.zeros(8 + 2 * nranks, dtype=np.uint32)
        # the stage lives in a torch tensor so the collective runs on it in place
        self.stage = torch.zeros(64 * self.Wpad8, dtype=torch.int64, device=dev)
        check(L.gf2cu_shard_set_stage(h, self._p(self.stage)))
        # One explicit stream for the library calls AND the torch copies /
        # collectives around them (run_sharded enters stream_ctx()); the legacy
        # default stream (handle 0) would leave them unordered.
        self.tstream = torch.cuda.Stream(device=dev)
        self.stream = stream if stream is not None else self.tstream.cuda_stream
        torch.cuda.synchronize(dev)

    def stream_ctx(self):
        return self.torch.cuda.stream(self.tstream)

    def _s(self):
        return C.c_void_p(self.stream)

    def close(self):
        if getattr(self, "h", None):
            self.L.gf2cu_shard_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _p(t):
        return C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_uint64))

    def download(self, out: np.ndarray):
        check(self.L.gf2cu_shard_download(self.h, out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                          out.shape[1], self._s()))

    def upload(self, words: np.ndarray):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        check(self.L.gf2cu_shard_upload(self.h, words.ctypes.data_as(C.POINTER(C.c_uint64)),
                                        words.shape[1] if words.ndim == 2 else 1, self._s()))

    def fill_ctr(self, seed: int):
        check(self.L.gf2cu_shard_fill_ctr(self.h, C.c_uint64(seed), self._s()))

    def begin(self):
        check(self.L.gf2cu_shard_begin(self.h, self._s()))

    def gather(self, lo: int, hi: int):
        check(self.L.gf2cu_shard_gather(self.h, self._p(self.pos_words), lo, hi, self._s()))
        return self.pos_words[lo:hi]

    def panel(self, w: int, window_only: bool) -> PanelStatus:
        check(self.L.gf2cu_shard_panel(self.h, w, self._p(self.pos_words), int(window_only),
                                       self.status.ctypes.data_as(C.POINTER(C.c_uint32)), self._s()))
        return PanelStatus.from_words(self.status, self.nranks)

    def apply(self, w: int):
        check(self.L.gf2cu_shard_apply(self.h, w, self._p(self.pack), self._s()))

    # --- asynchronous protocol (_run_steps) -----------------------------
    def step_gather(self, w: int):
        check(self.L.gf2cu_shard_step_gather(self.h, w, self._p(self.pos_words), self._s()))
        return self.pos_words

    def step_panel(self, w: int):
        check(self.L.gf2cu_shard_step_panel(self.h, w, self._p(self.pos_words), self._s()))
        if w + 1 >= self.W:
            return None
        x0 = (w + 1) & ~7
        return self.stage[(x0 >> 3) * 64 * 8:]

    def step_update(self, w: int):
        check(self.L.gf2cu_shard_step_update(self.h, w, self._s()))

    def gather_full(self, w: int):
        check(self.L.gf2cu_shard_gather(self.h, self._p(self.pos_words), 0, self.m, self._s()))
        return self.pos_words

    def panel_full(self, w: int):
        check(self.L.gf2cu_shard_panel(self.h, w, self._p(self.pos_words), 0, None, self._s()))

    def pack_stage(self, w: int):
        check(self.L.gf2cu_shard_pack_stage(self.h, w, self._s()))
        x0 = (w + 1) & ~7
        return self.stage[(x0 >> 3) * 64 * 8:]

    def apply_staged(self, w: int):
        check(self.L.gf2cu_shard_apply(self.h, w, None, self._s()))

    def pivots(self) -> int:
        v = C.c_size_t()
        check(self.L.gf2cu_shard_pivots(self.h, C.byref(v), self._s()))
        return int(v.value)

    def _tailw(self, w):
        x0 = (w + 1) & ~7
        return self.Wpad8 - x0

    def pack_view(self, w: int, cnt: int):
        return self.pack[: cnt * self._tailw(w)]

    def recv_view(self, w: int, cnt: int):
        return self.recv[: cnt * self._tailw(w)]

    def unpack(self, w: int, mask: int, buf):
        check(self.L.gf2cu_shard_unpack(self.h, w, C.c_uint64(mask), self._p(buf), self._s()))

    def trailing(self, w: int):
        check(self.L.gf2cu_shard_trailing(self.h, w, self._s()))

    def finish(self) -> ShardResult:
        cap = max(1, min(self.m, self.n))
        swaps = np.empty(cap, dtype=np.uintp)
        q = np.empty(cap, dtype=np.uintp)
        perm = np.empty(self.m, dtype=np.uint32)
        rank = C.c_size_t()
        szp = C.POINTER(C.c_size_t)
        check(self.L.gf2cu_shard_finish(self.h, swaps.ctypes.data_as(szp), q.ctypes.data_as(szp),
                                        C.byref(rank), perm.ctypes.data_as(C.POINTER(C.c_uint32)),
                                        self._s()))
        Wd = max(1, self.W)
        loc = np.zeros((max(1, self.m_local), Wd), dtype=np.uint64)
        check(self.L.gf2cu_shard_download(self.h, loc.ctypes.data_as(C.POINTER(C.c_uint64)), Wd,
                                          self._s()))
        r = int(rank.value)
        return ShardResult(r, swaps[:r].astype(np.uint64), q[:r].astype(np.uint64),
                           perm.astype(np.int64), loc[: self.m_local])


def sharded_block_iterative_ple(words: np.ndarray, m: int, n: int, block: int = 256,
                                group=None, device: Optional[int] = None):
    """block_iterative_ple of the m x n matrix `words` (host, all ranks pass the
    full matrix or None on non-zero ranks is not supported: every rank passes
    the same input) sharded over the default torch.distributed group.
    Returns (ShardResult of this rank, assembled L\\E on every rank)."""
    import torch
    import torch.distributed as dist
    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device() if device is None else device
    eng = GpuShardEngine(m, n, rank, nranks, block=block, device=dev)
    mine = local_rows(m, rank, nranks, block)
    eng.upload(words[mine])
    res = run_sharded(eng, dist, group)
    torch.cuda.synchronize(dev)
    # every rank gathers every rank's rows (padded to the largest share);
    # gloo has no all_gather on CUDA tensors, so it gathers host tensors
    gdev = torch.device("cpu") if dist.get_backend(group) == "gloo" else torch.device("cuda", dev)
    mloc = torch.tensor([res.local_words.shape[0]], device=gdev)
    sizes = [torch.zeros_like(mloc) for _ in range(nranks)]
    dist.all_gather(sizes, mloc, group=group)
    mx = int(max(int(s.item()) for s in sizes))
    Wd = res.local_words.shape[1]
    pad = np.zeros((mx, Wd), dtype=np.uint64)
    pad[: res.local_words.shape[0]] = res.local_words
    t = torch.from_numpy(pad.view(np.int64)).to(gdev)
    parts = [torch.zeros_like(t) for _ in range(nranks)]
    dist.all_gather(parts, t, group=group)
    results = []
    for o in range(nranks):
        lw = parts[o].cpu().numpy().view(np.uint64)[: int(sizes[o].item())]
        results.append(ShardResult(res.rank, res.swaps, res.q, res.perm, lw))
    eng.close()
    return res, assemble(results, m, n, nranks, block)
