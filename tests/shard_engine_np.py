"""TEST INFRASTRUCTURE: a numpy engine with the contract of the device shard
engine (paper_1111_6549_b200/shard.py::GpuShardEngine), so the multi-rank
orchestration `run_sharded` can be exercised with gloo on CPU. It restates the
per-step semantics of the kernels (panel_factor_body in window-only / full
mode, shard_apply_kernel, shard_unpack_kernel, trailing_update_kernel) on the
rank's own rows; results are checked against the oracle."""
import numpy as np
import torch

from paper_1111_6549_b200.shard import PanelStatus, ShardResult, WINDOW, local_rows, owner_of

U64 = np.uint64


def low_mask(k):
    return np.uint64((1 << k) - 1) if k < 64 else np.uint64(~0 & (2**64 - 1))


class NumpyShardEngine:
    def __init__(self, words_local, m, n, rank, nranks, block):
        self.m, self.n, self.rank, self.nranks, self.block = m, n, rank, nranks, block
        self.W = (n + 63) // 64
        self.Wpad8 = max(8, (self.W + 7) // 8 * 8)
        self.g_of = local_rows(m, rank, nranks, block)
        self.m_local = len(self.g_of)
        self.mat = np.zeros((max(1, self.m_local), self.Wpad8), dtype=U64)
        self.mat[: self.m_local, : self.W] = words_local[:, : self.W]
        self.pos_words = np.zeros(m, dtype=U64)
        self.pack = np.zeros(64 * self.Wpad8, dtype=U64)
        self.recv = np.zeros(64 * self.Wpad8, dtype=U64)
        self.stage = np.zeros((64, self.Wpad8), dtype=U64)
        # tile-major stage of the asynchronous protocol (the device layout):
        # word x of pivot slot t at ((x >> 3) * 64 + t) * 8 + (x & 7)
        self.stage_flat = np.zeros(64 * self.Wpad8, dtype=U64)

    # --- protocol -------------------------------------------------------
    def stream_ctx(self):
        import contextlib
        return contextlib.nullcontext()

    def begin(self):
        self.perm = np.arange(self.m, dtype=np.int64)
        self.inv = np.arange(self.m, dtype=np.int64)
        self.retired = np.zeros(self.m_local, dtype=bool)
        self.pbl = self.mat[: self.m_local, 0].copy()
        self.r, self.rb = 0, 0
        self.swaps, self.q = [], []

    def gather(self, lo, hi):
        self.pos_words[lo:hi] = 0
        for l in range(self.m_local):
            if self.retired[l]:
                continue
            pos = self.inv[self.g_of[l]]
            if lo <= pos < hi:
                self.pos_words[pos] = self.pbl[l]
        return torch.from_numpy(self.pos_words[lo:hi].view(np.int64))

    def panel(self, w, window_only):
        r = self.r + self.rb
        self.r, self.rb = r, 0
        m = self.m
        if r >= m:
            return PanelStatus(False, 0, r, np.zeros(self.nranks, dtype=U64))
        nrem = m - r
        nwin = min(nrem, WINDOW)
        jmax = min(64, self.n - 64 * w)
        raw = self.pos_words[r:m].copy()
        red = raw.copy()
        acc = np.zeros(nrem, dtype=U64)
        perm = self.perm[r:m].copy()
        E, D, Q, SW = [], [], [], []
        t = 0
        for j in range(jmax):
            if t >= nrem:
                break
            bit = (red[t:] >> U64(j)) & U64(1)
            win_hits = np.nonzero(bit[: max(0, nwin - t)])[0]
            if len(win_hits):
                p = t + int(win_hits[0])
            else:
                if nwin < nrem and window_only:
                    return PanelStatus(True, 0, r, np.zeros(self.nranks, dtype=U64))
                hits = np.nonzero(bit)[0]
                if not len(hits):
                    continue
                p = t + int(hits[0])
            # LAPACK swap of positions t and p
            for arr in (raw, red, acc, perm):
                arr[[t, p]] = arr[[p, t]]
            Et = red[t] & ~low_mask(j + 1)
            Dt = acc[t] ^ (U64(1) << U64(t))
            sel = np.nonzero((red[t + 1:] >> U64(j)) & U64(1))[0] + t + 1
            red[sel] ^= Et
            acc[sel] ^= Dt
            E.append(Et); D.append(Dt); Q.append(j); SW.append(p)
            t += 1
        self.pos_words[r:m] = raw
        self.perm[r:m] = perm
        self.inv[perm] = np.arange(r, m)
        self.E, self.D, self.Qb = E, D, Q
        for k in range(t):
            self.swaps.append(r + SW[k])
            self.q.append(64 * w + Q[k])
        self.rb = t
        owners = np.zeros(self.nranks, dtype=U64)
        for k in range(t):
            owners[owner_of(self.perm[r + k], self.nranks, self.block)] |= U64(1) << U64(k)
        return PanelStatus(False, t, r, owners)

    def apply(self, w):
        r, rb = self.r, self.rb
        x0 = (w + 1) & ~7
        tailw = self.Wpad8 - x0
        w0, b0 = r >> 6, r & 63
        own = [k for k in range(rb) if owner_of(self.perm[r + k], self.nranks, self.block) == self.rank]
        self.d = np.zeros(self.m_local, dtype=U64)
        self.active = ~self.retired.copy()
        for l in range(self.m_local):
            if self.retired[l]:
                continue
            off = int(self.inv[self.g_of[l]]) - r
            tl = min(off, rb)
            v, a, c = self.pbl[l], U64(0), 0
            for s in range(tl):
                if (int(v) >> self.Qb[s]) & 1:
                    v ^= self.E[s]; a ^= self.D[s]; c |= 1 << s
            epart = U64(0)
            if off < rb:
                c |= 1 << off
                epart = v & ~low_mask(self.Qb[off] + 1)
                self.retired[l] = True
                slot = own.index(off)
                self.pack[slot * tailw:(slot + 1) * tailw] = self.mat[l, x0:]
            self.d[l] = a
            row = self.mat[l]
            lo_ = U64((c << b0) & (2**64 - 1))
            hi_ = U64(c >> (64 - b0)) if b0 else U64(0)
            if w0 == w:
                row[w] = lo_ | epart
            else:
                row[w0] |= lo_
                if w0 + 1 == w:
                    row[w] = hi_ | epart
                else:
                    row[w0 + 1] |= hi_
                    row[w] = epart

    # --- asynchronous protocol (shard.py::_run_steps) --------------------
    def gather_full(self, w):
        return self.gather(0, self.m)

    def panel_full(self, w):
        self.panel(w, window_only=False)

    def pack_stage(self, w):
        x0 = (w + 1) & ~7
        lo = (x0 >> 3) * 64 * 8
        self.stage_flat[lo:] = 0
        r, rb = self.r, self.rb
        for t in range(rb):
            g = int(self.perm[r + t])
            if owner_of(g, self.nranks, self.block) != self.rank:
                continue
            l = int(np.nonzero(self.g_of == g)[0][0])
            for x in range(x0, self.Wpad8):
                self.stage_flat[((x >> 3) * 64 + t) * 8 + (x & 7)] = self.mat[l, x]
        return torch.from_numpy(self.stage_flat[lo:].view(np.int64))

    def apply_staged(self, w):
        """apply without the owner-ordered packing; the stage comes from the
        all-reduced stage_flat."""
        save = self.pack
        self.pack = np.zeros(64 * self.Wpad8, dtype=U64)
        try:
            self.apply(w)
        finally:
            self.pack = save
        x0 = (w + 1) & ~7
        for t in range(64):
            for x in range(x0, self.Wpad8):
                self.stage[t, x] = self.stage_flat[((x >> 3) * 64 + t) * 8 + (x & 7)]

    def pivots(self):
        return self.r + self.rb

    def step_gather(self, w):
        return self.gather_full(w)

    def step_panel(self, w):
        self.panel_full(w)
        return self.pack_stage(w) if w + 1 < self.W else None

    def step_update(self, w):
        self.apply_staged(w)
        self.trailing(w)

    def _tailw(self, w):
        return self.Wpad8 - ((w + 1) & ~7)

    def pack_view(self, w, cnt):
        return torch.from_numpy(self.pack[: cnt * self._tailw(w)].view(np.int64))

    def recv_view(self, w, cnt):
        return torch.from_numpy(self.recv[: cnt * self._tailw(w)].view(np.int64))

    def unpack(self, w, mask, buf):
        x0 = (w + 1) & ~7
        tailw = self.Wpad8 - x0
        data = buf.numpy().view(U64)
        ts = [k for k in range(64) if (mask >> k) & 1]
        for slot, t in enumerate(ts):
            self.stage[t, x0:] = data[slot * tailw:(slot + 1) * tailw]

    def trailing(self, w):
        if w + 1 >= self.W:
            return
        x0 = (w + 1) & ~7
        tail = self.stage[:, x0:].copy()
        # words <= w of the staged rows are not part of the update
        for x in range(x0, w + 1):
            tail[:, x - x0] = 0
        for l in range(self.m_local):
            if not self.active[l]:
                continue
            d = int(self.d[l])
            if d:
                acc = np.zeros(self.Wpad8 - x0, dtype=U64)
                for t in range(self.rb):
                    if (d >> t) & 1:
                        acc ^= tail[t]
                self.mat[l, x0:] ^= acc
            self.pbl[l] = self.mat[l, w + 1]

    def finish(self):
        rank = self.r + self.rb
        return ShardResult(rank, np.array(self.swaps[:rank], dtype=U64), np.array(self.q[:rank], dtype=U64),
                           self.perm.copy(), self.mat[: self.m_local, : max(1, self.W)].copy())
