"""CPU, world_size 2 and 4 over gloo: the host side of the device-driven
row-sharded PLE (paper_1111_6549_b200/peer.py) -- the IPC-handle all-gather
in rank order, the reset -> barrier -> run sequence, and the assembly of the
ranks' rows by the replicated position order -- with a test double in place
of the CUDA engine (the kernel itself is covered on the GPU by the
peer_ranks emulation tests)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1111_6549_b200.peer import exchange_handles, run_peer
from paper_1111_6549_b200.shard import ShardResult, assemble, local_of, owner_of

HB = 64  # GF2CU_PEER_HANDLE_BYTES


class FakePeerEngine:
    """Stands in for PeerEngine: handles encode (rank, nonce); finish()
    returns this rank's rows of the oracle's result in local order."""

    def __init__(self, full, m, n, rank, nranks, block):
        self.full, self.m, self.n = full, m, n
        self.rank, self.nranks, self.block = rank, nranks, block
        self.device = 0
        self.events = []
        self.handles = None

    def export(self):
        return bytes([self.rank, 0xA5] + [(self.rank * 7 + i) & 255 for i in range(HB - 2)])

    def connect(self, handles):
        self.handles = handles
        self.events.append("connect")

    def reset(self):
        self.events.append("reset")

    def run(self):
        assert self.events[-1] == "reset"
        self.events.append("run")
        return {}

    def finish(self):
        ref = self.full.copy()
        want = O.ple(ref, self.m, self.n)
        idx = np.arange(self.m)
        for i, s in enumerate(np.asarray(want.swaps, dtype=np.int64)):
            idx[i], idx[s] = idx[s], idx[i]
        inv = np.empty_like(idx)
        inv[idx] = np.arange(self.m)
        g = np.arange(self.m)
        mine = g[owner_of(g, self.nranks, self.block) == self.rank]
        assert np.array_equal(local_of(mine, self.nranks, self.block), np.arange(mine.size))
        return ShardResult(want.rank, want.swaps.astype(np.uint64), want.q.astype(np.uint64),
                           idx.astype(np.int64), ref[inv[mine]])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, block, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = O.fill_random(230, 170, 0.5, 11)
    eng = FakePeerEngine(a, 230, 170, rank, world, block)
    handles = exchange_handles(eng, dist)
    res1 = run_peer(eng, dist)
    res2 = run_peer(eng, dist)  # a second factorization re-resets first
    out_q.put((rank, handles, eng.events, res1, res2))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,block", [(2, 16), (4, 8)])
def test_peer_host_protocol_gloo(world, block):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, block, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in range(world):
            rk, handles, events, r1, r2 = q.get(timeout=300)
            got[rk] = (handles, events, r1, r2)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    for rk in range(world):
        handles, events, _, _ = got[rk]
        assert [h[0] for h in handles] == list(range(world))  # rank order
        assert all(len(h) == HB and h[1] == 0xA5 for h in handles)
        assert events == ["connect", "reset", "run", "reset", "run"]
    a = O.fill_random(230, 170, 0.5, 11)
    ref = a.copy()
    O.ple(ref, 230, 170)
    for k in (2, 3):
        rs = [got[r][k] for r in range(world)]
        assert np.array_equal(assemble(rs, 230, 170, world, block), ref)
