"""CPU, world_size 2 and 4 over gloo: the multi-rank orchestration of the
row-sharded PLE (paper_1111_6549_b200/shard.py::run_sharded) with the numpy
test engine, assembled and compared bit-exactly with the oracle. Covers the
asynchronous step protocol (sum all-reduce of the active panel column, full
scans on window misses, pivot tails packed into the stage by their owners and
summed -- small blocks give many owners per step), the lagged stop check and
the final assembly."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O  # noqa: E402
from paper_1111_6549_b200.shard import assemble, local_rows, run_sharded


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    "dense": lambda: (O.fill_random(150, 200, 0.5, 3), 150, 200),
    "tall_sparse": lambda: (O.fill_random(260, 130, 1 / 32, 4), 260, 130),
    "wide_ctr": lambda: (O.fill_ctr(90, 300, 5), 90, 300),
    "deficient": lambda: (O.mul(O.fill_ctr(200, 70, 6), 70, O.fill_ctr(70, 190, 7), 190), 200, 190),
}


def _worker(rank, world, port, case, block, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from shard_engine_np import NumpyShardEngine
    a, m, n = CASES[case]()
    eng = NumpyShardEngine(a[local_rows(m, rank, world, block)], m, n, rank, world, block)
    res = run_sharded(eng, dist)
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case,block", [("dense", 16), ("tall_sparse", 8), ("wide_ctr", 32),
                                        ("deficient", 4)])
def test_sharded_orchestration_gloo(world, case, block):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, block, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(world):
            rk, res = q.get(timeout=300)
            results[rk] = res
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    a, m, n = CASES[case]()
    ref = a.copy()
    want = O.ple(ref, m, n)
    rs = [results[r] for r in range(world)]
    for r in rs:  # replicated outcome identical on every rank
        assert r.rank == want.rank
        assert np.array_equal(r.swaps, want.swaps.astype(np.uint64))
        assert np.array_equal(r.q, want.q.astype(np.uint64))
    got = assemble(rs, m, n, world, block)
    assert np.array_equal(got, ref)
