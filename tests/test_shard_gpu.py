"""GPU: the row-sharded driver with the DEVICE engine (gf2cu_shard_* C ABI),
bit-exact vs the oracle. world_size 1 over NCCL, and world_size 2/3 as
processes sharing the one GPU with gloo collectives on CUDA tensors (the
per-rank kernels never wait on each other; all coordination is host-side
collectives, so this is safe on one device)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _make(case):
    if case == "dense":
        return O.fill_random(700, 900, 0.5, 11), 700, 900
    if case == "sparse":
        return O.fill_random(600, 600, 1 / 64, 12), 600, 600
    if case == "deficient":
        return O.mul(O.fill_ctr(500, 300, 13), 300, O.fill_ctr(300, 640, 14), 640), 500, 640
    if case == "big":
        return O.fill_ctr(4096, 4096, 15), 4096, 4096
    raise ValueError(case)


def _worker(rank, world, port, backend, case, block, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    kw = {"device_id": torch.device("cuda", 0)} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        from paper_1111_6549_b200.shard import sharded_block_iterative_ple
        a, m, n = _make(case)
        res, full = sharded_block_iterative_ple(a, m, n, block=block)
        q.put((rank, res.rank, res.swaps, res.q, full))
    except Exception as e:  # report instead of leaving the peer hanging
        import traceback
        q.put((rank, "error", traceback.format_exc(), None, None))
        os._exit(1)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,backend,case,block", [
    (1, "nccl", "dense", 256), (1, "nccl", "big", 256), (2, "gloo", "dense", 64),
    (2, "gloo", "sparse", 32), (3, "gloo", "deficient", 16), (2, "gloo", "big", 256)])
def test_sharded_device_engine(world, backend, case, block):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, case, block, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = []
    try:
        for _ in range(world):
            o = q.get(timeout=240)
            assert o[1] != "error", o[2]
            outs.append(o)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    a, m, n = _make(case)
    ref = a.copy()
    want = O.ple(ref, m, n)
    for (rk, rank, swaps, qq, full) in outs:
        assert rank == want.rank
        assert np.array_equal(swaps, want.swaps.astype(np.uint64))
        assert np.array_equal(qq, want.q.astype(np.uint64))
        assert np.array_equal(full, ref), f"rank {rk}"


def _peer_worker(port, case, block, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_1111_6549_b200.peer import peer_block_iterative_ple
        a, m, n = _make(case)
        res, full = peer_block_iterative_ple(a, m, n, block=block)
        q.put((0, res.rank, res.swaps, res.q, full))
    except Exception:
        import traceback
        q.put((0, "error", traceback.format_exc(), None, None))
        os._exit(1)
    dist.destroy_process_group()


@pytest.mark.parametrize("case,block", [("dense", 256), ("sparse", 64), ("deficient", 32), ("big", 256)])
def test_peer_multiprocess_api_world1(case, block):
    """The multi-process device-driven path (gf2cu_peer_*: create, handle
    exchange, reset, barrier, persistent kernel, finish, assembly) at
    world_size 1 over NCCL -- one GPU is all a test may use; more ranks run
    in the one-GPU emulation (peer_ranks tests)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_peer_worker, args=(_free_port(), case, block, q))
    p.start()
    try:
        o = q.get(timeout=240)
        assert o[1] != "error", o[2]
    finally:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    assert p.exitcode == 0
    a, m, n = _make(case)
    ref = a.copy()
    want = O.ple(ref, m, n)
    _, rank, swaps, qq, full = o
    assert rank == want.rank
    assert np.array_equal(swaps, want.swaps.astype(np.uint64))
    assert np.array_equal(qq, want.q.astype(np.uint64))
    assert np.array_equal(full, ref)


def _ping_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1111_6549_b200.peer import PeerEngine, exchange_handles
        eng = PeerEngine(3000, 2000, rank, world, block=64, device=0)
        exchange_handles(eng, dist)  # cudaIpcOpenMemHandle of every other rank
        eng.reset()
        dist.barrier()
        before = eng.ping(0)
        dist.barrier()
        eng.ping(0xC0DE00 + rank)  # stores into every rank's markers (no waiting)
        dist.barrier()
        after = eng.ping(0)
        q.put((rank, before, after))
        dist.barrier()
        eng.close()
    except Exception:
        import traceback
        q.put((rank, "error", traceback.format_exc()))
        os._exit(1)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_ipc_mappings_multiprocess(world):
    """The multi-process exchange buffers: every rank exports its buffer with
    CUDA IPC, the handles are all-gathered, every rank maps the others', and
    a store through each mapping lands in the right rank's marker word (the
    counters' offset inside the buffer included). Processes share the one
    GPU; no kernel waits on another, so this is safe on one device."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ping_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in range(world):
            o = q.get(timeout=240)
            assert o[1] != "error", o[2]
            got[o[0]] = o
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    for r in range(world):
        _, before, after = got[r]
        assert before == [0] * world
        assert after == [0xC0DE00 + s for s in range(world)]
