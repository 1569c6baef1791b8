import os, sys, time, socket
import numpy as np
import torch.multiprocessing as mp

def worker(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    import torch, torch.distributed as dist
    log = open(f"gpurun_out/shard_dbg_{rank}.log", "w", buffering=1)
    log.write("start\n")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    log.write("pg ok\n")
    import oracle as O
    from paper_1111_6549_b200 import shard as S
    a = O.fill_random(700, 900, 0.5, 11); m, n = 700, 900
    eng = S.GpuShardEngine(m, n, rank, world, block=64, device=0)
    log.write(f"engine ok m_local={eng.m_local}\n")
    eng.upload(a[S.local_rows(m, rank, world, 64)])
    class D:
        def __init__(s): s.d = dist
        def get_backend(s, g=None): return "gloo"
        def all_reduce(s, t, group=None):
            log.write(f"  all_reduce {tuple(t.shape)} {t.device}\n"); h = t.cpu(); dist.all_reduce(h); t.copy_(h)
        def broadcast(s, t, src, group=None):
            log.write(f"  bcast {tuple(t.shape)} src={src}\n"); h = t.cpu(); dist.broadcast(h, src=src); t.copy_(h)
    # instrument engine
    for name in ["begin", "gather", "panel", "apply", "unpack", "trailing", "finish"]:
        f = getattr(eng, name)
        def wrap(*a, _f=f, _n=name, **k):
            log.write(f"{time.time():.3f} {_n} {a[:2] if _n!='unpack' else a[:2]}\n"); r = _f(*a, **k)
            if _n == "panel": log.write(f"   -> {r}\n")
            return r
        setattr(eng, name, wrap)
    res = S.run_sharded(eng, D())
    log.write(f"done rank={res.rank}\n")
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, 2, port)) for r in range(2)]
    for p in ps: p.start()
    for p in ps: p.join(timeout=90)
    for p in ps:
        if p.is_alive(): p.kill(); print("killed", p.pid)
    print("exit", [p.exitcode for p in ps])
