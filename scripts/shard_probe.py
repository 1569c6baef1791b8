"""Time the sharded driver at world_size 1 (NCCL) vs the persistent driver."""
import os, sys, time
import numpy as np, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_1111_6549_b200 as G
from paper_1111_6549_b200 import shard as S
for n in [int(x) for x in sys.argv[1:]]:
    a = G.BitMatrix(n, n); G.fill_ctr(a, 1)
    eng = S.GpuShardEngine(n, n, 0, 1, block=256, device=0)
    for it in range(2):
        eng.upload(a.words)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        res = S.run_sharded(eng, dist)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(f"sharded world1 n={n} it={it}: {1e3*(t1-t0):.1f} ms rank {res.rank}", flush=True)
    eng.close()
dist.destroy_process_group()
