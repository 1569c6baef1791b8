"""Where the sharded driver's time goes at world_size 1 (NCCL): wall time of
run_sharded vs the summed device time of its kernels (torch.profiler / CUPTI),
per kernel name. usage: python scripts/shard_prof.py 16384 32768"""
import os
import sys
import time
from collections import defaultdict

import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29541")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_1111_6549_b200 as G  # noqa: E402
from paper_1111_6549_b200 import shard as S  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [16384]:
    eng = S.GpuShardEngine(n, n, 0, 1, block=256, device=0)
    for it in range(3):
        eng.fill_ctr(1)
        torch.cuda.synchronize()
        prof = None
        if it == 2:
            prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA])
            prof.__enter__()
        t0 = time.perf_counter()
        res = S.run_sharded(eng, dist)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if prof is not None:
            prof.__exit__(None, None, None)
            agg = defaultdict(lambda: [0, 0.0])
            for e in prof.events():
                if e.device_type == torch.autograd.DeviceType.CUDA:
                    agg[e.name][0] += 1
                    agg[e.name][1] += e.device_time_total / 1e3
            tot = sum(v[1] for v in agg.values())
            print(f"n={n}: device-busy {tot:.2f} ms of {1e3 * (t1 - t0):.2f} ms wall")
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
                print(f"   {v[1]:9.3f} ms {v[0]:6d}x  {k[:90]}")
        else:
            print(f"n={n} it={it}: {1e3 * (t1 - t0):.2f} ms rank {res.rank}", flush=True)
    eng.close()
dist.destroy_process_group()
