"""Where a bench step's time goes beyond the PLE kernel (device-resident
65536^2): restore copy, the C call's other launches and host round trips."""
import time

import torch

import paper_1111_6549_b200 as G

n = 65536
pristine, work = G.DeviceMatrix(n, n), G.DeviceMatrix(n, n)
pristine.fill_ctr(1)
for timing in (True, False):
    cfg = G.PleConfig(time_kernels=timing)
    for it in range(5):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        e[0].record()
        work.copy_from(pristine)
        e[1].record()
        h0 = time.perf_counter()
        o = G.block_iterative_ple(work, cfg)
        h1 = time.perf_counter()
        e[2].record()
        torch.cuda.synchronize()
        if it >= 2:
            print(f"time_kernels={timing}: copy {e[0].elapsed_time(e[1]):.3f} ms, ple call (device) "
                  f"{e[1].elapsed_time(e[2]):.3f} ms, host {1e3 * (h1 - h0):.3f} ms, kernel "
                  f"{o.stats['kernel_ms']:.3f} ms")
