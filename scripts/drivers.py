"""Kernel time of the super-step driver vs the single-panel persistent driver."""
import sys

import torch

import paper_1111_6549_b200 as G

for spec in sys.argv[1:]:
    m, n = (int(x) for x in spec.split("x")) if "x" in spec else (int(spec), int(spec))
    a, b = G.DeviceMatrix(m, n), G.DeviceMatrix(m, n)
    b.fill_ctr(1)
    for single in (False, True):
        ts = []
        for it in range(3):
            a.copy_from(b)
            torch.cuda.synchronize()
            o = G.block_iterative_ple(a, G.PleConfig(time_kernels=True, single_panel=single))
            ts.append(o.stats["kernel_ms"])
        print(f"{m}x{n} {'single-panel' if single else 'super-step  '} kernel ms {min(ts):.3f} "
              f"(rank {o.rank}, {16 * o.stats['alg_bytes'] / 16 / min(ts) / 1e6:.0f} GB/s effective)", flush=True)
