"""Median kernel time (CUDA events around the persistent launch) of the
device-resident PLE of ctr(seed 1) matrices, with the result checksum.
usage: python scripts/kprobe.py [n ...]   (n or MxN)"""
import os
import sys

import numpy as np

import paper_1111_6549_b200 as G

for arg in sys.argv[1:] or ["4096", "16384", "32768", "65536"]:
    m, n = (int(x) for x in arg.split("x")) if "x" in arg else (int(arg), int(arg))
    a, b = G.DeviceMatrix(m, n), G.DeviceMatrix(m, n)
    b.fill_ctr(1)
    ks = []
    for it in range(6):
        a.copy_from(b)
        drv = os.environ.get("KPROBE_DRIVER", "")
        peer = int(os.environ.get("KPROBE_PEER", "0"))  # emulated peer ranks (one launch)
        o = G.block_iterative_ple(a, G.PleConfig(time_kernels=True, single_panel=drv == "single",
                                                 super_step=drv == "super", peer_ranks=peer))
        if it:
            ks.append(o.stats["kernel_ms"])
    print(f"{m}x{n}: kernel median {np.median(ks):.3f} ms (min {min(ks):.3f}) rank {o.rank} "
          f"checksum {a.checksum():#x}", flush=True)
