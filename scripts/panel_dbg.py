"""Pivot-loop breakdown of the single-panel driver (GF2CU_DUMP_PHASES slot 4):
cycles the leader warp spends taking pivots alone vs the rest of the loop
(epoch barriers, catch-up of the other warps, cross-warp steps).
usage: python scripts/panel_dbg.py [n ...]"""
import os
import sys

import numpy as np

import paper_1111_6549_b200 as G

for n in [int(x) for x in sys.argv[1:]] or [4096, 16384]:
    a, b = G.DeviceMatrix(n, n), G.DeviceMatrix(n, n)
    b.fill_ctr(1)
    path = f"gpurun_out/pdbg{n}.txt"
    for it in range(2):
        a.copy_from(b)
        if it == 1:
            os.environ["GF2CU_DUMP_PHASES"] = path
        o = G.block_iterative_ple(a, G.PleConfig(time_kernels=True, single_panel=True))
    os.environ.pop("GF2CU_DUMP_PHASES")
    d = np.loadtxt(path, skiprows=1, comments="#", dtype=np.float64)
    raw = np.array([int(l.split()[7]) for l in open(path) if l[:1].isdigit()], dtype=np.uint64)
    ok = d[:, 10] > d[:, 9]
    loop_us = (d[:, 10] - d[:, 9])[ok] / 1e3
    lead_cyc = (raw >> np.uint64(32))[ok].astype(np.float64)
    lead_piv = ((raw >> np.uint64(16)) & np.uint64(0xffff))[ok].astype(np.float64)
    cross = ((raw >> np.uint64(8)) & np.uint64(0xff))[ok].astype(np.float64)
    epochs = (raw & np.uint64(0xff))[ok].astype(np.float64)
    rb = d[ok, 2]
    print(f"n={n} kernel {o.stats['kernel_ms']:.3f} ms; per panel: loop {loop_us.mean():.2f} us, "
          f"pivots {rb.mean():.1f}, leader pivots {lead_piv.mean():.1f} in {lead_cyc.mean() / 1965:.2f} us "
          f"({lead_cyc.sum() / max(1, lead_piv.sum()):.0f} cyc/pivot), epochs {epochs.mean():.2f}, "
          f"cross steps {cross.mean():.2f}")
