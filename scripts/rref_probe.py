"""Time device rref_from_ple / echelonize after a device PLE (ctr inputs)."""
import sys
import time

import paper_1111_6549_b200 as G

for spec in sys.argv[1:]:
    m, n = (int(x) for x in spec.split("x"))
    dm = G.DeviceMatrix(m, n)
    for rep in range(3):
        dm.fill_ctr(1)
        t0 = time.perf_counter()
        out = G.block_iterative_ple(dm)
        t1 = time.perf_counter()
        G.rref_from_ple(dm, out, True)
        t2 = time.perf_counter()
        print(f"{m}x{n} rank {out.rank} ple {1e3*(t1-t0):.2f} ms  rref(full) {1e3*(t2-t1):.2f} ms", flush=True)
    dm.close()
