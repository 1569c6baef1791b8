"""Time the device GF(2) product c = a * b (ctr inputs), e.g. 32768x24576x32768."""
import sys
import time

import paper_1111_6549_b200 as G

for spec in sys.argv[1:]:
    m, l, n = (int(x) for x in spec.split("x"))
    da, db, dc = G.DeviceMatrix(m, l), G.DeviceMatrix(l, n), G.DeviceMatrix(m, n)
    da.fill_ctr(11)
    db.fill_ctr(12)
    for rep in range(3):
        t0 = time.perf_counter()
        G.mul_into(dc, da, db)
        t1 = time.perf_counter()
        lookup_bytes = m * ((l + 63) // 64) * ((n + 511) // 512) * 8 * 64
        print(f"{m}x{l}x{n}: {1e3*(t1-t0):.2f} ms  ({lookup_bytes/(t1-t0)/1e12:.1f} TB/s table lookups)",
              flush=True)
    for x in (da, db, dc):
        x.close()
