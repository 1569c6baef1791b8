"""PCIe paths for a 512 MiB host matrix (65536^2): pinned vs pageable
uploads / downloads through gf2cu_matrix_upload / download, the cost of
cudaHostRegister on the pageable buffer, and the e2e drop-in call on each.
usage: PYTHONPATH=. python scripts/pageable_probe.py"""
import time

import numpy as np
import torch

import paper_1111_6549_b200 as G

n = 65536
W = n // 64
pin = torch.empty((n, W), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
page = np.empty((n, W), dtype=np.uint64)
d = G.DeviceMatrix(n, n)
d.fill_ctr(1)
d.download(pin)
page[:] = pin
for name, buf in (("pinned", pin), ("pageable", page)):
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.upload(buf)
        t1 = time.perf_counter()
        d.download(buf)
        t2 = time.perf_counter()
        print(f"{name}: upload {1e3 * (t1 - t0):.2f} ms ({buf.nbytes / (t1 - t0) / 1e9:.1f} GB/s), "
              f"download {1e3 * (t2 - t1):.2f} ms ({buf.nbytes / (t2 - t1) / 1e9:.1f} GB/s)", flush=True)
rt = torch.cuda.cudart()
for it in range(2):
    t0 = time.perf_counter()
    rt.cudaHostRegister(page.ctypes.data, page.nbytes, 0)
    t1 = time.perf_counter()
    d.upload(page)
    t2 = time.perf_counter()
    rt.cudaHostUnregister(page.ctypes.data)
    t3 = time.perf_counter()
    print(f"cudaHostRegister {1e3 * (t1 - t0):.2f} ms, upload registered {1e3 * (t2 - t1):.2f} ms, "
          f"unregister {1e3 * (t3 - t2):.2f} ms", flush=True)
src = pin.copy()
for name, buf in (("pinned", pin), ("pageable", page)):
    v = G.MatrixView(buf, W, 0, n, n)
    ts = []
    for it in range(3):
        buf[:] = src
        t0 = time.perf_counter()
        o = G.block_iterative_ple(v, G.PleConfig(time_kernels=True))
        ts.append(time.perf_counter() - t0)
    print(f"e2e {name}: {[round(1e3 * t, 2) for t in ts]} ms, kernel {o.stats['kernel_ms']:.2f} ms", flush=True)
