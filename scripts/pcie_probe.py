import torch, time
n = 512 * 1024 * 1024 // 8
h = torch.empty(n, dtype=torch.int64, pin_memory=True)
d = torch.empty(n, dtype=torch.int64, device="cuda")
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    h.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"H2D {1e3*(t1-t0):.2f} ms ({n*8/(t1-t0)/1e9:.1f} GB/s)  D2H {1e3*(t2-t1):.2f} ms ({n*8/(t2-t1)/1e9:.1f} GB/s)")
