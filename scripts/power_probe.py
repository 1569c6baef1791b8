"""SM clock and power draw sampled by nvidia-smi while 65536^2 PLEs run back
to back (is the sweep power-capped?)."""
import subprocess
import time

import paper_1111_6549_b200 as G

n = 65536
a, b = G.DeviceMatrix(n, n), G.DeviceMatrix(n, n)
b.fill_ctr(1)
a.copy_from(b)
G.block_iterative_ple(a)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active",
                        "--format=csv,noheader", "-lms", "20"], stdout=subprocess.PIPE, text=True)
time.sleep(0.5)
t0 = time.time()
for _ in range(30):
    a.copy_from(b)
    G.block_iterative_ple(a)
t1 = time.time()
time.sleep(0.3)
smi.terminate()
out = smi.stdout.read().strip().splitlines()
print(f"30 PLEs in {t1 - t0:.2f} s")
for line in out[::5]:
    print(line)
