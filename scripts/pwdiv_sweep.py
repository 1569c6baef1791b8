"""Kernel time vs the pre-work chunk knob (GF2CU_PW_DIV) at one size."""
import os
import subprocess
import sys

n = sys.argv[1] if len(sys.argv) > 1 else "65536"
for dv in sys.argv[2:] or ["2048", "4096", "8192", "16384", "32768"]:
    env = dict(os.environ, GF2CU_PW_DIV=dv)
    code = (f"import paper_1111_6549_b200 as G\n"
            f"d=G.DeviceMatrix({n},{n}); ts=[]\n"
            f"for _ in range(3):\n"
            f"    d.fill_ctr(1); ts.append(G.block_iterative_ple(d, G.PleConfig(time_kernels=True)).stats['kernel_ms'])\n"
            f"print('{n} pw_div {dv}:', round(min(ts), 3), 'ms')\n")
    print(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.strip(),
          flush=True)
