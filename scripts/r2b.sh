python -m pytest tests -m gpu -x -q > gpurun_out/r2b_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_tests.log
tail -3 gpurun_out/r2b_tests.log
PYTHONPATH=. python scripts/kprobe.py 4096 16384 32768 65536 2>&1 | tee gpurun_out/r2b_kprobe.log
KPROBE_PEER=1 PYTHONPATH=. python scripts/kprobe.py 65536 32768 2>&1 | tee -a gpurun_out/r2b_kprobe.log
PYTHONPATH=. python scripts/pageable_probe.py 2>&1 | tee gpurun_out/r2b_pageable.log
