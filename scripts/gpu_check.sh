export PYTHONPATH=.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python -m pytest tests/test_ple_gpu.py -x -q 2>&1 | tail -15
timeout 300 python scripts/probe.py ${PROBE_SIZES:-4096 16384 65536}
