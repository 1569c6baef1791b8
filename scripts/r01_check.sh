export PYTHONPATH=.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests/ -x -q -m gpu --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc $?
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log
