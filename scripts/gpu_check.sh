set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputests.log
tail -5 gpurun_out/r2_gputests.log
python __graft_entry__.py > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench rc=$?
cat gpurun_out/r2_bench.json
