#!/bin/bash
# Round-2 evidence: GPU tests + smoke, the default bench line, its launch list,
# and full ncu captures of the 65536^2 super-step kernel and of the 4096^2
# single-panel kernel (config 1, panel-bound). TAG names the outputs.
export PYTHONPATH=.
TAG=${TAG:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
if [ -z "$NO_TESTS" ]; then
  python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_gputests.log
  tail -3 gpurun_out/${TAG}_gputests.log
  python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?
fi
python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
cat gpurun_out/${TAG}_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo launches rc=$?
[ -n "$NO_NCU" ] && exit 0
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ple_super_kernel -c 1 \
    -o gpurun_out/${TAG}_super_65536 python scripts/one_ple.py 65536 > gpurun_out/${TAG}_ncu_super.log 2>&1
echo ncu super rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ple_persistent_kernel -c 1 \
    -o gpurun_out/${TAG}_persistent_4096 python scripts/one_ple.py 4096 > gpurun_out/${TAG}_ncu_p4096.log 2>&1
echo ncu p4096 rc=$?
ls -la gpurun_out | tail -12
