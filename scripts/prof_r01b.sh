#!/bin/bash
# Round-1 (second half) profiles: bench launch list, one full capture of the
# super-step kernel at 65536^2, and the peer-driver kernel at 65536^2 (1 rank).
export PYTHONPATH=.
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
python scripts/one_ple.py 65536 > gpurun_out/one_plain.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ple_super_kernel -c 1 \
    -o gpurun_out/super_65536_r01b python scripts/one_ple.py 65536 > gpurun_out/ncu_super.log 2>&1
ls -la gpurun_out
