#!/bin/bash
# Round-1 (third session) evidence: the default bench line, its launch list,
# one full capture of the super-step kernel at 65536^2 and of the single-panel
# persistent kernel at 16384^2 (config 2, panel-bound).
export PYTHONPATH=.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r01c.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_bench_r01c.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
python scripts/one_ple.py 65536 > gpurun_out/one_plain.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ple_super_kernel -c 1 \
    -o gpurun_out/super_65536_r01c python scripts/one_ple.py 65536 > gpurun_out/ncu_super.log 2>&1
python scripts/one_ple.py 16384 > gpurun_out/one_plain16.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ple_persistent_kernel -c 1 \
    -o gpurun_out/persistent_16384_r01c python scripts/one_ple.py 16384 > gpurun_out/ncu_pers16.log 2>&1
ls -la gpurun_out | tail -12
