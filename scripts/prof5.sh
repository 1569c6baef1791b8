export PYTHONPATH=.
set -x
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
python scripts/prof_step.py 16384 > gpurun_out/plain2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:ple_persistent -c 1 -o gpurun_out/prof_persistent16k python scripts/prof_step.py 16384 > gpurun_out/ncu_p.log 2>&1
python scripts/prof_panel.py 65536 > gpurun_out/plain3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:trailing_update -s 30 -c 1 -o gpurun_out/prof_trailing65k python scripts/prof_panel.py 65536 > gpurun_out/ncu_t.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:trailing_update -s 0 -c 1023 --csv --log-file gpurun_out/trailing_traffic65k.csv python scripts/prof_panel.py 65536 > gpurun_out/ncu_tt.log 2>&1
ls -la gpurun_out
