export PYTHONPATH=.
python scripts/prof_step.py 65536 > gpurun_out/plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:trailing -s 20 -c 1 -o gpurun_out/prof_trail65k python scripts/prof_step.py 65536 > gpurun_out/ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:trailing -s 100 -c 8 --csv --log-file gpurun_out/trail_traffic.csv python scripts/prof_step.py 65536 > gpurun_out/ncu2.log 2>&1
