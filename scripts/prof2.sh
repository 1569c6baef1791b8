export PYTHONPATH=.
python scripts/prof_step.py 16384 > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none -c 800 --csv --log-file gpurun_out/launches16k.csv python scripts/prof_step.py 16384 > gpurun_out/ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel_factor -s 100 -c 1 -o gpurun_out/prof_panel2 python scripts/prof_step.py 16384 > gpurun_out/ncu1.log 2>&1
