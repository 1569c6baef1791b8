export PYTHONPATH=.
python scripts/prof_step.py 16384 > gpurun_out/plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:panel_factor -s 100 -c 1 -o gpurun_out/prof_panel python scripts/prof_step.py 16384 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel_apply -s 100 -c 1 -o gpurun_out/prof_apply python scripts/prof_step.py 16384 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:trailing -s 60 -c 1 -o gpurun_out/prof_trail python scripts/prof_step.py 16384 > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
