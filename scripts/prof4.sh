export PYTHONPATH=.
python scripts/prof_panel.py 16384 > gpurun_out/plain.log 2>&1 || exit 1
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:panel_factor -s 100 -c 1 -o gpurun_out/prof_panel3 python scripts/prof_panel.py 16384 > gpurun_out/ncu1.log 2>&1
