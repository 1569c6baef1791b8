#!/bin/bash
# Soak: the GPU suite several times in a row plus a long mixed stress;
# every failure is logged (gpurun_out/soak_*.log).
export PYTHONPATH=.
mkdir -p gpurun_out
for i in $(seq 1 ${SOAK_SUITES:-3}); do
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/soak_suite_$i.log
  echo "suite $i: $(tail -1 gpurun_out/soak_suite_$i.log)"
done
timeout ${SOAK_STRESS_S:-900} python scripts/stress_mixed.py ${SOAK_STRESS_N:-20000} 11 > gpurun_out/soak_stress.log 2>&1
echo "stress rc=$?: $(tail -1 gpurun_out/soak_stress.log)"; grep MISMATCH gpurun_out/soak_stress.log | head
