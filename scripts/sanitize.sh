#!/bin/bash
# Race / sync / init / memory checks of the device path on small mixed cases
# (scripts/stress_mixed.py) under compute-sanitizer; logs into gpurun_out/.
export PYTHONPATH=.
export GF2CU_WATCHDOG_S=600
mkdir -p gpurun_out
N=${SAN_ITERS:-25}
timeout 900 python scripts/stress_mixed.py ${STRESS_ITERS:-1500} 7 > gpurun_out/stress_mixed.log 2>&1
echo "stress rc=$?"; tail -2 gpurun_out/stress_mixed.log
for tool in ${SAN_TOOLS:-memcheck synccheck racecheck initcheck}; do
  timeout ${SAN_TIMEOUT:-600} compute-sanitizer --tool $tool --print-limit 20 python scripts/stress_mixed.py $N 3 \
    > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|stress_mixed|MISMATCH" gpurun_out/san_$tool.log | tail -3
done
