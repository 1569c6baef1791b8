# Check-mode soak (VERDICT r01 "next" #2): stress_mixed.py -- random shapes,
# kinds and entry points, every PLE on one of five drivers, each result
# compared with the oracle -- under GF2CU_CHECK=1 (device invariants asserted
# every step) for every panel-schedule x pre-work-chunk setting.
# usage: bash scripts/soak_check.sh [calls per setting]
export PYTHONPATH=.:tests GF2CU_CHECK=1
N=${1:-17000}
mkdir -p gpurun_out
i=0
for f in 0 3 7; do
  for d in 64 8192; do
    i=$((i + 1))
    GF2CU_PANEL_FLAGS=$f GF2CU_PW_DIV=$d timeout 1200 python scripts/stress_mixed.py $N $((100 + i)) \
      > gpurun_out/soak_check_f${f}_d${d}.log 2>&1
    echo "flags=$f pw_div=$d rc=$?: $(tail -1 gpurun_out/soak_check_f${f}_d${d}.log)"
    grep -h MISMATCH gpurun_out/soak_check_f${f}_d${d}.log | head -5
  done
done
