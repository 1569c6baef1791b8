# A/B of the panel tuning bits (GF2CU_PANEL_FLAGS) on kernel time, after a
# parity pass of the panel tests. usage: bash scripts/ab_panel.sh "3 7" "4096 16384 32768 65536"
FLAGS=${1:-"3 7"}
SIZES=${2:-"4096 16384 32768 65536"}
[ -n "$SKIP_TESTS" ] || python -m pytest tests/test_ple_gpu.py -x -q -k "tuning or medium or small_shapes" 2>&1 | tail -3
for f in $FLAGS; do
  echo "== GF2CU_PANEL_FLAGS=$f"
  GF2CU_PANEL_FLAGS=$f PYTHONPATH=. python scripts/kprobe.py $SIZES
done
