#!/bin/bash
# A/B of the panel tuning bits (GF2CU_PANEL_FLAGS) on the small configs and
# the 65536^2 kernel time.
export PYTHONPATH=.
for f in ${FLAGS:-0 1}; do
  echo "== GF2CU_PANEL_FLAGS=$f"
  GF2CU_PANEL_FLAGS=$f timeout 300 python scripts/panel_dbg.py 4096 16384
  GF2CU_PANEL_FLAGS=$f timeout 300 python scripts/kprobe.py ${PROBE_SIZES:-4096 16384 16384x65536 32768 65536}
done
