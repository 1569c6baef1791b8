# Scratch-buffer poisoning (GF2CU_POISON=<byte>): the parity suites with every
# factorization's scratch filled with a fixed byte before each run, so a
# result that reads a stale or uninitialized scratch word fails every time.
export PYTHONPATH=.:tests
for b in 0xa5 0xff 0x00; do
  GF2CU_POISON=$b timeout 900 python -m pytest tests/test_golden_gpu.py tests/test_ple_gpu.py -q -x \
    -k "suite_golden or small_shapes or medium or tuning" -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/poison_$b.log
  echo "poison $b: $(tail -1 gpurun_out/poison_$b.log)"
  grep -E "^E  |FAILED" gpurun_out/poison_$b.log | head -5
done
