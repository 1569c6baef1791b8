#!/bin/bash
# End-of-round check: GPU suite, smoke, the default bench line, launch list,
# one full capture of the super-step kernel at 65536^2 and of the
# single-panel kernel at 16384^2.
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
bash scripts/prof_r01c.sh > gpurun_out/final_prof.log 2>&1
cat gpurun_out/final_pytest.log gpurun_out/final_smoke.log
