set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_1111_6549_b200 as G; print(G.device_count())"
timeout 600 python -m pytest tests/test_ple_gpu.py -x -q 2>&1 | tail -30
