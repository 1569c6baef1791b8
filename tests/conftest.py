"""Test configuration: the `gpu` marker (tests that need a B200) and repo
paths. `-m "not gpu"` runs on the CPU container; `-m gpu` on the GPU box."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (B200)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")
