"""The reference's OWN test sources, unmodified, run against the B200 path.

tests/cpp/b200_redirect.hpp is the INTEGRATION.md binding a maintainer adds:
force-included ahead of proj/tests/acceptance/acceptance_main.cpp and
proj/tests/test_ple.cpp, it rebinds block_iterative_ple, recursive_ple,
rref_from_ple, echelonize (and, in the *_all / acceptance builds, partial_ple
and undo_column_swaps) to gf2::b200:: so every call those sources make runs
on the device. __graft_entry__.build() compiles them where /root/reference
exists; the binaries travel to the GPU box.

Not applicable to a device path (documented in DESIGN.md section 6):
  * acceptance criterion 8 (timing ordinals of CPU base cases: the device
    runs every strategy through the same kernels) and criterion 9 and
    test_ple's OperationCounts (the reference's thread_local row-XOR counter,
    op_count.hpp:14, which the device path does not maintain).
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

CPP = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp")


def run(name, *args, timeout=600):
    exe = os.path.join(CPP, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    out = subprocess.run([exe, *args], capture_output=True, text=True, timeout=timeout)
    return out.returncode, out.stdout + out.stderr


def test_acceptance_gate_through_the_binding():
    rc, out = run("acceptance_b200")
    print(out)
    status = {int(m.group(2)): m.group(1) for m in re.finditer(r"\[(PASS|FAIL)\] criterion (\d+)", out)}
    assert len(status) == 10, out
    for c in (1, 2, 3, 4, 5, 6, 7, 10):
        assert status[c] == "PASS", f"criterion {c}: {out}"


@pytest.mark.parametrize("binary", ["test_ple_b200", "test_ple_b200_all"])
def test_reference_test_ple_through_the_binding(binary):
    skip = ["--skip", "OperationCounts.BlockStripesBeatLazyOnDenseInputs"] if binary.endswith("_all") else []
    rc, out = run(binary, *skip)
    print(out)
    assert "[  FAILED  ]" not in out and rc == 0, out
    assert re.search(r"\[==========\] 20 passed|\[==========\] 19 passed, 0 failed, 1 skipped", out), out
