"""The reference's own hot-path unit tests (workload_test.cpp,
balancer_test.cpp), compiled unchanged through oracle/gtest_shim against the
reference library built from its sources (oracle/_ref).  Pins the shim and
the build recipe; the same files against libyatt_b200.so run in
test_gpu_integer.py::test_reference_unit_tests_pass_against_b200_library."""
import subprocess
from pathlib import Path

import pytest

EXE = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "reftests_ref"


@pytest.mark.skipif(not EXE.exists(), reason="oracle/_ref not built (no reference tree)")
def test_reference_unit_tests_pass_against_reference():
    res = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "31 tests, 0 failed" in res.stdout
