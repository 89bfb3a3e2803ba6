"""The C++ host path: examples/yatt_rank.cpp, a controller rank written only
against include/yatt/*.hpp and linked to libyatt_b200.so, runs on the B200."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
EXE = Path(__file__).resolve().parents[1] / "examples" / "_build" / "yatt_rank"


def test_cpp_rank_example_runs(cuda):
    assert EXE.exists(), "built by __graft_entry__.build() (make -C examples)"
    res = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "rank ok" in res.stdout
    assert "padding waste" in res.stdout
