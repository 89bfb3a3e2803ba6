"""N >= 2 GPUs of one box: the C-ABI NCCL communicator, the sharded GRPO
step and global compaction (tools/mgpu_check.py under torchrun).  Skipped on
single-GPU boxes; the same host logic runs on CPU in test_multiproc_cpu.py."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_multi_gpu_rank_path(cuda):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={min(n, 8)}", "--master-addr", "127.0.0.1", "--master-port",
           str(_port()), str(ROOT / "tools" / "mgpu_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                         env={**os.environ, "NCCL_DEBUG": "WARN"})
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "mgpu ok" in res.stdout
