"""Multi-rank path on a real GPU box, including the driver's 1-GPU box.

* test_peer_world_oversubscribed: world 2 / 3 / 7 / 8 ranks (torchrun, gloo for the
  plumbing) mapped onto however many GPUs the box has (rank r -> GPU r % n;
  same-device CUDA IPC works between processes).  tools/peer_world8.py runs
  the NVLink peer-memory collectives for real and checks, against the
  single-process results: the sharded GRPO step's loss sums (fp64
  reassociation only, <= 1e-12, also under CUDA-graph replay), the global
  dynamic-sampling compaction (byte-exact packed layout from per-rank
  filters + a peer-memory scan of survivor counts), the rank-major
  all-gather, and the dynamic-sampling round loop whose reports travel only
  over peer memory (== api.run_rollout_rounds, the reference's
  TraceIsIndependentOfControllerCount invariance, simcore_test.cpp:219-244).
* test_nccl_rank_path: tools/mgpu_check.py over the C-ABI NCCL communicator
  (yatt_comm_*), one rank per GPU (NCCL refuses two ranks on one device, so a
  1-GPU box runs it at world 1)."""
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


def _torchrun(world, script, timeout):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(_port()), str(ROOT / "tools" / script)]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout,
                          env={**os.environ, "NCCL_DEBUG": "WARN", "OMP_NUM_THREADS": "1"})


@pytest.mark.parametrize("world", [2, 3, 7, 8])
def test_peer_world_oversubscribed(cuda, world):
    res = _torchrun(world, "peer_world8.py", 900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert f"peer world{world} ok" in res.stdout


def test_nccl_rank_path(cuda):
    world = min(torch.cuda.device_count(), 8)
    res = _torchrun(world, "mgpu_check.py", 600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert f"mgpu ok world={world}" in res.stdout
