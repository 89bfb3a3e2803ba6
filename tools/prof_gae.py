"""Profiling driver: GAE over 2048 packed sequences, lengths U[1, 8192]."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2508_07970_b200 import api, ops  # noqa: E402
lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 8192, 8192), 2048, 20250814)
cu = torch.zeros(2049, dtype=torch.int64, device="cuda")
cu[1:] = torch.cumsum(torch.tensor(lens, device="cuda"), 0)
n = int(cu[-1])
v = ops.synth_floats(1, 106, 0, n, "value")
r = ops.synth_floats(1, 111, 0, n, "kl")
m = torch.ones(n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ops.gae(v, r, cu, m, 1.0, 0.95)
torch.cuda.synchronize()
print("ok")
