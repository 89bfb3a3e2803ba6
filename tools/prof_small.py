"""Profiling driver for the small per-token kernels at config-4 size (~8.4M
tokens): GAE scan, policy loss (token-mean and seq-mean), masked moments."""
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
lp = ops.synth_floats(1, 107, 0, n, "logp")
old = ops.synth_floats(1, 104, 0, n, "old_delta", base=lp)
ws = ops.LossWorkspace()
for _ in range(2):
    ops.gae(v, r, cu, m, 1.0, 0.95)
    ops.policy_loss(lp, old, v, r, r, m, None, None, ws)
    ops.policy_loss(lp, old, v, r, r, m, cu, ops.loss_config(agg_mode="seq-mean-token-mean"), ws)
    ops.masked_moments(v, m)
torch.cuda.synchronize()
print("ok")
