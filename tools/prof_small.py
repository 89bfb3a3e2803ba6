"""Profiling driver for the per-token / per-sample kernels besides A1, at the
BASELINE shapes: GAE + moments + whiten + broadcast + policy loss (token and
seq mean) over configs[3]'s ~8.4M packed tokens, and the fused 17 B/token
payload gather of configs[4] (135M tokens, ~63M kept)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2508_07970_b200 import api, ops  # noqa: E402

dev = "cuda"
lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 8192, 8192), 2048, 20250814)
cu = torch.zeros(2049, dtype=torch.int64, device=dev)
cu[1:] = torch.cumsum(torch.tensor(lens, device=dev), 0)
n = int(cu[-1])
v = ops.synth_floats(1, 106, 0, n, "value")
r = ops.synth_floats(1, 111, 0, n, "kl")
m = torch.ones(n, dtype=torch.uint8, device=dev)
lp = ops.synth_floats(1, 107, 0, n, "logp")
old = ops.synth_floats(1, 104, 0, n, "old_delta", base=lp)
ws = ops.LossWorkspace()
out = torch.empty(n, device=dev)
# configs[4] payload
G, ns = 16, 16384
glens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 16384, 16384), ns, 20250814)
d_lens = torch.tensor(glens, dtype=torch.int64, device=dev) + 64
rew = ops.synth_floats(20250814, 105, 0, ns, "reward", G)
plan = ops.filter_compact(rew, d_lens, G)
old_cu = torch.zeros(ns + 1, dtype=torch.int64, device=dev)
old_cu[1:] = torch.cumsum(d_lens, 0)
tot, kt = int(old_cu[-1]), int(plan["counts"][1])
srcs = [torch.empty(tot, dtype=t, device=dev) for t in
        (torch.int32, torch.float32, torch.float32, torch.float32, torch.uint8)]
dsts = [torch.empty(kt, dtype=s.dtype, device=dev) for s in srcs]
print("tokens", n, "payload kept tokens", kt)
for _ in range(2):
    adv, ret = ops.gae(v, r, cu, m, 1.0, 0.95)
    mom = ops.masked_moments(adv, m)
    ops.whiten(adv, mom, m)
    ops.broadcast_to_tokens(v[:2048].contiguous(), cu, n, None, out)
    ops.policy_loss(lp, old, v, r, r, m, None, None, ws)
    ops.policy_loss(lp, old, v, r, r, m, cu, ops.loss_config(agg_mode="seq-mean-token-mean"), ws)
    ops.gather_varlen_multi(srcs, old_cu, plan["index_map"], plan["new_cu"], plan["counts"][:1],
                            ns, dsts)
torch.cuda.synchronize()
print("ok")
