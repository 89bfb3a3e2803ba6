"""Small invocation of every kernel (A1 TMA + generic, backward, GRPO, GAE,
moments, loss, filter/gathers, sort, shard round, LM head) — written for
`compute-sanitizer --tool memcheck`, which is closed on this pool; it now runs
plain as a launch-everything smoke (the out-of-bounds evidence is
tests/test_gpu_guard.py).  Prints "sanitize ok" when all calls return."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_07970_b200 import api, ops  # noqa: E402
from paper_2508_07970_b200._lib import check, lib  # noqa: E402

dev = torch.device("cuda:0")
# A1 (TMA path, generic path, full KL, masked rows) + fix-up
for rows, V in [(37, 4096), (9, 8200), (5, 1001)]:
    pol, ref, tgt = (ops.synth_logits(1, 0, rows, V, device=dev) if V % 8 == 0 else
                     (torch.randn(rows, V, device=dev).to(torch.bfloat16),
                      torch.randn(rows, V, device=dev).to(torch.bfloat16),
                      torch.randint(0, V, (rows,), device=dev, dtype=torch.int32)))
    mask = (torch.arange(rows, device=dev) % 3 != 1).to(torch.uint8)
    for mode in ("k3", "full"):
        out = ops.token_stats(pol, ref, tgt, mask, mode)
    if V % 8 == 0:  # backward (policy-only and FULL)
        lp, rl, en, kl = ops.token_stats(pol, ref, tgt, None, "full")
        adv = torch.randn(rows, device=dev)
        cu = torch.tensor([0, rows // 2, rows], dtype=torch.int64, device=dev)
        for mode in ("k3", "full"):
            ops.logits_grad(pol, ref, tgt, lp, rl, lp + 0.01, adv, en, kl, mask, cu,
                            ops.loss_config(agg_mode="seq-mean-token-mean"), mode, 2.0)
# A2 / A3 / A4
r = ops.synth_floats(1, 105, 0, 96, "reward", 8, device=dev)
ops.grpo_advantages(r, 8)
ops.grpo_advantages(r[3:70].contiguous(), 8, first_sample_id=3,
                    moments=ops.grpo_group_moments(r[3:70].contiguous(), 8, 3))
cu = torch.tensor([0, 1, 1, 40, 5000, 9100], dtype=torch.int64, device=dev)
v = torch.randn(9100, device=dev)
m = (torch.rand(9100, device=dev) < 0.8).to(torch.uint8)
adv, ret = ops.gae(v, v * 0.5, cu, m)
ops.whiten(adv, ops.masked_moments(adv, m), m)
for agg in ("token-mean", "seq-mean-token-mean", "seq-mean-token-sum"):
    ops.policy_loss(v, v + 0.1, adv, v.abs(), v.abs(), m, cu, ops.loss_config(agg_mode=agg))
# A5 / A6 / R4 / R10
lens = torch.randint(1, 300, (256,), dtype=torch.int64, device=dev)
rw = ops.synth_floats(2, 105, 0, 256, "reward", 16, device=dev)
plan = ops.filter_compact(rw, lens, 16)
ocu = torch.zeros(257, dtype=torch.int64, device=dev)
ocu[1:] = torch.cumsum(lens, 0)
src = torch.arange(int(ocu[-1]), dtype=torch.int32, device=dev)
dst = torch.empty(int(plan["counts"][1]), dtype=torch.int32, device=dev)
ops.gather_varlen(src, ocu, plan["index_map"], plan["new_cu"], plan["counts"][:1], 256, dst)
ops.gather_rows(torch.arange(1024, device=dev).view(256, 4), plan["index_map"],
                plan["counts"][:1], 256, torch.empty((256, 4), dtype=torch.int64, device=dev))
ops.microbatch_aggregates(lens.to(torch.int32), lens.to(torch.int32), 7)
ops.sort_order_desc(torch.randint(0, 50, (9000,), dtype=torch.int32, device=dev))
# R3-R6 (3 shards, misaligned)
batch = api.RolloutBatch(0, [api.RolloutSample(i, 10 + i % 5) for i in range(700)])
api.run_rollout_rounds(batch, 3, api.RoundParams(api.LengthDistribution(api.NORMAL, 300, 80,
                                                                        1024),
                                                 api.RejectionConfig(0.4, True, 8), 3, 16, 4))
api.rejection_process(batch, 2, api.RejectionConfig(0.3, False, 1), 5)
# lm head (tcgen05)
h = torch.randn(200, 256, device=dev).to(torch.bfloat16)
w = (torch.randn(1000, 256, device=dev) * 0.05).to(torch.bfloat16)
y = torch.randint(0, 1000, (200,), device=dev, dtype=torch.int32)
lp = ops.lmhead_token_stats(h, w, y, n_split=3)[0]
ops.kl_from_logps(lp, lp * 0.9, "k3")
rep = torch.zeros(6 * 4, dtype=torch.int64, device=dev)
out = torch.empty(6, dtype=torch.int64, device=dev)
check(lib().yatt_reduce_round_reports(rep.data_ptr(), 4, out.data_ptr(), None))
torch.cuda.synchronize()
print("sanitize ok")
