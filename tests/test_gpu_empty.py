"""Zero-size inputs through every device entry point.

The reference handles empty batches without special cases (an empty shard
reports zero counts, simcore_test.cpp `Step.EmptyBatchCostsOnlyOverheads`;
shard_dataset gives empty ranges when controllers outnumber samples,
workload_test.cpp:166-197).  Every op here must return YATT_OK, launch
nothing that faults, and leave well-defined outputs: zero counts / sums,
cu_seqlens = [0], untouched destinations.
"""
import numpy as np
import pytest
import torch

from paper_2508_07970_b200 import api, ops

pytestmark = pytest.mark.gpu


def _sync():
    torch.cuda.synchronize()


def test_token_stats_and_fused_paths_with_zero_rows(cuda):
    for V in (8, 50257, 152064):
        pol = torch.empty((0, V), dtype=torch.bfloat16, device=cuda)
        tgt = torch.empty((0,), dtype=torch.int32, device=cuda)
        for mode in ("k1", "k3", "full"):
            out = ops.token_stats(pol, pol, tgt, None, mode)
            assert len(out) == 4 and all(t.numel() == 0 for t in out)
    V = 4096
    pol = torch.empty((0, V), dtype=torch.bfloat16, device=cuda)
    tgt = torch.empty((0,), dtype=torch.int32, device=cuda)
    f = torch.empty((0,), device=cuda)
    for mode in ("k3", "full"):
        lp, ent, kl, grad = ops.policy_loss_grad(pol, tgt, f, f, f if mode != "full" else None,
                                                 None, None, mode, 1.0,
                                                 ref_logits=pol if mode == "full" else None)
        assert lp.numel() == 0 and grad.numel() == 0
    lp, en, ls = ops.lmhead_token_stats(torch.empty((0, 64), dtype=torch.bfloat16, device=cuda),
                                        torch.zeros((256, 64), dtype=torch.bfloat16, device=cuda),
                                        tgt)
    assert lp.numel() == 0
    assert ops.kl_from_logps(f, f).numel() == 0
    host = ops.token_stats_host(np.empty((0, 16), np.uint16), np.empty((0, 16), np.uint16),
                                np.empty((0,), np.int32))
    assert host.shape == (4, 0)
    _sync()


def test_advantages_loss_and_moments_with_zero_tokens(cuda):
    e = torch.empty((0,), device=cuda)
    assert ops.grpo_group_moments(e, 8).shape == (0, 3)
    assert ops.grpo_advantages(e, 8).numel() == 0
    cu0 = torch.zeros((1,), dtype=torch.int64, device=cuda)
    assert ops.broadcast_to_tokens(e, cu0, 0).numel() == 0
    adv, ret, mom = ops.gae(e, e, cu0, None, 1.0, 0.95, return_moments=True)
    assert adv.numel() == 0 and mom.cpu().tolist() == [0.0, 0.0, 0.0]
    assert ops.masked_moments(e).cpu().tolist() == [0.0, 0.0, 0.0]
    ops.whiten(e, torch.zeros(3, dtype=torch.float64, device=cuda))
    for agg in ("token-mean", "seq-mean-token-mean", "seq-mean-token-sum"):
        cfg = ops.loss_config(0.2, 0.2, 0.0, 0.001, 0.001, agg)
        sums = ops.policy_loss(e, e, e, e, e, None, cu0 if agg != "token-mean" else None, cfg)
        assert sums.cpu().tolist() == [0.0] * 8
        assert ops.loss_finalize(sums.cpu(), cfg) == 0.0
    _sync()


def test_filter_compaction_and_gathers_with_zero_samples(cuda):
    e = torch.empty((0,), device=cuda)
    lens = torch.empty((0,), dtype=torch.int64, device=cuda)
    plan = ops.filter_compact(e, lens, 8)
    assert plan["counts"].cpu().tolist() == [0, 0, 0]
    assert plan["new_cu"].cpu().tolist() == [0]
    assert plan["keep_groups"].numel() == 0
    # a shard of a sample-level split that received no samples
    rec = ops.filter_boundary_record(e, 8, 24)
    plan = ops.filter_compact(e, lens, 8, 24, rec.reshape(1, -1), 1)
    assert plan["counts"].cpu().tolist() == [0, 0, 0]
    # nothing kept: the gathers leave the destination untouched
    src = torch.arange(64, dtype=torch.int32, device=cuda)
    dst = torch.full((16,), -7, dtype=torch.int32, device=cuda)
    old_cu = torch.tensor([0, 64], dtype=torch.int64, device=cuda)
    imap = torch.zeros((1,), dtype=torch.int32, device=cuda)
    new_cu = torch.zeros((2,), dtype=torch.int64, device=cuda)
    n0 = torch.zeros((1,), dtype=torch.int64, device=cuda)
    ops.gather_varlen(src, old_cu, imap, new_cu, n0, 1, dst)
    ops.gather_varlen_multi([src], old_cu, imap, new_cu, n0, 1, [dst])
    ops.gather_rows(src.reshape(8, 8), imap, n0, 1, dst.reshape(2, 8))
    assert torch.all(dst == -7)
    assert ops.sort_order_desc(torch.empty((0,), dtype=torch.int32, device=cuda)).numel() == 0
    pl = torch.empty((0,), dtype=torch.int32, device=cuda)
    assert ops.microbatch_aggregates(pl, pl, 4).shape[0] == 0
    _sync()


def test_rollout_rounds_with_empty_batches_and_shards(cuda):
    """An empty batch, and more controller shards than samples (empty
    shards report zero counts), through the one-kernel round loop; the
    per-shard reports equal the reference's rules (active = pending +
    newly accepted, no microbatches for an empty shard)."""
    params = api.RoundParams(out_dist=api.LengthDistribution(api.UNIFORM, 1, 64, 64),
                             rejection=api.RejectionConfig(0.5, True, 4), seed=3,
                             microbatch_size=2, max_rounds=3)
    rounds = api.run_rollout_rounds(api.RolloutBatch(step_index=1, samples=[]), 4, params)
    for reports in rounds:
        assert all(r.active_count == 0 and not r.microbatches for r in reports)
    batch = api.RolloutBatch(step_index=2, samples=[
        api.RolloutSample(sample_id=i, prompt_len_tokens=8) for i in range(3)])
    rounds = api.run_rollout_rounds(batch, 8, params)
    assert rounds and len(rounds[0]) == 8
    for reports in rounds:
        for r in reports:
            assert r.active_count == r.pending_count + r.newly_accepted_count
            if r.active_count == 0:
                assert not r.microbatches
    assert all(s.accepted for s in batch.samples)
