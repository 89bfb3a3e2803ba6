"""Fused training-side op (yatt_policy_loss_grad, ops.policy_loss_grad): the
per-token loss terms and d(loss)/d(policy logits) from the policy logits
alone, each row streamed twice (second read from L2).

Checked against the fp64 oracle: logp / entropy to the A1 bar (1e-5), the
KL estimator against the stored ref_logp, the gradient with the same bf16 +
conditioning bound as test_gpu_backward.py (oracle fed the exact fp64 logp),
and against the two-kernel device path (yatt_policy_grad_coef +
yatt_logits_backward).  Masked rows are exactly zero; rows sum to ~0."""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2508_07970_b200 import ConfigError, ops

pytestmark = pytest.mark.gpu


def bf16_np(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def to_f64(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _case(cuda, rows, V, kl_mode, ent_coef=0.01, masked=False, seed=5, with_ref=True,
          agg="token-mean"):
    pol, ref, tgt = ops.synth_logits(seed, 0, rows, V, device=cuda)
    mask = None
    if masked:
        mask = torch.as_tensor((np.arange(rows) % 4 != 1).astype(np.uint8), device=cuda)
    # the experience stage's stored reference log-probs and old log-probs
    dlp, drl, _, _ = ops.token_stats(pol, ref, tgt, None, "k3")
    rlogp = drl if with_ref else None
    old = ops.synth_floats(seed, 104, 0, rows, "old_delta", base=dlp, device=cuda)
    adv = ops.synth_floats(seed, 108, 0, rows, "adv", device=cuda)
    cfg = ops.loss_config(0.2, 0.28, 0.0, 0.05, ent_coef, agg)
    nvalid = rows if mask is None else int(mask.sum())
    cu = None
    if agg != "token-mean":  # three sequences, one of them empty -> norm = 2 sequences
        cu = torch.tensor([0, rows // 3, rows // 3, rows], dtype=torch.int64, device=cuda)
        nvalid = 2
    full = kl_mode == "full"
    lp, ent, kl, grad = ops.policy_loss_grad(pol, tgt, old, adv, None if full else rlogp, mask,
                                             cfg, kl_mode, float(nvalid), cu_seqlens=cu,
                                             ref_logits=ref if full else None)
    torch.cuda.synchronize()
    hp = bf16_np(pol)
    ht = tgt.cpu().numpy()
    m = None if mask is None else mask.cpu().numpy()
    valid = np.ones(rows, bool) if m is None else m.astype(bool)
    # per-token terms vs the fp64 oracle
    hr = bf16_np(ref)
    e_lp, _, e_ent, e_klf = O.token_stats(hp, hr, ht, None, "full")
    assert O.max_rel_error(lp.cpu().numpy()[valid], e_lp[valid]) <= 1e-5
    assert O.max_rel_error(ent.cpu().numpy()[valid], e_ent[valid]) <= 1e-5
    e_rl = drl.cpu().numpy().astype(np.float64) if with_ref else e_lp
    d = e_rl - e_lp
    e_kl = {"k1": -d, "k2": 0.5 * d * d, "k3": np.expm1(d) - d, "full": e_klf}[kl_mode]
    gk = kl.cpu().numpy().astype(np.float64)
    # kl of (rl - logp): conditioned on |d| (logp carries the 1e-5 A1 bar);
    # full KL: the A1 bar
    tol_kl = (1e-5 * np.abs(e_kl) + 2e-5 * np.abs(e_lp) * (np.abs(d) + 1.0) if not full
              else 1e-5 * np.abs(e_kl) + 1e-7 * np.log(V))
    assert np.all(np.abs(gk[valid] - e_kl[valid]) <= tol_kl[valid])
    if m is not None:
        assert np.all(lp.cpu().numpy()[~valid] == 0)
    # gradient vs the fp64 oracle backward, fed the exact logp
    eg, ecoef = O.logits_backward(hp, hr, ht, e_lp, e_rl if with_ref else None,
                                  old.cpu().numpy(), adv.cpu().numpy(), m,
                                  None if cu is None else cu.cpu().numpy(), 0.2, 0.28, 0.0,
                                  0.05, ent_coef, ops.AGG_MODES[agg], kl_mode, float(nvalid))
    got = to_f64(bf16_np(grad))
    x = to_f64(hp)
    lpv = x - ecoef[:, 3:4]
    p = np.exp(lpv)
    H = -(p * lpv).sum(1, keepdims=True)
    cond = np.abs(ecoef[:, 0:1]) + np.abs(ecoef[:, 1:2]) * (np.abs(lpv) + H)
    if full:
        z = to_f64(hr)
        zm = z.max(1, keepdims=True)
        lq = z - (zm + np.log(np.exp(z - zm).sum(1, keepdims=True)))
        cond = cond + np.abs(ecoef[:, 2:3]) * (np.abs(lpv) + np.abs(lq) + 1.0)
    tol = 2.0 ** -8 * np.abs(eg) + 1e-5 * p * cond + 1e-30
    # the target element carries + g: relative 1e-5 of g from the logp used
    tol[np.arange(rows), ht] += 1e-5 * np.abs(ecoef[:, 0])
    bad = np.abs(got - eg) > tol
    assert not bad.any(), (np.argwhere(bad)[:5], got[bad][:5], eg[bad][:5])
    if m is not None:
        assert np.all(got[~valid] == 0)
    return pol, ref, tgt, mask, old, adv, rlogp, cfg, nvalid, got


@pytest.mark.parametrize("kl_mode", ["k1", "k2", "k3", "full"])
def test_fused_loss_grad_matches_oracle(cuda, kl_mode):
    _case(cuda, 40, 32000, kl_mode)


@pytest.mark.parametrize("agg", ["token-mean", "seq-mean-token-mean"])
def test_fused_full_kl(cuda, agg):
    """The full-vocabulary KL: policy AND reference tiles in every stage,
    lse_q and sum p (x - z) in pass 1, the f term in pass 2."""
    _case(cuda, 20, 152064, "full", masked=True, agg=agg)
    _case(cuda, 33, 4096, "full", agg=agg)


@pytest.mark.parametrize("agg", ["seq-mean-token-mean", "seq-mean-token-sum"])
@pytest.mark.parametrize("masked", [False, True])
def test_fused_seq_aggregations(cuda, agg, masked):
    """The seq modes: per-token scale 1 / (sequences * valid tokens of the
    sequence) for seq-mean-token-mean (a pre-kernel over cu_seqlens), 1 /
    sequences for seq-mean-token-sum — same gradient as the fp64 oracle."""
    _case(cuda, 45, 4096, "k3", masked=masked, agg=agg)
    _case(cuda, 6, 152064, "k2", agg=agg)


def test_fused_masked_rows_and_no_reference(cuda):
    _case(cuda, 37, 4096, "k3", masked=True)
    _case(cuda, 16, 4096, "k3", with_ref=False)


def test_fused_qwen_vocab_rows_sum_to_zero(cuda):
    *_, got = _case(cuda, 8, 152064, "k3", ent_coef=0.001)
    assert np.all(np.abs(got.sum(1)) <= 2e-3 * np.abs(got).max(1) * np.sqrt(got.shape[1]) / 10)


def test_fused_matches_two_kernel_path(cuda):
    """Many rows per CTA (2 x 148 CTAs): the fused gradient equals the
    two-kernel path's (coef from the same per-token values) to bf16 rounding
    and the fused kernel's fp32 coefficient rounding."""
    rows, V = 1200, 8192
    pol, ref, tgt, mask, old, adv, rlogp, cfg, nvalid, got = _case(cuda, rows, V, "k3")
    lp, ent, kl, _ = ops.policy_loss_grad(pol, tgt, old, adv, rlogp, mask, cfg, "k3",
                                          float(nvalid))
    g2, coef = ops.logits_grad(pol, ref, tgt, lp, rlogp, old, adv, ent, kl, mask, None, cfg,
                               "k3", float(nvalid))
    two = to_f64(bf16_np(g2))
    # bf16 rounding of each, plus the fused kernel's fp32 row coefficients
    # (relative ~1e-7 each) where p (h (log p + H) - g) cancels
    c = coef.cpu().numpy().astype(np.float64)
    lpv = to_f64(bf16_np(pol)) - c[:, 3:4]  # coef[3] = lse_p (nats)
    cond = np.exp(lpv) * (np.abs(c[:, 0:1]) + np.abs(c[:, 1:2]) * (np.abs(lpv) + np.abs(c[:, 5:6])))
    assert np.all(np.abs(got - two) <= 2.0 ** -7 * np.abs(two) + 1e-5 * cond
                  + 1e-12 * np.abs(two).max())


def test_fused_loss_sums_from_outputs(cuda):
    """The loss sums follow from the fused per-token outputs."""
    rows, V = 64, 4096
    pol, ref, tgt = ops.synth_logits(9, 0, rows, V, device=cuda)
    dlp, drl, dent, dkl = ops.token_stats(pol, ref, tgt, None, "k3")
    old = ops.synth_floats(9, 104, 0, rows, "old_delta", base=dlp, device=cuda)
    adv = ops.synth_floats(9, 108, 0, rows, "adv", device=cuda)
    cfg = ops.loss_config(0.2, 0.2, 0.0, 0.01, 0.0, "token-mean")
    lp, ent, kl, _ = ops.policy_loss_grad(pol, tgt, old, adv, drl, None, cfg, "k3", float(rows))
    a = ops.policy_loss(lp, old, adv, kl, ent, None, None, cfg).cpu().numpy()
    b = ops.policy_loss(dlp, old, adv, dkl, dent, None, None, cfg).cpu().numpy()
    assert O.max_rel_error(a, b) <= 1e-5


def test_fused_errors(cuda):
    pol = torch.zeros((2, 12), dtype=torch.bfloat16, device=cuda)
    tgt = torch.zeros(2, dtype=torch.int32, device=cuda)
    f = torch.zeros(2, device=cuda)
    with pytest.raises(ConfigError):  # vocab % 8 != 0
        ops.policy_loss_grad(pol, tgt, f, f)
    pol = torch.zeros((2, 16), dtype=torch.bfloat16, device=cuda)
    with pytest.raises(ConfigError):  # full-vocabulary KL needs the reference logits
        ops.policy_loss_grad(pol, tgt, f, f, kl_mode="full", ref_logits=None)
    with pytest.raises(ConfigError):  # seq-mean-token-mean needs cu_seqlens
        ops.policy_loss_grad(pol, tgt, f, f, config=ops.loss_config(agg_mode="seq-mean-token-mean"))
    with pytest.raises(ConfigError):
        ops.policy_loss_grad(pol, tgt, f, f, norm=0.0)


@pytest.mark.parametrize("rows,V", [(1, 8), (3, 16), (5, 8200), (2, 24576)])
def test_fused_edge_shapes(cuda, rows, V):
    """One row, the smallest vocabularies, a vocabulary that is not a tile
    multiple (partial last tile) and one that is exactly three tiles."""
    _case(cuda, rows, V, "k3", masked=rows > 2)


def test_fused_all_rows_masked(cuda):
    rows, V = 6, 4096
    pol, ref, tgt = ops.synth_logits(1, 0, rows, V, device=cuda)
    f = torch.zeros(rows, device=cuda)
    mask = torch.zeros(rows, dtype=torch.uint8, device=cuda)
    grad = torch.full_like(pol, 1.0)
    lp, ent, kl, g = ops.policy_loss_grad(pol, tgt, f, f, f, mask, None, "k3", 1.0, grad)
    torch.cuda.synchronize()
    assert torch.all(g.float() == 0) and torch.all(lp == 0) and torch.all(ent == 0)


@pytest.mark.parametrize("kl_mode", ["k3", "full"])
def test_fused_extreme_rows(cuda, kl_mode):
    """The rows that overflow A1's first-tile fast path (a logit 100 nats above
    the first tile, a fully -inf first tile, constant rows, a late jump just
    below the threshold): the fused kernel rebases per tile, so its logp /
    entropy / KL must come back exact (vs the fp64 oracle) and its gradient
    finite with rows summing to ~0."""
    rows, vocab = 8, 152064
    pol, ref, tgt = ops.synth_logits(9, 0, rows, vocab, device=cuda)
    ar = torch.arange(rows, device=cuda)
    keep_p, keep_r = pol[ar, tgt.long()].clone(), ref[ar, tgt.long()].clone()
    pol[0, 150000] = 100.0
    ref[1, 149000] = 96.0
    pol[2, :8192] = float("-inf")
    ref[2, :8192] = float("-inf")
    pol[3, :8192] -= 30.0
    pol[3, 140000:140100] = 40.0
    pol[4, :] = 60.0
    ref[4, :] = -60.0
    pol[5, 100000] = 88.0
    pol[ar, tgt.long()], ref[ar, tgt.long()] = keep_p, keep_r
    hp, hr = bf16_np(pol), bf16_np(ref)
    exp = O.token_stats(hp, hr, tgt.cpu().numpy(), None, "full" if kl_mode == "full" else "k3")
    old = torch.as_tensor(exp[0], dtype=torch.float32, device=cuda) - 0.05
    adv = torch.ones(rows, device=cuda)
    rl = torch.as_tensor(exp[1], dtype=torch.float32, device=cuda)
    lp, ent, kl, grad = ops.policy_loss_grad(pol, tgt, old, adv, rl, None, None, kl_mode,
                                             float(rows), ref_logits=ref)
    torch.cuda.synchronize()
    got = [t.cpu().numpy().astype(np.float64) for t in (lp, ent, kl)]
    for g_, e_ in zip(got, (exp[0], exp[2], exp[3])):
        assert np.all(np.abs(g_ - e_) <= 1e-5 * np.abs(e_) + 4e-6)
    gf = grad.float()
    assert bool(torch.isfinite(gf).all())
    assert float((gf.sum(1).abs() / (gf.abs().amax(1) * vocab ** 0.5 + 1e-30)).max()) < 1e-2


@pytest.mark.parametrize("shape", ["1:1:0", "1:0:0", "1:1:1", "2:1:1", "2:0:0"])
@pytest.mark.parametrize("kl_mode", ["k3", "full"])
def test_fused_pipelined_many_rows_per_cta(cuda, kl_mode, shape, monkeypatch):
    """Large vocabulary with several rows per CTA, so the double-buffered
    partials / coefficients of the epilogue-warp kernel cycle, in both
    compiled shapes (YATT_FUSED_PIPE = 1 large / 2 small), both pass-2 tile
    orders and with / without the one-row lag, against the fp64 oracle,
    masked rows included."""
    kernel, order, lag = shape.split(":")
    monkeypatch.setenv("YATT_FUSED_PIPE", kernel)
    monkeypatch.setenv("YATT_FUSED_ORDER", order)  # pass-2 tile order: forward / reverse
    monkeypatch.setenv("YATT_FUSED_LAG", lag)  # pass 1 of the next row before pass 2
    _case(cuda, 3 * 148 + 13, 65536, kl_mode, masked=True, ent_coef=0.001)
    # ragged tile counts: a last tile of one vector, a partial last tile
    _case(cuda, 2 * 148 + 3, 65544, kl_mode, ent_coef=0.001)
    _case(cuda, 148 + 11, 98312, kl_mode, masked=True, ent_coef=0.001)
