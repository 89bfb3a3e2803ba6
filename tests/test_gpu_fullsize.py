"""Parity at the BASELINE sizes themselves (not only at oracle-friendly sizes):
size-independent properties over the whole output plus oracle checks on
sampled rows / the full arrays where the C oracle is fast enough.

* A1 over one bench chunk (32,768 rows x V=152,064, 20 GB of logits):
  ranges (logp <= 0, 0 <= H <= ln V, k3 KL >= 0, all finite), 32 sampled
  rows vs the fp64 oracle (max_rel_error <= 1e-5), and bit-exact row
  permutation equivariance (each row's result is independent of where and
  with which CTA it ran).
* GAE over configs[3]'s 2,048 packed sequences (~8.4M tokens) vs the oracle.
* A4 over the same ~8.4M tokens vs the oracle, all three aggregations.
* The fused loss + gradient (§8f#1) over the same bench chunk (k3 and the
  full-vocabulary KL; gradient offsets past 2^31 elements): per-token terms
  equal A1's to the 1e-5 bar, 8 sampled gradient rows vs the fp64 oracle
  backward, bit-exact row permutation equivariance.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2508_07970_b200 import api, ops

pytestmark = pytest.mark.gpu
TOL = 1e-5
SEED = 20250814


def test_token_stats_full_bench_chunk(cuda):
    rows, V = 32768, 152064
    pol, ref, tgt = ops.synth_logits(SEED, 0, rows, V, device=cuda)
    lp, rl, ent, kl = ops.token_stats(pol, ref, tgt, None, "k3")
    torch.cuda.synchronize()
    for t in (lp, rl, ent, kl):
        assert bool(torch.isfinite(t).all())
    assert bool((lp <= 0).all()) and bool((rl <= 0).all())
    assert bool((ent >= -1e-6).all()) and bool((ent <= np.log(V) + 1e-4).all())
    assert bool((kl >= -1e-6).all())
    # sampled rows vs the fp64 oracle
    idx = np.random.default_rng(1).choice(rows, size=32, replace=False)
    sel = torch.as_tensor(idx, device=cuda)
    sp = pol.index_select(0, sel).view(torch.int16).cpu().numpy().view(np.uint16)
    sr = ref.index_select(0, sel).view(torch.int16).cpu().numpy().view(np.uint16)
    st = tgt.index_select(0, sel).cpu().numpy()
    exp = O.token_stats(sp, sr, st, None, "k3")
    got = torch.stack([lp, rl, ent, kl])[:, sel].cpu().numpy()
    for k in range(4):
        assert O.max_rel_error(got[k], exp[k].astype(np.float32)) <= TOL, k
    # permutation equivariance on 4,096 rows (bit-exact)
    perm = torch.randperm(rows, generator=torch.Generator().manual_seed(3))[:4096].to(cuda)
    p2 = ops.token_stats(pol.index_select(0, perm), ref.index_select(0, perm),
                         tgt.index_select(0, perm), None, "k3")
    for a, b in zip(p2, (lp, rl, ent, kl)):
        assert torch.equal(a, b.index_select(0, perm))
    del pol, ref


def test_gae_full_config4(cuda):
    lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 8192, 8192), 2048, SEED)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(cu[-1])
    v = ops.synth_floats(SEED, 106, 0, n, "value", device=cuda)
    r = (ops.synth_floats(SEED, 111, 0, n, "kl", device=cuda) * 4 - 0.5).contiguous()
    m = (ops.synth_floats(SEED, 112, 0, n, "kl", device=cuda) < 0.95).to(torch.uint8)
    adv, ret = ops.gae(v, r, torch.as_tensor(cu, device=cuda), m, 1.0, 0.95)
    e_adv, e_ret = O.gae(v.cpu().numpy(), r.cpu().numpy(), cu, m.cpu().numpy(), 1.0, 0.95)
    assert O.max_rel_error(adv.cpu().numpy(), e_adv.astype(np.float32)) <= TOL
    assert O.max_rel_error(ret.cpu().numpy(), e_ret.astype(np.float32)) <= TOL


@pytest.mark.parametrize("agg", ["token-mean", "seq-mean-token-mean", "seq-mean-token-sum"])
def test_policy_loss_full_token_count(cuda, agg):
    lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 8192, 8192), 2048, SEED)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(cu[-1])
    logp = ops.synth_floats(SEED, 107, 0, n, "logp", device=cuda)
    old = ops.synth_floats(SEED, 104, 0, n, "old_delta", base=logp, device=cuda)
    adv = ops.synth_floats(SEED, 108, 0, n, "adv", device=cuda)
    kl = ops.synth_floats(SEED, 109, 0, n, "kl", device=cuda)
    ent = ops.synth_floats(SEED, 110, 0, n, "kl", device=cuda)
    mask = (ops.synth_floats(SEED, 113, 0, n, "kl", device=cuda) < 0.9).to(torch.uint8)
    cfg = ops.loss_config(0.2, 0.28, 3.0, 0.01, 0.001, agg)
    got = ops.policy_loss(logp, old, adv, kl, ent, mask, torch.as_tensor(cu, device=cuda),
                          cfg).cpu().numpy()
    exp = O.policy_loss(*(t.cpu().numpy() for t in (logp, old, adv, kl, ent)),
                        mask.cpu().numpy(), cu, 0.2, 0.28, 3.0, 0.01, 0.001, ops.AGG_MODES[agg])
    assert O.max_rel_error(got, exp) <= TOL


def _bf16_np(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def _to_f64(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("kl_mode", ["k3", "full"])
def test_fused_loss_grad_full_bench_chunk(cuda, kl_mode):
    rows, V = 32768, 152064
    full = kl_mode == "full"
    pol, ref, tgt = ops.synth_logits(SEED, 0, rows, V, device=cuda)
    lp1, rl1, ent1, kl1 = ops.token_stats(pol, ref, tgt, None, "full" if full else "k3")
    old = ops.synth_floats(SEED, 104, 0, rows, "old_delta", base=lp1, device=cuda)
    adv = ops.synth_floats(SEED, 108, 0, rows, "adv", device=cuda)
    cfg = ops.loss_config(0.2, 0.28, 0.0, 0.05, 0.01, "token-mean")
    args = dict(config=cfg, kl_mode=kl_mode, norm=float(rows),
                ref_logits=ref if full else None)
    lp, ent, kl, grad = ops.policy_loss_grad(pol, tgt, old, adv, None if full else rl1, None,
                                             **args)
    torch.cuda.synchronize()
    # per-token terms: A1's (parity-checked against the oracle) to the 1e-5 bar
    assert O.max_rel_error(lp.cpu().numpy(), lp1.cpu().numpy().astype(np.float64)) <= TOL
    assert O.max_rel_error(ent.cpu().numpy(), ent1.cpu().numpy().astype(np.float64)) <= TOL
    if full:
        assert O.max_rel_error(kl.cpu().numpy(), kl1.cpu().numpy().astype(np.float64)) <= TOL
    assert bool(torch.isfinite(grad.float()[:: rows // 64]).all())
    # 8 sampled gradient rows (incl. the last: offsets past 2^31) vs the oracle
    idx = np.sort(np.concatenate([np.random.default_rng(2).choice(rows - 1, 7, replace=False),
                                  [rows - 1]]))
    sel = torch.as_tensor(idx, device=cuda)
    hp, hr = _bf16_np(pol.index_select(0, sel)), _bf16_np(ref.index_select(0, sel))
    ht = tgt.index_select(0, sel).cpu().numpy()
    e_lp = O.token_stats(hp, hr, ht, None, "k3")[0]
    s_rl = rl1.index_select(0, sel).cpu().numpy().astype(np.float64)  # the stored ref log-probs
    eg, ecoef = O.logits_backward(hp, hr, ht, e_lp, None if full else s_rl,
                                  old.index_select(0, sel).cpu().numpy(),
                                  adv.index_select(0, sel).cpu().numpy(), None, None, 0.2, 0.28,
                                  0.0, 0.05, 0.01, ops.AGG_MODES["token-mean"], kl_mode,
                                  float(rows))
    got = _to_f64(_bf16_np(grad.index_select(0, sel)))
    x = _to_f64(hp)
    lpv = x - ecoef[:, 3:4]
    p = np.exp(lpv)
    H = -(p * lpv).sum(1, keepdims=True)
    cond = np.abs(ecoef[:, 0:1]) + np.abs(ecoef[:, 1:2]) * (np.abs(lpv) + H)
    if full:
        z = _to_f64(hr)
        zm = z.max(1, keepdims=True)
        lq = z - (zm + np.log(np.exp(z - zm).sum(1, keepdims=True)))
        cond = cond + np.abs(ecoef[:, 2:3]) * (np.abs(lpv) + np.abs(lq) + 1.0)
    tol = 2.0 ** -8 * np.abs(eg) + 1e-5 * p * cond + 1e-30
    tol[np.arange(len(idx)), ht] += 1e-5 * np.abs(ecoef[:, 0])
    bad = np.abs(got - eg) > tol
    assert not bad.any(), (np.argwhere(bad)[:5], got[bad][:5], eg[bad][:5])
    # bit-exact row permutation equivariance on 2,048 rows
    perm = torch.randperm(rows, generator=torch.Generator().manual_seed(4))[:2048].to(cuda)
    out2 = ops.policy_loss_grad(pol.index_select(0, perm), tgt.index_select(0, perm),
                                old.index_select(0, perm), adv.index_select(0, perm),
                                None if full else rl1.index_select(0, perm), None,
                                **{**args, "ref_logits": ref.index_select(0, perm) if full
                                   else None})
    for a, b in zip(out2, (lp, ent, kl, grad)):
        assert torch.equal(a, b.index_select(0, perm))
    del pol, ref, grad
