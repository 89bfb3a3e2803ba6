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
