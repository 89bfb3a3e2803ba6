"""A2 GRPO advantages, A3 GAE (+ whitening), A4 policy loss on the B200 vs the
fp64 CPU oracle: max_rel_error <= 1e-5 (north star; the reference's metric,
proj/src/distattn.cpp:234-244).  Inputs are generated identically on both
sides (synth recipe), never derived from a previous kernel's outputs."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2508_07970_b200 import ConfigError, ops

pytestmark = pytest.mark.gpu
TOL = 1e-5


# ------------------------------------------------------------------- A2 ----
@pytest.mark.parametrize("G,n", [(8, 2048), (16, 16384), (5, 1000), (1, 7)])
@pytest.mark.parametrize("norm", [True, False])
def test_grpo_advantages_match_oracle(cuda, G, n, norm):
    r = ops.synth_floats(20250814, 105, 0, n, "reward", G, device=cuda)
    got = ops.grpo_advantages(r, G, 1e-6, norm).cpu().numpy()
    exp = O.grpo_advantages(r.cpu().numpy(), G, 1e-6, norm)
    assert O.max_rel_error(got, exp.astype(np.float32)) <= TOL
    # zero-variance groups: exactly zero signal (DAPO filter consistency)
    e = exp.reshape(-1, G) if n % G == 0 else None
    if e is not None:
        assert np.all(got.reshape(-1, G)[np.all(e == 0, axis=1)] == 0.0)


def test_grpo_continuous_rewards(cuda):
    n, G = 4096, 8
    r = torch.randn(n, device=cuda) * 3 + 1
    got = ops.grpo_advantages(r, G).cpu().numpy()
    exp = O.grpo_advantages(r.cpu().numpy(), G)
    assert O.max_rel_error(got, exp.astype(np.float32)) <= TOL


def test_grpo_groups_straddling_ranks(cuda):
    """Misaligned shards (P=3 over 96 samples, G=8): local moments per rank,
    merged for the straddling groups (Chan et al.), equal the single-rank
    result.  The exchange itself is yatt_comm_allgather in production."""
    n, G, P = 96, 8, 3
    r_all = torch.randn(n, device=cuda)
    full = ops.grpo_advantages(r_all, G).cpu().numpy()
    bounds = [(0, 35), (35, 70), (70, 96)]
    moms = {}
    for b, e in bounds:  # each rank: local (n, mean, M2) per overlapped group
        m = ops.grpo_group_moments(r_all[b:e].contiguous(), G, b).cpu().numpy()
        for k, row in enumerate(m):
            g = b // G + k
            if g in moms:  # Chan merge
                na, ma, qa = moms[g]
                nb, mb, qb = row
                nn = na + nb
                d = mb - ma
                moms[g] = (nn, ma + d * nb / nn, qa + qb + d * d * na * nb / nn)
            else:
                moms[g] = tuple(row)
    for b, e in bounds:
        g0, g1 = b // G, (e - 1) // G
        table = torch.tensor([moms[g] for g in range(g0, g1 + 1)], dtype=torch.float64,
                             device=cuda)
        got = ops.grpo_advantages(r_all[b:e].contiguous(), G, first_sample_id=b,
                                  moments=table).cpu().numpy()
        assert O.max_rel_error(got, full[b:e]) <= TOL


def test_broadcast_to_tokens(cuda):
    vals = torch.randn(5, device=cuda)
    cu = torch.tensor([0, 3, 3, 10, 11, 20], dtype=torch.int64, device=cuda)
    mask = (torch.arange(20, device=cuda) % 4 != 0).to(torch.uint8)
    out = ops.broadcast_to_tokens(vals, cu, 20, mask).cpu()
    exp = torch.repeat_interleave(vals.cpu(), torch.tensor([3, 0, 7, 1, 9])) * mask.cpu()
    assert torch.equal(out, exp)


# ------------------------------------------------------------------- A3 ----
@pytest.mark.parametrize("masked", [False, True])
def test_gae_matches_oracle(cuda, masked):
    rng = np.random.default_rng(1)
    lens = np.concatenate([[1, 2, 31, 32, 33, 8192], rng.integers(1, 8193, size=58)])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(cu[-1])
    v = ops.synth_floats(3, 106, 0, n, "value", device=cuda)
    r = (ops.synth_floats(3, 111, 0, n, "kl", device=cuda) * 4 - 0.5).contiguous()
    m = torch.as_tensor((rng.random(n) < 0.85).astype(np.uint8), device=cuda) if masked else None
    d_cu = torch.as_tensor(cu, device=cuda)
    adv, ret = ops.gae(v, r, d_cu, m, 1.0, 0.95)
    e_adv, e_ret = O.gae(v.cpu().numpy(), r.cpu().numpy(), cu,
                         None if m is None else m.cpu().numpy(), 1.0, 0.95)
    assert O.max_rel_error(adv.cpu().numpy(), e_adv.astype(np.float32)) <= TOL
    assert O.max_rel_error(ret.cpu().numpy(), e_ret.astype(np.float32)) <= TOL


@pytest.mark.parametrize("layout", ["multi_tile", "tiny_seqs", "offset_and_pad", "unaligned"])
def test_gae_tiled_scan_layouts(cuda, layout):
    """The scan's tile carries: sequences spanning several 4,096-token tiles,
    thousands of 1-token sequences per tile, packed arrays that start after
    token 0 / end before n_tokens (untouched outside), and an unaligned view
    (scalar path)."""
    rng = np.random.default_rng(7)
    lead, tail, shift = 0, 0, 0
    if layout == "multi_tile":
        lens = np.array([3 * 4096 + 5, 4096, 1, 4095, 20000, 3])
    elif layout == "tiny_seqs":
        lens = np.concatenate([np.ones(5000, dtype=np.int64), [4097], np.ones(3000, dtype=np.int64),
                               rng.integers(1, 6, size=2000)])
    elif layout == "offset_and_pad":
        lens, lead, tail = rng.integers(1, 9000, size=40), 4093, 5000
    else:
        lens, shift = rng.integers(1, 9000, size=40), 1
    n = lead + int(lens.sum()) + tail
    cu = np.concatenate([[lead], lead + np.cumsum(lens)]).astype(np.int64)
    buf = ops.synth_floats(5, 106, 0, n + shift, "value", device=cuda)
    v = buf[shift:]
    r = (ops.synth_floats(5, 111, 0, n, "kl", device=cuda) * 4 - 0.5).contiguous()
    for masked in (False, True):
        m = torch.as_tensor((rng.random(n) < 0.8).astype(np.uint8), device=cuda) if masked else None
        adv, ret = ops.gae(v, r, torch.as_tensor(cu, device=cuda), m, 0.99, 0.95)
        hv, hr = v.cpu().numpy(), r.cpu().numpy()
        e_adv, e_ret = O.gae(hv, hr, cu, None if m is None else m.cpu().numpy(), 0.99, 0.95)
        sl = slice(lead, n - tail)
        assert O.max_rel_error(adv.cpu().numpy()[sl], e_adv[sl].astype(np.float32)) <= TOL
        assert O.max_rel_error(ret.cpu().numpy()[sl], e_ret[sl].astype(np.float32)) <= TOL
    if lead or tail:  # tokens outside [cu[0], cu[n_seqs]) keep their contents
        from paper_2508_07970_b200._lib import check, lib
        a = torch.full((n,), 7.0, device=cuda)
        b = torch.full((n,), 7.0, device=cuda)
        wsb = lib().yatt_gae_workspace_bytes(n)
        ws = torch.empty((wsb,), dtype=torch.uint8, device=cuda)
        d_cu = torch.as_tensor(cu, device=cuda)
        check(lib().yatt_gae(v.data_ptr(), r.data_ptr(), None, d_cu.data_ptr(), len(lens), n,
                             0.99, 0.95, a.data_ptr(), b.data_ptr(), ws.data_ptr(), wsb,
                             torch.cuda.current_stream().cuda_stream))
        out = torch.cat([a[:lead], a[n - tail:], b[:lead], b[n - tail:]])
        assert bool((out == 7.0).all())
        with pytest.raises(ConfigError):  # workspace sized for fewer tokens
            check(lib().yatt_gae(v.data_ptr(), r.data_ptr(), None, d_cu.data_ptr(), len(lens), n,
                                 0.99, 0.95, a.data_ptr(), b.data_ptr(), ws.data_ptr(),
                                 lib().yatt_gae_workspace_bytes(n - 4096), None))


def test_gae_gamma_lambda_sweep_and_empty(cuda):
    cu = torch.tensor([0, 100, 100, 300], dtype=torch.int64, device=cuda)
    v = torch.randn(300, device=cuda)
    r = torch.randn(300, device=cuda)
    for g, lam in [(0.99, 0.95), (1.0, 1.0), (0.5, 0.0), (0.0, 0.9)]:
        adv, ret = ops.gae(v, r, cu, None, g, lam)
        e_adv, e_ret = O.gae(v.cpu().numpy(), r.cpu().numpy(), cu.cpu().numpy(), None, g, lam)
        assert O.max_rel_error(adv.cpu().numpy(), e_adv.astype(np.float32)) <= TOL
    a, _ = ops.gae(torch.empty(0, device=cuda), torch.empty(0, device=cuda),
                   torch.zeros(1, dtype=torch.int64, device=cuda))
    assert a.numel() == 0


def test_masked_moments_and_whiten(cuda):
    n = 1_000_003
    x = torch.randn(n, device=cuda) * 2 + 0.5
    m = (torch.rand(n, device=cuda) < 0.7).to(torch.uint8)
    mom = ops.masked_moments(x, m)
    e = O.masked_moments(x.cpu().numpy(), m.cpu().numpy())
    assert O.max_rel_error(mom.cpu().numpy(), e) <= 1e-12
    y = x.clone()
    ops.whiten(y, mom, m, shift_mean=True)
    xm = x.cpu().double().numpy()[m.cpu().numpy() == 1]
    exp = (xm - xm.mean()) / np.sqrt(xm.var(ddof=1) + 1e-8)
    got = y.cpu().numpy()[m.cpu().numpy() == 1]
    assert O.max_rel_error(got, exp.astype(np.float32)) <= TOL
    assert torch.equal(y[m == 0], x[m == 0])


# ------------------------------------------------------------------- A4 ----
def _loss_inputs(cuda, n, seed=1):
    logp = ops.synth_floats(seed, 107, 0, n, "logp", device=cuda)
    old = ops.synth_floats(seed, 104, 0, n, "old_delta", base=logp, device=cuda)
    adv = ops.synth_floats(seed, 108, 0, n, "adv", device=cuda)
    kl = ops.synth_floats(seed, 109, 0, n, "kl", device=cuda)
    ent = ops.synth_floats(seed, 110, 0, n, "kl", device=cuda)
    return logp, old, adv, kl, ent


@pytest.mark.parametrize("agg", ["token-mean", "seq-mean-token-mean", "seq-mean-token-sum"])
@pytest.mark.parametrize("clip_c", [0.0, 3.0])
def test_policy_loss_matches_oracle(cuda, agg, clip_c):
    rng = np.random.default_rng(2)
    lens = rng.integers(0, 4097, size=300)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(cu[-1])
    logp, old, adv, kl, ent = _loss_inputs(cuda, n)
    mask = torch.as_tensor((rng.random(n) < 0.9).astype(np.uint8), device=cuda)
    cfg = ops.loss_config(0.2, 0.28, clip_c, 0.01, 0.001, agg)
    sums = ops.policy_loss(logp, old, adv, kl, ent, mask, torch.as_tensor(cu, device=cuda), cfg)
    got = sums.cpu().numpy()
    exp = O.policy_loss(*(t.cpu().numpy() for t in (logp, old, adv, kl, ent)),
                        mask.cpu().numpy(), cu, 0.2, 0.28, clip_c, 0.01, 0.001,
                        ops.AGG_MODES[agg])
    assert O.max_rel_error(got, exp) <= TOL
    assert got[4] > 0  # clipping exercised
    assert abs(ops.loss_finalize(got, cfg) - ops.loss_finalize(exp, cfg)) <= \
        TOL * abs(ops.loss_finalize(exp, cfg))


def test_policy_loss_config_errors(cuda):
    logp, old, adv, kl, ent = _loss_inputs(cuda, 16)
    with pytest.raises(ConfigError):
        ops.policy_loss(logp, old, adv, kl, ent, config=ops.loss_config(clip_low=1.5))
    with pytest.raises(ConfigError):
        ops.policy_loss(logp, old, adv, kl, ent, config=ops.loss_config(agg_mode=1))


def test_grpo_step_host_matches_device_pipeline(cuda):
    """yatt_grpo_step_host (host buffers, one C-ABI call) == the same ops
    composed on the device."""
    R, T, V, seed = 8, 96, 32000, 5
    rows = R * T
    pol, ref, tgt = ops.synth_logits(seed, 0, rows, V, device=cuda)
    rew = ops.synth_floats(seed, 105, 0, R, "reward", R, device=cuda)
    logp, rlogp, ent, kl = ops.token_stats(pol, ref, tgt, None, "k3")
    old = ops.synth_floats(seed, 104, 0, rows, "old_delta", base=logp, device=cuda)
    cu = torch.arange(R + 1, dtype=torch.int64, device=cuda) * T
    tadv = ops.broadcast_to_tokens(ops.grpo_advantages(rew, R), cu, rows)
    cfg = ops.loss_config(0.2, 0.28, 0.0, 0.01, 0.001)
    dev_sums = ops.policy_loss(logp, old, tadv, kl, ent, None, None, cfg).cpu().numpy()
    stats = np.empty((4, rows), dtype=np.float32)
    host_sums = ops.grpo_step_host(pol.cpu(), ref.cpu(), tgt.cpu(), rew.cpu(), old.cpu(), R,
                                   None, 0, cfg, "k3", stats)
    assert O.max_rel_error(np.array(host_sums), dev_sums) <= 1e-12
    assert np.array_equal(stats, torch.stack([logp, rlogp, ent, kl]).cpu().numpy())


# ------------------------------------------------------ end-to-end, cfg 1 ---
def test_config1_experience_pipeline_matches_oracle(cuda):
    """BASELINE configs[0]: 16 prompts x 8 responses, T=256, V=32000 —
    A1 -> A2 -> token broadcast -> A4, end to end vs the CPU oracle."""
    P, R, T, V, seed = 16, 8, 256, 32000, 20250814
    rows = P * R * T
    pol, ref, tgt = ops.synth_logits(seed, 0, rows, V, device=cuda)
    logp, rlogp, ent, kl = ops.token_stats(pol, ref, tgt, None, "k3")
    rewards = ops.synth_floats(seed, 105, 0, P * R, "reward", R, device=cuda)
    adv = ops.grpo_advantages(rewards, R)
    cu = torch.arange(P * R + 1, dtype=torch.int64, device=cuda) * T
    tadv = ops.broadcast_to_tokens(adv, cu, rows)
    old = ops.synth_floats(seed, 104, 0, rows, "old_delta", base=logp, device=cuda)
    cfg = ops.loss_config(0.2, 0.2, 0.0, 0.001, 0.0, "token-mean")
    sums = ops.policy_loss(logp, old, tadv, kl, ent, None, None, cfg).cpu().numpy()

    hp, hr, ht = O.synth_logits(seed, 0, rows, V)
    st = O.token_stats(hp, hr, ht, None, "k3")
    for i, t in enumerate((logp, rlogp, ent, kl)):
        assert O.max_rel_error(t.cpu().numpy(), st[i]) <= TOL
    e_adv = O.grpo_advantages(rewards.cpu().numpy(), R)
    e_tadv = np.repeat(e_adv, T).astype(np.float32)
    e_old = (st[0].astype(np.float32) + (old - logp).cpu().numpy()).astype(np.float32)
    e_sums = O.policy_loss(st[0].astype(np.float32), e_old, e_tadv, st[3].astype(np.float32),
                           st[2].astype(np.float32))
    # fields: loss, pg, kl, entropy, clip_count, ratio, token_count, seq_count
    # (a) A4 over the device's own A1 outputs: every field at 1e-5, counts exact
    e_dev = O.policy_loss(logp.cpu().numpy(), old.cpu().numpy(), e_tadv, kl.cpu().numpy(),
                          ent.cpu().numpy())
    assert O.max_rel_error(sums, e_dev) <= TOL, (sums, e_dev)
    assert sums[4] == e_dev[4] and sums[6] == e_dev[6] and sums[7] == e_dev[7]
    # (b) the whole chain against the oracle's own A1: counts exact, the float
    # sums and the finalized loss at 1e-5 relative
    assert sums[6] == e_sums[6] and sums[7] == e_sums[7]
    assert sums[4] == e_sums[4], (sums[4], e_sums[4])
    for f in (0, 1, 2, 3, 5):
        assert O.max_rel_error(sums[f:f + 1], e_sums[f:f + 1]) <= TOL, (f, sums[f], e_sums[f])
    lf, ef = ops.loss_finalize(sums, cfg), ops.loss_finalize(e_sums, cfg)
    assert abs(lf - ef) <= TOL * abs(ef), (lf, ef)


def test_ops_reject_strided_and_mistyped_inputs(cuda):
    """The kernels read dense arrays: a strided view or a wrong dtype must be
    rejected in the ops layer instead of being read as if it were dense."""
    x = torch.randn(64, device=cuda)
    with pytest.raises(ValueError, match="contiguous"):
        ops.policy_loss(x[::2], x[::2].contiguous(), x[:32], x[:32], x[:32])
    with pytest.raises(TypeError):
        ops.policy_loss(x.double(), x, x, x, x)
    with pytest.raises(ValueError, match="contiguous"):
        ops.masked_moments(x[::2])
    with pytest.raises(ValueError, match="contiguous"):
        ops.gather_varlen(x[::2], torch.zeros(2, dtype=torch.int64, device=cuda),
                          torch.zeros(1, dtype=torch.int32, device=cuda),
                          torch.zeros(2, dtype=torch.int64, device=cuda),
                          torch.zeros(1, dtype=torch.int64, device=cuda), 1, x[:16])


def test_ops_reject_short_per_token_arrays(cuda):
    """Every per-token / per-sample array must hold the op's n elements: a
    shorter one would be read past its end by the kernel."""
    x = torch.randn(64, device=cuda)
    m = torch.ones(63, dtype=torch.uint8, device=cuda)
    cu = torch.tensor([0, 64], dtype=torch.int64, device=cuda)
    with pytest.raises(ValueError, match="elements"):
        ops.policy_loss(x, x, x[:32], x, x)
    with pytest.raises(ValueError, match="elements"):
        ops.policy_loss(x, x, x, x, x, m)
    with pytest.raises(ValueError, match="elements"):
        ops.gae(x, x[:63], cu)
    with pytest.raises(ValueError, match="elements"):
        ops.masked_moments(x, m)
    with pytest.raises(ValueError, match="elements"):
        ops.filter_compact(x, torch.ones(63, dtype=torch.int64, device=cuda), 8)
    pol = torch.zeros((4, 16), dtype=torch.bfloat16, device=cuda)
    tgt = torch.zeros(4, dtype=torch.int32, device=cuda)
    with pytest.raises(ValueError, match="elements"):
        ops.token_stats(pol, pol, tgt, m)
    with pytest.raises(ValueError, match="elements"):
        ops.policy_loss_grad(pol, tgt, x[:4], x[:3])
    with pytest.raises(ValueError, match="shape"):
        ops.policy_loss_grad(pol, tgt, x[:4], x[:4], grad=pol[:2])
    # token_stats `out`: a column slice of a wider [4, N] buffer (dense rows,
    # as bench.py passes per rank) is accepted and written in place
    pol2, ref2, tgt2 = ops.synth_logits(3, 0, 4, 4096, device=cuda)
    wide = torch.zeros((4, 10), device=cuda)
    ops.token_stats(pol2, ref2, tgt2, None, "k3", out=wide[:, 3:7])
    want = torch.stack(ops.token_stats(pol2, ref2, tgt2, None, "k3"))
    assert torch.equal(wide[:, 3:7], want) and torch.all(wide[:, :3] == 0)
    with pytest.raises(ValueError, match="dense rows"):
        ops.token_stats(pol2, ref2, tgt2, None, "k3", out=torch.zeros((4, 8), device=cuda)[:, ::2])


@pytest.mark.parametrize("masked", [False, True])
def test_gae_fused_whitening_moments(cuda, masked):
    """yatt_gae_with_moments: the advantages' masked moments come out of the
    scan itself and equal yatt_masked_moments over the stored advantages."""
    rng = np.random.default_rng(5)
    lens = rng.integers(1, 9000, size=300)
    cu = torch.as_tensor(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64), device=cuda)
    n = int(cu[-1])
    v = ops.synth_floats(7, 106, 0, n, "value", device=cuda)
    r = (ops.synth_floats(7, 111, 0, n, "kl", device=cuda) * 4 - 0.5).contiguous()
    m = torch.as_tensor((rng.random(n) < 0.8).astype(np.uint8), device=cuda) if masked else None
    adv, ret, mom = ops.gae(v, r, cu, m, 0.99, 0.95, return_moments=True)
    adv2, ret2 = ops.gae(v, r, cu, m, 0.99, 0.95)
    assert torch.equal(adv, adv2) and torch.equal(ret, ret2)
    ref = ops.masked_moments(adv, m).cpu().numpy()
    got = mom.cpu().numpy()
    assert got[0] == ref[0]
    assert np.all(np.abs(got - ref) <= 1e-12 * np.abs(ref) + 1e-9)


@pytest.mark.parametrize("agg", ["token-mean", "seq-mean-token-mean", "seq-mean-token-sum"])
def test_fully_masked_batches(cuda, agg):
    """Everything masked: A1 writes zeros, the loss sums are all zero (and the
    host finalize gives 0, not NaN), GAE leaves every advantage at the zero
    carry and returns = values, the moments count zero tokens — equal to the
    oracle on the same inputs."""
    rows, V = 24, 4096
    pol, ref, tgt = ops.synth_logits(4, 0, rows, V, device=cuda)
    m0 = torch.zeros(rows, dtype=torch.uint8, device=cuda)
    lp, rl, ent, kl = ops.token_stats(pol, ref, tgt, m0, "k3")
    assert all(torch.all(t == 0) for t in (lp, rl, ent, kl))
    x = ops.synth_floats(4, 107, 0, rows, "logp", device=cuda)
    cu = torch.tensor([0, 10, 10, rows], dtype=torch.int64, device=cuda)
    cfg = ops.loss_config(agg_mode=agg)
    sums = ops.policy_loss(x, x, x, x, x, m0, cu, cfg)
    assert torch.all(sums == 0)
    assert ops.loss_finalize(sums, cfg) == 0.0
    e = O.policy_loss(*(t.cpu().numpy() for t in (x, x, x, x, x)), m0.cpu().numpy(),
                      cu.cpu().numpy(), 0.2, 0.2, 0.0, 0.001, 0.0, ops.AGG_MODES[agg])
    assert np.all(e == 0)
    v = ops.synth_floats(4, 106, 0, rows, "value", device=cuda)
    adv, ret, mom = ops.gae(v, x, cu, m0, 1.0, 0.95, return_moments=True)
    e_adv, e_ret = O.gae(v.cpu().numpy(), x.cpu().numpy(), cu.cpu().numpy(), m0.cpu().numpy(),
                         1.0, 0.95)
    assert np.array_equal(adv.cpu().numpy(), e_adv.astype(np.float32))
    assert np.array_equal(ret.cpu().numpy(), e_ret.astype(np.float32))
    assert torch.all(adv == 0) and torch.equal(ret, v)
    assert mom.tolist() == [0.0, 0.0, 0.0]
