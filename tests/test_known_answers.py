"""Known-answer tests for the float path (A1-A4): closed-form cases derived
from the definitions alone, checked against BOTH the CPU oracle and the CUDA
kernels.  The reference has no float implementation to pin against
(SURVEY.md §8c), so these, together with the torch / pure-Python cross-checks
in test_oracle_float.py, are what pin the conventions: entropy in nats,
Bessel-corrected group std, GAE bootstrapping to 0 at a sequence end,
token-level clipped surrogate with clip-higher bounds 1 - eps_low / 1 + eps_high.

Most answers are exactly representable (integers, halves), so the integer /
exact cases are asserted bit-for-bit; the rest to 1e-12 (oracle, fp64) or
1e-6 (device fp32 outputs of fp64 math)."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle as O

BACKENDS = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]


def _dev():
    return torch.device("cuda", 0)


def _token_stats(backend, pol_bits, ref_bits, tgt, mode):
    if backend == "oracle":
        return O.token_stats(pol_bits, ref_bits, tgt, None, mode, threads=2)
    from paper_2508_07970_b200 import ops
    d = _dev()
    as_bf16 = lambda b: torch.from_numpy(b.view(np.int16)).to(d).view(torch.bfloat16)  # noqa: E731
    out = ops.token_stats(as_bf16(pol_bits), as_bf16(ref_bits),
                          torch.from_numpy(tgt.astype(np.int32)).to(d), None, mode)
    return [t.double().cpu().numpy() for t in out]


def _tol(backend):
    return 1e-12 if backend == "oracle" else 1e-6


# ---------------------------------------------------------------- A1 ----
@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("V", [8, 4096, 152064])
@pytest.mark.parametrize("mode", ["k3", "full"])
def test_a1_uniform_logits(backend, V, mode):
    """All logits equal: p = q = uniform -> logp = -ln V, H = ln V, KL = 0."""
    rows = 3
    pol = np.full((rows, V), 0x3F80, dtype=np.uint16)  # bf16 1.0
    tgt = np.array([0, V // 2, V - 1], dtype=np.int32)
    lp, rl, ent, kl = _token_stats(backend, pol, pol.copy(), tgt, mode)
    lnv = math.log(V)
    assert O.max_rel_error(lp, np.full(rows, -lnv)) <= _tol(backend)
    assert O.max_rel_error(rl, np.full(rows, -lnv)) <= _tol(backend)
    assert O.max_rel_error(ent, np.full(rows, lnv)) <= _tol(backend)
    assert np.all(np.abs(kl) <= 1e-6), kl


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("V", [8, 32000, 152064])
def test_a1_one_raised_logit(backend, V):
    """Policy: 0 everywhere but a = 2 at the target; reference: uniform.
    Z = e^a + V - 1, logp = a - ln Z, H = ln Z - a e^a / Z, ref_logp = -ln V,
    k3 = e^D - 1 - D with D = ref_logp - logp, full KL = ln V - H."""
    a, rows = 2.0, 2
    pol = np.zeros((rows, V), dtype=np.uint16)
    tgt = np.array([1, V - 2], dtype=np.int32)
    pol[np.arange(rows), tgt] = 0x4000  # bf16 2.0
    ref = np.zeros((rows, V), dtype=np.uint16)
    Z = math.exp(a) + V - 1
    logp = a - math.log(Z)
    H = math.log(Z) - a * math.exp(a) / Z
    D = -math.log(V) - logp
    for mode, kl_exp in [("k3", math.expm1(D) - D), ("full", math.log(V) - H)]:
        lp, rl, ent, kl = _token_stats(backend, pol, ref, tgt, mode)
        assert O.max_rel_error(lp, np.full(rows, logp)) <= _tol(backend)
        assert O.max_rel_error(rl, np.full(rows, -math.log(V))) <= _tol(backend)
        assert O.max_rel_error(ent, np.full(rows, H)) <= _tol(backend)
        if backend == "gpu" and mode == "full":
            # full-vocab KL = sum p (x - y) - (lse_p - lse_q): here KL ~ 5e-5 is
            # formed from fp32 sums of size ~ln V, so the device bound is the
            # fp32 cancellation floor (absolute, ~1e-8 measured), as in
            # DESIGN.md §4 / test_gpu_token_stats.py
            assert np.all(np.abs(kl - kl_exp) <= 1e-5 * abs(kl_exp) + 2e-8 * (1 + math.log(V)))
        else:
            assert O.max_rel_error(kl, np.full(rows, kl_exp)) <= max(_tol(backend), 1e-5), mode


# ---------------------------------------------------------------- A2 ----
@pytest.mark.parametrize("backend", BACKENDS)
def test_grpo_closed_form(backend):
    """(r - mean) / (std + eps), Bessel-corrected std, G = 4.  eps = 0:
    [1,0,0,0] -> mean 1/4, std 1/2 -> (1.5, -.5, -.5, -.5) exactly;
    [1,1,0,0] -> +-0.5 / sqrt(1/3).  eps = 1e-6: a zero-variance group
    [0,0,0,0] -> exactly 0 (with eps = 0 it is 0/0, as in torch)."""
    def adv(r, eps):
        r = np.asarray(r, dtype=np.float32)
        if backend == "oracle":
            return O.grpo_advantages(r, 4, eps, True)
        from paper_2508_07970_b200 import ops
        return ops.grpo_advantages(torch.from_numpy(r).to(_dev()), 4, eps,
                                   True).double().cpu().numpy()
    s = 0.5 / math.sqrt(1.0 / 3.0)
    got = adv([1, 0, 0, 0, 1, 1, 0, 0], 0.0)
    assert np.array_equal(got[:4], [1.5, -.5, -.5, -.5])  # exact
    assert O.max_rel_error(got[4:], [s, s, -s, -s]) <= _tol(backend)
    got = adv([0, 0, 0, 0, 1, 1, 1, 1], 1e-6)
    assert np.array_equal(got, np.zeros(8))


# ---------------------------------------------------------------- A3 ----
def _gae(backend, v, r, cu, gamma, lam):
    if backend == "oracle":
        return O.gae(v, r, cu, None, gamma, lam)
    from paper_2508_07970_b200 import ops
    d = _dev()
    a, rt = ops.gae(torch.from_numpy(v).to(d), torch.from_numpy(r).to(d),
                    torch.from_numpy(cu).to(d), None, gamma, lam)
    return a.double().cpu().numpy(), rt.double().cpu().numpy()


@pytest.mark.parametrize("backend", BACKENDS)
def test_gae_closed_forms(backend):
    """gamma = lambda = 1: deltas telescope, A_t = sum_{k>=t} r_k - V_t and
    R_t = sum_{k>=t} r_k (V bootstraps to 0 at a sequence end); gamma = 0:
    A_t = r_t - V_t.  Integer data: exact in fp32 and fp64."""
    lens = [5, 3, 1, 700]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(cu[-1])
    rng = np.random.default_rng(7)
    v = rng.integers(-4, 5, n).astype(np.float32)
    r = rng.integers(-3, 4, n).astype(np.float32)
    rtg = np.zeros(n)
    for s in range(len(lens)):
        acc = 0.0
        for t in range(int(cu[s + 1]) - 1, int(cu[s]) - 1, -1):
            acc += float(r[t])
            rtg[t] = acc
    adv, ret = _gae(backend, v, r, cu, 1.0, 1.0)
    assert np.array_equal(adv, rtg - v) and np.array_equal(ret, rtg)
    adv, ret = _gae(backend, v, r, cu, 0.0, 0.95)
    assert np.array_equal(adv, r.astype(np.float64) - v) and np.array_equal(ret, r.astype(np.float64))


# ---------------------------------------------------------------- A4 ----
def _loss(backend, logp, old, adv, kl, ent, **cfg):
    if backend == "oracle":
        return O.policy_loss(logp, old, adv, kl, ent, None, None, cfg.get("clip_low", 0.2),
                             cfg.get("clip_high", 0.2), 0.0, cfg.get("kl_coef", 0.001), 0.0, 0)
    from paper_2508_07970_b200 import ops
    d = _dev()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(d)  # noqa: E731
    c = ops.loss_config(cfg.get("clip_low", 0.2), cfg.get("clip_high", 0.2), 0.0,
                        cfg.get("kl_coef", 0.001), 0.0, "token-mean")
    return ops.policy_loss(t(logp), t(old), t(adv), t(kl), t(ent), None, None, c).cpu().numpy()


@pytest.mark.parametrize("backend", BACKENDS)
def test_loss_ratio_one(backend):
    """logp == old_logp: ratio 1, never clipped, pg_t = -A_t."""
    n = 1000
    f = lambda x: np.full(n, x, dtype=np.float32)  # noqa: E731
    s = _loss(backend, f(-1.0), f(-1.0), f(0.5), f(0.25), f(0.125))
    beta = float(np.float32(0.001))
    exp = [-500.0 + beta * 250.0, -500.0, 250.0, 125.0, 0.0, 1000.0, 1000.0]
    assert np.array_equal(s[1:7], exp[1:7])  # exact sums
    assert O.max_rel_error(s[:1], exp[:1]) <= 1e-12


@pytest.mark.parametrize("backend", BACKENDS)
def test_loss_clip_higher(backend):
    """ratio = e (logp - old = 1): A = +1 -> clipped at 1 + eps_high
    (pg = -(1 + eps_high)), counted; A = -1 -> pg = e, not clipped.
    eps_low 0.2, eps_high 0.28 (DAPO clip-higher)."""
    n = 512
    logp = np.zeros(2 * n, dtype=np.float32)
    old = np.full(2 * n, -1.0, dtype=np.float32)
    adv = np.concatenate([np.ones(n), -np.ones(n)]).astype(np.float32)
    z = np.zeros(2 * n, dtype=np.float32)
    s = _loss(backend, logp, old, adv, z, z, clip_low=0.2, clip_high=0.28)
    hi = 1.0 + float(np.float32(0.28))
    pg = n * (-hi) + n * math.e
    # the oracle is fp64 throughout; the device forms each ratio in fp32
    # (ex2, ~1e-7 relative; every clip decision is still the fp64 one, so the
    # count is exact) — 100x inside the north star's 1e-5
    tol = 1e-12 if backend == "oracle" else 1e-6
    assert O.max_rel_error(s[1:2], [pg]) <= tol
    assert s[4] == n  # clip count
    assert O.max_rel_error(s[5:6], [2 * n * math.e]) <= tol
    assert s[6] == 2 * n
