"""§8f #1: gradient of the A4 loss w.r.t. the policy logits vs the fp64
oracle (oracle/yatt_oracle.c yo_logits_backward).

The device writes bf16, so the bar is bf16 rounding of the exact value plus
the fp32 conditioning of the expression (cancellation between the g and h
terms): |got - exp| <= 2^-8 |exp| + 1e-5 * p_v * (|g| + |h| (|log p_v| + H) +
|f| (|log p_v| + |log q_v| + KL)).  Rows must also sum to ~0 (softmax
gradient identity) and masked rows are exactly zero."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2508_07970_b200 import ConfigError, ops

pytestmark = pytest.mark.gpu


def bf16_np(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def to_f64(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _logits(cuda, rows, V, seed, shifted):
    """synth_logits when the TMA kernel applies; otherwise (V % 8 != 0, or a
    view 2 bytes off 16-byte alignment) the generic kernel's inputs."""
    if V % 8 == 0 and not shifted:
        return ops.synth_logits(seed, 0, rows, V, device=cuda)
    g = torch.Generator(device=cuda).manual_seed(seed)

    def mat():
        buf = torch.empty(rows * V + 1, dtype=torch.bfloat16, device=cuda)
        t = buf[1:] if shifted else buf[:-1]
        t.copy_((torch.randn(rows * V, device=cuda, generator=g) * 3).to(torch.bfloat16))
        return t.view(rows, V)
    pol, ref = mat(), mat()
    tgt = torch.randint(0, V, (rows,), device=cuda, generator=g, dtype=torch.int32)
    return pol, ref, tgt


def _case(cuda, rows, V, kl_mode, agg, ent_coef, clip_c=0.0, masked=False, seed=3, shifted=False):
    pol, ref, tgt = _logits(cuda, rows, V, seed, shifted)
    mask = None
    if masked:
        mask = torch.as_tensor((np.arange(rows) % 5 != 2).astype(np.uint8), device=cuda)
    logp, rlogp, ent, kl = ops.token_stats(pol, ref, tgt, mask, kl_mode)
    old = ops.synth_floats(seed, 104, 0, rows, "old_delta", base=logp, device=cuda)
    adv = ops.synth_floats(seed, 108, 0, rows, "adv", device=cuda)
    cu = torch.tensor([0, rows // 3, rows // 3, rows], dtype=torch.int64, device=cuda)
    cfg = ops.loss_config(0.2, 0.28, clip_c, 0.05, ent_coef, agg)
    norm = float(rows if agg == "token-mean" else 2)  # non-empty sequences
    grad, coef = ops.logits_grad(pol, ref, tgt, logp, rlogp, old, adv, ent, kl, mask, cu, cfg,
                                 kl_mode, norm)
    torch.cuda.synchronize()
    hp, hr = bf16_np(pol.contiguous()), bf16_np(ref.contiguous())
    m = None if mask is None else mask.cpu().numpy()
    eg, ecoef = O.logits_backward(hp, hr, tgt.cpu().numpy(), logp.cpu().numpy(),
                                  rlogp.cpu().numpy(), old.cpu().numpy(), adv.cpu().numpy(), m,
                                  cu.cpu().numpy(), 0.2, 0.28, clip_c, 0.05, ent_coef,
                                  ops.AGG_MODES[agg], kl_mode, norm)
    got = to_f64(bf16_np(grad))
    # conditioning bound per element
    x = to_f64(hp)
    lse = ecoef[:, 3:4]
    lp = x - lse
    p = np.exp(lp)
    H = -(p * lp).sum(1, keepdims=True)
    cond = np.abs(ecoef[:, 0:1]) + np.abs(ecoef[:, 1:2]) * (np.abs(lp) + H)
    if kl_mode == "full":
        z = to_f64(hr)
        lq = z - (z.max(1, keepdims=True) + np.log(np.exp(z - z.max(1, keepdims=True)).sum(1,
                                                                                     keepdims=True)))
        cond = cond + np.abs(ecoef[:, 2:3]) * (np.abs(lp) + np.abs(lq) + 1.0)
    tol = 2.0 ** -8 * np.abs(eg) + 1e-5 * p * cond + 1e-30
    bad = np.abs(got - eg) > tol
    assert not bad.any(), (np.argwhere(bad)[:5], got[bad][:5], eg[bad][:5])
    if m is not None:
        assert np.all(got[m == 0] == 0)
    return got, eg


@pytest.mark.parametrize("kl_mode", ["k1", "k2", "k3", "full"])
def test_logits_backward_matches_oracle(cuda, kl_mode):
    _case(cuda, 48, 32000, kl_mode, "token-mean", 0.01)


@pytest.mark.parametrize("agg", ["seq-mean-token-mean", "seq-mean-token-sum"])
def test_logits_backward_seq_aggregations_and_mask(cuda, agg):
    _case(cuda, 60, 4096, "k3", agg, 0.0, clip_c=3.0, masked=True)


def test_logits_backward_qwen_vocab_rows_sum_to_zero(cuda):
    got, eg = _case(cuda, 8, 152064, "k3", "token-mean", 0.001)
    # sum_v dL/dx_v = 0 for a softmax-based loss; bf16 rounding leaves ~1e-3 relative of max
    assert np.all(np.abs(got.sum(1)) <= 2e-3 * np.abs(got).max(1) * np.sqrt(got.shape[1]) / 10)


@pytest.mark.parametrize("V,shifted", [(1001, False), (12, False), (4096, True), (9001, True)])
@pytest.mark.parametrize("kl_mode", ["k3", "full"])
def test_logits_backward_generic_path(cuda, V, shifted, kl_mode):
    """Any vocab and 2-byte-aligned views take the generic kernel: same bar."""
    _case(cuda, 19, V, kl_mode, "seq-mean-token-mean", 0.01, masked=True, shifted=shifted)


def test_logits_backward_errors(cuda):
    pol = torch.zeros((2, 12), dtype=torch.bfloat16, device=cuda)
    coef = torch.zeros((2, 8), device=cuda)
    from paper_2508_07970_b200._lib import check, lib
    with pytest.raises(ConfigError):
        check(lib().yatt_logits_backward(pol.data_ptr(), None, None, None, 2, 12,
                                         coef.data_ptr(), 0, pol.data_ptr(), None))
