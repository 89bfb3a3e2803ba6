"""Cross-check the float half of the oracle (A1-A4) against an independent
second implementation (torch fp64, written from the definitions), the same
pattern as the reference's naive-softmax oracle check
(proj/tests/distattn_test.cpp:15-45).  The reference has no float path, so
this is what pins the oracle's conventions."""
import numpy as np
import pytest
import torch

from oracle import oracle as O


def bf16_to_f64(bits):
    return torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).double()


@pytest.mark.parametrize("kl_mode", ["k1", "k2", "k3", "full"])
def test_token_stats_oracle_vs_torch(kl_mode):
    pol, ref, tgt = O.synth_logits(5, 0, 24, 4096)
    got = O.token_stats(pol, ref, tgt, None, kl_mode, threads=4)
    x, z = bf16_to_f64(pol), bf16_to_f64(ref)
    lp, lq = torch.log_softmax(x, -1), torch.log_softmax(z, -1)
    t = torch.from_numpy(tgt).long()
    logp = lp.gather(1, t[:, None])[:, 0]
    rlogp = lq.gather(1, t[:, None])[:, 0]
    ent = -(lp.exp() * lp).sum(-1)
    d = rlogp - logp
    kl = {"k1": -d, "k2": 0.5 * d * d, "k3": torch.expm1(d) - d,
          "full": (lp.exp() * (lp - lq)).sum(-1)}[kl_mode]
    for a, b in zip(got, [logp, rlogp, ent, kl]):
        assert np.allclose(a, b.numpy(), rtol=1e-12, atol=1e-13)


def test_synthetic_target_offset_keeps_kl_conditioned():
    pol, ref, tgt = O.synth_logits(20250814, 0, 64, 32000)
    s = O.token_stats(pol, ref, tgt, None, "k3")
    assert np.min(np.abs(s[1] - s[0])) > 0.15


def test_grpo_oracle_vs_torch():
    r = O.synth_floats(3, 105, 0, 64, "reward", 8)
    got = O.grpo_advantages(r, 8, 1e-6, True)
    rt = torch.from_numpy(r).double().view(-1, 8)
    exp = (rt - rt.mean(1, keepdim=True)) / (rt.std(1, keepdim=True) + np.float32(1e-6))
    assert np.allclose(got, exp.flatten().numpy(), rtol=1e-13, atol=1e-13)
    # zero-variance groups give exactly zero advantage
    zero = rt.std(1) == 0
    assert np.all(got.reshape(-1, 8)[zero.numpy()] == 0.0)


def test_gae_oracle_vs_python_loop():
    rng = np.random.default_rng(0)
    lens = [1, 5, 33, 70]
    cu = np.concatenate([[0], np.cumsum(lens)])
    v = rng.standard_normal(cu[-1]).astype(np.float32)
    r = rng.standard_normal(cu[-1]).astype(np.float32)
    m = (rng.random(cu[-1]) < 0.8).astype(np.uint8)
    adv, ret = O.gae(v, r, cu, m, 0.99, 0.95)
    g, lam = float(np.float32(0.99)), float(np.float32(0.95))
    for s in range(len(lens)):
        A = Vn = 0.0
        for t in range(cu[s + 1] - 1, cu[s] - 1, -1):
            if m[t]:
                A = float(r[t]) + g * Vn - float(v[t]) + g * lam * A
                Vn = float(v[t])
            assert adv[t] == pytest.approx(A, rel=1e-15, abs=1e-15)
            assert ret[t] == pytest.approx(A + float(v[t]), rel=1e-15, abs=1e-15)


@pytest.mark.parametrize("agg", [0, 1, 2])
def test_policy_loss_oracle_vs_torch(agg):
    n = 300
    logp = O.synth_floats(1, 107, 0, n, "logp")
    old = O.synth_floats(1, 104, 0, n, "old_delta", base=logp)
    adv = O.synth_floats(1, 108, 0, n, "adv")
    kl = O.synth_floats(1, 109, 0, n, "kl")
    ent = O.synth_floats(1, 110, 0, n, "kl")
    mask = (np.arange(n) % 5 != 0).astype(np.uint8)
    cu = np.array([0, 17, 100, 100, 250, 300])
    got = O.policy_loss(logp, old, adv, kl, ent, mask, cu, 0.2, 0.28, 3.0, 0.01, 0.001, agg)
    t = lambda a: torch.from_numpy(np.asarray(a)).double()  # noqa: E731
    ratio = torch.exp(t(logp) - t(old))
    A = t(adv)
    f32 = lambda v: float(np.float32(v))  # noqa: E731  (configs are fp32 in the ABI)
    pg1, pg2 = -A * ratio, -A * ratio.clamp(1 - f32(0.2), 1 + f32(0.28))
    pg = torch.maximum(pg1, pg2)
    pg = torch.where(A < 0, torch.minimum(pg, -A * 3.0), pg)
    L = pg + f32(0.01) * t(kl) - f32(0.001) * t(ent)
    mk = t(mask)
    if agg == 0:
        loss_sum, cnt_seq = float((L * mk).sum()), 0.0
    else:
        terms = []
        for s in range(len(cu) - 1):
            sl = slice(cu[s], cu[s + 1])
            c = float(mk[sl].sum())
            if c > 0:
                terms.append(float((L[sl] * mk[sl]).sum()) / (c if agg == 1 else 1.0))
        loss_sum, cnt_seq = sum(terms), float(len(terms))
    exp = [loss_sum, float((pg * mk).sum()), float((t(kl) * mk).sum()),
           float((t(ent) * mk).sum()), float(((pg2 > pg1).double() * mk).sum()),
           float((ratio * mk).sum()), float(mk.sum()), cnt_seq]
    assert np.allclose(got, exp, rtol=1e-12, atol=1e-12)


def test_filter_compact_oracle_semantics():
    G = 4
    r = np.array([1, 1, 1, 1, 0, 1, 0, 0, 0.5, 0.5, 0.5, 0.5, 2, 2, 2, 3], dtype=np.float32)
    lens = np.arange(1, 17, dtype=np.int64)
    out = O.filter_compact(r, lens, G)
    assert out["keep_groups"].tolist() == [0, 1, 0, 1]
    assert out["index_map"].tolist() == [4, 5, 6, 7, 12, 13, 14, 15]
    kept = lens[out["index_map"]]
    assert out["new_cu"].tolist() == [0] + np.cumsum(kept).tolist()
    assert out["counts"].tolist() == [8, int(kept.sum()), 2]
    # -0.0 and 0.0 differ bitwise: a group mixing them is kept (bitwise rule)
    r2 = np.array([0.0, -0.0, 0.0, 0.0], dtype=np.float32)
    assert O.filter_compact(r2, lens[:4], 4)["keep_groups"].tolist() == [1]


def test_token_stats_oracle_pinned_to_reference_softmax():
    """The oracle's A1 quantities against the reference's OWN fp64 softmax
    (yatt::distattn::reference_attention, distattn.cpp:79-123, run here by
    oracle/softmax_pin.cpp; tests/golden/softmax_pin.json from
    oracle/softmax_golden.py): one attention head per token row whose scores
    are the logits gives E_p[x], p_y and E_p[z], hence logp = ln p_y,
    lse = x_y - logp, H = lse - E_p[x] and the full KL; keyed rows (V = 2,048
    and odd 1,000) plus edge rows (uniform, one dominant logit, target 60
    nats below the rest, ties, large offsets)."""
    import json
    from pathlib import Path

    from oracle.softmax_golden import inputs, to_f64
    g = json.loads((Path(__file__).parent / "golden" / "softmax_pin.json").read_text())
    checked = 0
    for case in g["cases"]:
        pol, ref, tgt = inputs(case)
        assert tgt.tolist() == case["targets"]
        x, z = to_f64(pol), to_f64(ref)
        r = np.arange(len(tgt))
        P = np.array([o["pol"] for o in case["rows_out"]])
        Q = np.array([o["ref"] for o in case["rows_out"]])
        assert np.allclose(P[:, 3], 1.0, rtol=0, atol=1e-14)
        logp, rlogp = np.log(P[:, 1]), np.log(Q[:, 1])
        lse_p, lse_q = x[r, tgt] - logp, z[r, tgt] - rlogp
        ent = lse_p - P[:, 0]
        d = rlogp - logp
        want = {"k1": -d, "k2": 0.5 * d * d, "k3": np.expm1(d) - d,
                "full": P[:, 0] - lse_p - P[:, 2] + lse_q}
        for mode, kl in want.items():
            got = O.token_stats(pol, ref, tgt, None, mode, threads=2)
            for a, b in zip(got, (logp, rlogp, ent, kl)):
                assert np.all(np.abs(a - b) <= 1e-12 * np.maximum(np.abs(a), np.abs(b)) + 1e-12), \
                    (case["name"], mode, a, b)
            checked += 1
    assert checked == 12


def test_lmhead_oracle_pinned_to_reference_softmax():
    """The LM-head tests' fp64 oracle (numpy GEMM of the bf16 operands + two-
    pass softmax, tests/test_gpu_lmhead.py::_oracle) against the reference's
    attention softmax with the hidden row as the query and the vocabulary
    rows as keys (tests/golden/softmax_pin.json "lmhead_cases")."""
    import json
    from pathlib import Path

    from oracle.softmax_golden import lmhead_inputs, to_f64
    g = json.loads((Path(__file__).parent / "golden" / "softmax_pin.json").read_text())
    assert len(g["lmhead_cases"]) == 2
    for case in g["lmhead_cases"]:
        hb, wb, y = lmhead_inputs(case)
        assert y.tolist() == case["targets"]
        h, w = to_f64(hb), to_f64(wb)
        logits = h @ w.T
        mx = logits.max(1, keepdims=True)
        lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(1))
        lp = logits - lse[:, None]
        r = np.arange(len(y))
        py = np.array([o["p_y"] for o in case["rows_out"]])
        ew = np.array([o["E_p_W"] for o in case["rows_out"]])
        want_lp = np.log(py)
        want_lse = logits[r, y] - want_lp
        want_ent = want_lse - (h * ew).sum(1)
        assert np.allclose(lp[r, y], want_lp, rtol=1e-12, atol=1e-12)
        assert np.allclose(lse, want_lse, rtol=1e-12, atol=1e-12)
        assert np.allclose(-(np.exp(lp) * lp).sum(1), want_ent, rtol=1e-11, atol=1e-12)
