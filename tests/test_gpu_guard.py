"""Out-of-bounds write checks for every kernel (compute-sanitizer is closed on
this pool): each output lives inside a larger allocation whose head and tail
are filled with a sentinel byte, offset by one element from the allocation's
alignment, and the test checks that every sentinel byte is intact after the call.
Sizes are chosen off every tile/vector boundary the kernels use."""
import ctypes as C

import pytest
import torch

from paper_2508_07970_b200 import api, ops
from paper_2508_07970_b200._lib import ReportC, SampleC, MbAggC, check, lib

pytestmark = pytest.mark.gpu
SENT = 0xA5
PAD = 4096


class Guarded:
    """`n` elements of `dtype` at byte offset PAD + shift inside a sentinel buffer."""

    def __init__(self, n, dtype, dev, shift=None):
        esz = torch.empty((), dtype=dtype).element_size()
        self.shift = esz if shift is None else shift
        self.nbytes = n * esz
        self.buf = torch.full((self.nbytes + 2 * PAD + 64,), SENT, dtype=torch.uint8, device=dev)
        self.lo = PAD + self.shift
        self.t = self.buf[self.lo: self.lo + self.nbytes].view(dtype) if n else \
            torch.empty((0,), dtype=dtype, device=dev)

    @property
    def p(self):
        return self.buf.data_ptr() + self.lo

    def intact(self):
        head = self.buf[: self.lo]
        tail = self.buf[self.lo + self.nbytes:]
        return bool((head == SENT).all()) and bool((tail == SENT).all())


def _st():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("rows,vocab", [(37, 4096), (3, 8200), (9, 1001), (1, 152064)])
@pytest.mark.parametrize("mode", ["k3", "full"])
def test_token_stats_guard(cuda, rows, vocab, mode):
    if vocab % 8 == 0:
        pol, ref, tgt = ops.synth_logits(3, 0, rows, vocab, device=cuda)
    else:
        g = torch.Generator(device=cuda).manual_seed(1)
        pol = torch.randn(rows, vocab, device=cuda, generator=g).to(torch.bfloat16)
        ref = torch.randn(rows, vocab, device=cuda, generator=g).to(torch.bfloat16)
        tgt = torch.randint(0, vocab, (rows,), device=cuda, dtype=torch.int32, generator=g)
    outs = [Guarded(rows, torch.float32, cuda) for _ in range(4)]
    check(lib().yatt_token_stats(pol.data_ptr(), ref.data_ptr(), tgt.data_ptr(), None, rows, vocab,
                                 ops.KL_MODES[mode], *[o.p for o in outs], _st()))
    torch.cuda.synchronize()
    assert all(o.intact() for o in outs)
    want = ops.token_stats(pol, ref, tgt, None, mode)
    for o, w in zip(outs, want):
        assert torch.equal(o.t, w)


@pytest.mark.parametrize("rows,vocab", [(5, 4096), (3, 8200)])
@pytest.mark.parametrize("mode", ["k3", "full"])
def test_logits_backward_guard(cuda, rows, vocab, mode):
    pol, ref, tgt = ops.synth_logits(4, 0, rows, vocab, device=cuda)
    lp, rl, en, kl = ops.token_stats(pol, ref, tgt, None, "full")
    adv = torch.linspace(-1, 1, rows, device=cuda)
    cu = torch.tensor([0, rows // 2, rows], dtype=torch.int64, device=cuda)
    coef = Guarded(rows * 8, torch.float32, cuda, shift=0)  # coef rows are read as float4
    grad = Guarded(rows * vocab, torch.bfloat16, cuda, shift=0)  # TMA-stored tiles: 16 B aligned
    cfg = ops.loss_config(agg_mode="seq-mean-token-mean")
    check(lib().yatt_policy_grad_coef(pol.data_ptr(), ref.data_ptr(), tgt.data_ptr(), lp.data_ptr(),
                                      rl.data_ptr(), (lp + 0.01).data_ptr(), adv.data_ptr(),
                                      en.data_ptr(), kl.data_ptr(), None, rows, vocab,
                                      cu.data_ptr(), 2, C.byref(cfg), ops.KL_MODES[mode], 2.0,
                                      coef.p, _st()))
    full = int(mode == "full")
    check(lib().yatt_logits_backward(pol.data_ptr(), ref.data_ptr() if full else None,
                                     tgt.data_ptr(), None, rows, vocab, coef.p, full, grad.p,
                                     _st()))
    torch.cuda.synchronize()
    assert coef.intact() and grad.intact()


@pytest.mark.parametrize("n,G,first", [(1, 1, 0), (97, 8, 0), (1029, 16, 5)])
def test_grpo_guard(cuda, n, G, first):
    r = ops.synth_floats(5, 105, 0, n, "reward", G, device=cuda)
    ng = lib().yatt_grpo_num_local_groups(n, first, G)
    mom = Guarded(ng * 3, torch.float64, cuda)
    adv = Guarded(n, torch.float32, cuda)
    check(lib().yatt_grpo_group_moments(r.data_ptr(), n, first, G, mom.p, _st()))
    check(lib().yatt_grpo_advantages(r.data_ptr(), n, first, G, 1e-6, 1, mom.p, adv.p, _st()))
    cu = torch.arange(n + 1, dtype=torch.int64, device=cuda) * 3
    tok = Guarded(3 * n + 1, torch.float32, cuda)
    check(lib().yatt_broadcast_to_tokens(adv.p, cu.data_ptr(), n, None, tok.p, 3 * n + 1, _st()))
    torch.cuda.synchronize()
    assert mom.intact() and adv.intact() and tok.intact()


@pytest.mark.parametrize("lens", [[1], [0, 5, 4097], [300] * 7 + [1, 70001]])
def test_gae_moments_whiten_loss_guard(cuda, lens):
    cu = torch.zeros(len(lens) + 1, dtype=torch.int64, device=cuda)
    cu[1:] = torch.cumsum(torch.tensor(lens, device=cuda), 0)
    n = int(cu[-1])
    v = torch.randn(n, device=cuda)
    m = (torch.rand(n, device=cuda) < 0.7).to(torch.uint8)
    adv, ret = Guarded(n, torch.float32, cuda), Guarded(n, torch.float32, cuda)
    gwb = lib().yatt_gae_workspace_bytes(n)
    gws = Guarded(gwb, torch.uint8, cuda, shift=0)
    check(lib().yatt_gae(v.data_ptr(), (v * 0.3).data_ptr(), m.data_ptr(), cu.data_ptr(),
                         len(lens), n, 1.0, 0.95, adv.p, ret.p, gws.p, gwb, _st()))
    mom = Guarded(3, torch.float64, cuda)
    wsb = lib().yatt_masked_moments_workspace_bytes()
    ws = Guarded(wsb, torch.uint8, cuda, shift=0)
    check(lib().yatt_masked_moments(adv.p, m.data_ptr(), n, mom.p, ws.p, wsb, _st()))
    check(lib().yatt_whiten(adv.p, m.data_ptr(), n, mom.p, 1, _st()))
    for agg in ("token-mean", "seq-mean-token-mean", "seq-mean-token-sum"):
        cfg = ops.loss_config(agg_mode=agg)
        lwb = lib().yatt_policy_loss_workspace_bytes(n, len(lens), cfg.agg_mode)
        lws = Guarded(lwb, torch.uint8, cuda, shift=0)
        sums = Guarded(8, torch.float64, cuda)
        check(lib().yatt_policy_loss(v.data_ptr(), (v + 0.1).data_ptr(), adv.p, v.abs().data_ptr(),
                                     v.abs().data_ptr(), m.data_ptr(), n, cu.data_ptr(), len(lens),
                                     C.byref(cfg), sums.p, lws.p, lwb, _st()))
        torch.cuda.synchronize()
        assert sums.intact() and lws.intact()
    torch.cuda.synchronize()
    assert adv.intact() and ret.intact() and mom.intact() and ws.intact() and gws.intact()


@pytest.mark.parametrize("n,G", [(16, 16), (1000, 8), (5000, 4)])
@pytest.mark.parametrize("esz", [1, 2, 4, 8])  # gather_rows rows are 3*esz bytes
def test_filter_gather_guard(cuda, n, G, esz):
    lens = torch.randint(1, 200, (n,), dtype=torch.int64, device=cuda)
    r = ops.synth_floats(6, 105, 0, n, "reward", G, device=cuda)
    keep, imap = Guarded(n // G, torch.uint8, cuda), Guarded(n, torch.int32, cuda)
    ncu, cnt = Guarded(n + 1, torch.int64, cuda), Guarded(3, torch.int64, cuda)
    wsb = lib().yatt_filter_compact_workspace_bytes(n)
    ws = Guarded(wsb, torch.uint8, cuda, shift=0)
    check(lib().yatt_filter_compact(r.data_ptr(), lens.data_ptr(), n, G, keep.p, imap.p, ncu.p,
                                    cnt.p, ws.p, wsb, _st()))
    torch.cuda.synchronize()
    assert keep.intact() and imap.intact() and ncu.intact() and cnt.intact() and ws.intact()
    ocu = torch.zeros(n + 1, dtype=torch.int64, device=cuda)
    ocu[1:] = torch.cumsum(lens, 0)
    kt, kept = int(cnt.t[1]), int(cnt.t[0])
    src = torch.randint(0, 255, (int(ocu[-1]) * esz,), dtype=torch.uint8, device=cuda)
    dst = Guarded(kt * esz, torch.uint8, cuda, shift=esz)
    check(lib().yatt_gather_varlen(src.data_ptr(), ocu.data_ptr(), imap.p, ncu.p, cnt.p, n, None,
                                   esz, dst.p, _st()))
    rows = Guarded(kept * 3 * esz, torch.uint8, cuda, shift=esz)
    check(lib().yatt_gather_rows(src.data_ptr(), imap.p, cnt.p, n, 3 * esz, None, rows.p, _st()))
    torch.cuda.synchronize()
    assert dst.intact() and rows.intact()
    # payload content: survivors' token ranges concatenated in order
    idx = imap.t[:kept].long().tolist()
    h_ocu = ocu.tolist()
    want = torch.cat([src[h_ocu[i] * esz: h_ocu[i + 1] * esz] for i in idx]) if idx else \
        torch.empty((0,), dtype=torch.uint8, device=cuda)
    assert torch.equal(dst.t, want)


@pytest.mark.parametrize("n", [1, 4095, 4097, 70001])
def test_sort_mb_offset_guard(cuda, n):
    lens = torch.randint(0, 1000, (n,), dtype=torch.int32, device=cuda)
    order = Guarded(n, torch.int32, cuda)
    wsb = lib().yatt_sort_order_workspace_bytes(n)
    ws = Guarded(wsb, torch.uint8, cuda, shift=0)
    check(lib().yatt_sort_order_desc(lens.data_ptr(), n, order.p, ws.p, wsb, _st()))
    mb = 7
    nmb = -(-n // mb)
    agg = Guarded(nmb * 3, torch.int64, cuda)  # yatt_mb_agg holds an int64: 8-byte aligned
    check(lib().yatt_microbatch_aggregates(lens.data_ptr(), lens.data_ptr(), None, n, mb, 0, agg.p,
                                           _st()))
    counts = torch.randint(0, 9, (4 * 3,), dtype=torch.int64, device=cuda)
    off = Guarded(1, torch.int64, cuda)
    check(lib().yatt_exclusive_offset(counts.data_ptr(), 4, 2, 3, 1, off.p, _st()))
    torch.cuda.synchronize()
    assert order.intact() and ws.intact() and agg.intact() and off.intact()
    assert torch.equal(lens[order.t.long()], torch.sort(lens, descending=True, stable=True)[0])


@pytest.mark.parametrize("sizes", [[1], [700], [300, 0, 513]])
def test_shard_round_guard(cuda, sizes):
    n = sum(sizes)
    samples = [api.ShardSampleState(i, 10 + i % 5) for i in range(n)]
    params = api.RoundParams(api.LengthDistribution(api.NORMAL, 300, 80, 1024),
                             api.RejectionConfig(0.4, True, 8), 3, 16, 4)
    packed = torch.from_numpy(api._pack(samples, "out_len_tokens")).to(cuda)
    smp = Guarded(n * C.sizeof(SampleC), torch.uint8, cuda, shift=0)
    smp.t.copy_(packed)
    slots = sum(-(-s // 16) for s in sizes)
    rep = Guarded(len(sizes) * C.sizeof(ReportC), torch.uint8, cuda, shift=0)
    mbs = Guarded(max(slots, 1) * C.sizeof(MbAggC), torch.uint8, cuda, shift=0)
    off = [0]
    for s in sizes:
        off.append(off[-1] + s)
    h_off = (C.c_int64 * len(off))(*off)
    for rnd in range(3):
        check(lib().yatt_shard_round(smp.p, h_off, len(sizes), 0, 0, rnd, C.byref(params.c()),
                                     rep.p, mbs.p, _st()))
    red = Guarded(6, torch.int64, cuda)
    check(lib().yatt_reduce_round_reports(rep.p, len(sizes), red.p, _st()))
    torch.cuda.synchronize()
    assert smp.intact() and rep.intact() and mbs.intact() and red.intact()


@pytest.mark.parametrize("rows,d,vocab,split", [(1, 64, 8, 1), (200, 256, 1000, 3),
                                                (129, 128, 4099, 5)])
def test_lmhead_guard(cuda, rows, d, vocab, split):
    g = torch.Generator(device=cuda).manual_seed(7)
    h = torch.randn(rows, d, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(vocab, d, device=cuda, generator=g) * 0.05).to(torch.bfloat16)
    y = torch.randint(0, vocab, (rows,), device=cuda, dtype=torch.int32, generator=g)
    outs = [Guarded(rows, torch.float32, cuda) for _ in range(3)]
    wsb = lib().yatt_lmhead_workspace_bytes(rows, vocab, split)
    ws = Guarded(max(wsb, 16), torch.uint8, cuda, shift=0)
    check(lib().yatt_lmhead_token_stats(h.data_ptr(), w.data_ptr(), y.data_ptr(), rows, d, vocab,
                                        split, *[o.p for o in outs], ws.p, wsb, _st()))
    kl = Guarded(rows, torch.float32, cuda)
    check(lib().yatt_kl_from_logps(outs[0].p, outs[0].p, rows, 1, kl.p, _st()))
    torch.cuda.synchronize()
    assert all(o.intact() for o in outs) and ws.intact() and kl.intact()
    logits = h.float() @ w.float().T
    lp = torch.log_softmax(logits.double(), -1).gather(1, y.long()[:, None])[:, 0]
    assert torch.allclose(outs[0].t.double(), lp, atol=2e-3, rtol=1e-4)


def test_synth_guard(cuda):
    rows, vocab = 3, 1000
    pol, ref = (Guarded(rows * vocab, torch.bfloat16, cuda, shift=0) for _ in range(2))
    tgt = Guarded(rows, torch.int32, cuda)
    check(lib().yatt_synth_logits(1, 5, rows, vocab, pol.p, ref.p, tgt.p, _st()))
    f = Guarded(1001, torch.float32, cuda)
    check(lib().yatt_synth_floats(1, 105, 3, 1001, ops.SYNTH["reward"], 8, None, f.p, _st()))
    torch.cuda.synchronize()
    assert pol.intact() and ref.intact() and tgt.intact() and f.intact()


@pytest.mark.parametrize("vocab", [4096, 1001])
def test_invalid_targets_are_loud_and_in_bounds(cuda, vocab):
    """Targets outside [0, V) are a caller error: those rows get NaN log-probs
    / KL (and a NaN gradient row), entropy stays valid, every other row is
    unchanged, and nothing outside the outputs is touched."""
    rows = 8
    g = torch.Generator(device=cuda).manual_seed(11)
    pol = (torch.randn(rows, vocab, device=cuda, generator=g) * 2).to(torch.bfloat16)
    ref = (torch.randn(rows, vocab, device=cuda, generator=g) * 2).to(torch.bfloat16)
    good = torch.randint(0, vocab, (rows,), device=cuda, dtype=torch.int32, generator=g)
    tgt = good.clone()
    bad = [1, 3, 6]
    tgt[1], tgt[3], tgt[6] = -1, vocab, vocab + 5
    lp, rl, ent, kl = ops.token_stats(pol, ref, tgt, None, "k3")
    lp0, rl0, ent0, kl0 = ops.token_stats(pol, ref, good, None, "k3")
    torch.cuda.synchronize()
    ok = [r for r in range(rows) if r not in bad]
    assert torch.isnan(lp[bad]).all() and torch.isnan(rl[bad]).all() and torch.isnan(kl[bad]).all()
    assert torch.equal(ent, ent0)
    assert torch.equal(lp[ok], lp0[ok]) and torch.equal(kl[ok], kl0[ok])
    # the backward: NaN rows for the bad targets, the gradient buffer's
    # neighbours untouched, good rows as with valid targets everywhere
    old = lp0.clone()
    adv = torch.ones(rows, device=cuda)
    gd = Guarded(rows * vocab, torch.bfloat16, cuda, shift=0)
    coef = Guarded(rows * 8, torch.float32, cuda, shift=0)
    cfg = ops.loss_config()
    check(lib().yatt_policy_grad_coef(pol.data_ptr(), ref.data_ptr(), tgt.data_ptr(), lp.data_ptr(),
                                      rl.data_ptr(), old.data_ptr(), adv.data_ptr(), ent.data_ptr(),
                                      kl.data_ptr(), None, rows, vocab, None, 0,
                                      C.byref(cfg), 2, float(rows), coef.p, _st()))
    check(lib().yatt_logits_backward(pol.data_ptr(), None, tgt.data_ptr(), None, rows, vocab,
                                     coef.p, 0, gd.p, _st()))
    torch.cuda.synchronize()
    assert gd.intact() and coef.intact()
    gr = gd.t.view(rows, vocab).float()
    assert torch.isnan(gr[bad]).all(dim=1).all()
    assert torch.isfinite(gr[ok]).all()
    if vocab % 8 == 0:  # the fused op
        gf = Guarded(rows * vocab, torch.bfloat16, cuda, shift=0)
        flp, fent, fkl, _ = ops.policy_loss_grad(pol, tgt, old, adv, rl0, None, None, "k3",
                                                 float(rows), gf.t.view(rows, vocab))
        torch.cuda.synchronize()
        assert gf.intact()
        assert torch.isnan(flp[bad]).all() and torch.isfinite(flp[ok]).all()
        assert torch.isnan(gf.t.view(rows, vocab).float()[bad]).all(dim=1).all()
