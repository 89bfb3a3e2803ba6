"""The C ABI under CUDA graphs and concurrent streams.

* Every hot-path entry point is stream-ordered with caller workspaces and no
  host sync, so a whole experience step (A1 -> GRPO -> broadcast -> A4, plus
  GAE / moments / filter / gather) can be captured into one CUDA graph; the
  replay must reproduce the eager results bit for bit.
* Reentrancy (yatt_cuda.h "Conventions"): the same ops on two streams at once,
  each with its own buffers and workspaces, give the single-stream results —
  including the GAE scan, whose tiles exchange carries through the workspace.
"""
import pytest
import torch

from paper_2508_07970_b200 import ConfigError, api, ops

pytestmark = pytest.mark.gpu


def _inputs(dev, seed=7, rows=4096, V=32000, G=8):
    pol, ref, tgt = ops.synth_logits(seed, 0, rows, V, device=dev)
    n_samples = rows // 512
    rew = ops.synth_floats(seed, 105, 0, n_samples, "reward", G, device=dev)
    cu = torch.arange(n_samples + 1, dtype=torch.int64, device=dev) * 512
    old = ops.synth_floats(seed, 104, 0, rows, "old_delta", device=dev)
    lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 3000, 3000), 64, seed)
    gcu = torch.zeros(65, dtype=torch.int64, device=dev)
    gcu[1:] = torch.cumsum(torch.tensor(lens, device=dev), 0)
    nt = int(gcu[-1])
    v = ops.synth_floats(seed, 106, 0, nt, "value", device=dev)
    r = ops.synth_floats(seed, 111, 0, nt, "kl", device=dev)
    return dict(pol=pol, ref=ref, tgt=tgt, rew=rew, cu=cu, old=old, G=G, gcu=gcu, v=v, r=r,
                d_lens=gcu[1:] - gcu[:-1])


class Step:
    """All outputs and workspaces preallocated, so the step is capturable."""

    def __init__(self, x, dev):
        self.x = x
        rows = x["pol"].shape[0]
        self.stats = torch.empty((4, rows), device=dev)
        self.tadv = torch.empty(rows, device=dev)
        self.ws = ops.LossWorkspace(dev)
        self.sums = torch.empty(8, dtype=torch.float64, device=dev)
        self.adv_out = None

    def __call__(self):
        x = self.x
        ops.token_stats(x["pol"], x["ref"], x["tgt"], None, "k3", out=self.stats)
        adv = ops.grpo_advantages(x["rew"], x["G"])
        ops.broadcast_to_tokens(adv, x["cu"], self.tadv.numel(), None, self.tadv)
        ops.policy_loss(self.stats[0], x["old"], self.tadv, self.stats[3], self.stats[2], None,
                        None, None, self.ws, self.sums)
        gadv, gret = ops.gae(x["v"], x["r"], x["gcu"], None, 0.99, 0.95)
        mom = ops.masked_moments(gadv)
        plan = ops.filter_compact(x["rew"], x["d_lens"][: x["rew"].numel()], x["G"])
        self.outs = [self.stats, self.tadv, self.sums, gadv, gret, mom, plan["index_map"],
                     plan["new_cu"], plan["counts"]]
        return self.outs


def test_experience_step_replays_bit_exact_from_a_cuda_graph(cuda):
    x = _inputs(cuda)
    step = Step(x, cuda)
    eager = [t.clone() for t in step()]
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()  # warm-up on a side stream (torch's capture recipe)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        outs = step()
    for t in outs:
        t.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, outs):
        assert torch.equal(a, b)


def test_two_streams_run_the_path_concurrently(cuda):
    xa, xb = _inputs(cuda, seed=1), _inputs(cuda, seed=2)
    ref_a = [t.clone() for t in Step(xa, cuda)()]
    ref_b = [t.clone() for t in Step(xb, cuda)()]
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    step_a, step_b = Step(xa, cuda), Step(xb, cuda)
    for _ in range(3):
        with torch.cuda.stream(sa):
            oa = step_a()
        with torch.cuda.stream(sb):
            ob = step_b()
    torch.cuda.synchronize()
    for r_, o in zip(ref_a, oa):
        assert torch.equal(r_, o)
    for r_, o in zip(ref_b, ob):
        assert torch.equal(r_, o)


def test_gae_scan_is_run_to_run_bit_deterministic(cuda):
    """Tile records depend only on each tile's own tokens, so the look-back
    composes the same maps in the same order however the warps interleave."""
    lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 40000, 40000), 300, 5)
    cu = torch.zeros(301, dtype=torch.int64, device=cuda)
    cu[1:] = torch.cumsum(torch.tensor(lens, device=cuda), 0)
    n = int(cu[-1])
    v = ops.synth_floats(5, 106, 0, n, "value", device=cuda)
    r = ops.synth_floats(5, 111, 0, n, "kl", device=cuda)
    m = (ops.synth_floats(5, 112, 0, n, "kl", device=cuda) < 0.9).to(torch.uint8)
    a0, r0 = ops.gae(v, r, cu, m, 1.0, 0.95)
    for _ in range(10):
        a, rr = ops.gae(v, r, cu, m, 1.0, 0.95)
        assert torch.equal(a, a0) and torch.equal(rr, r0)


def test_peer_group_single_rank_matches_plain_ops(cuda):
    """yatt_peer_* with world = 1 (the multi-rank runs are tools/mgpu_check.py
    under torchrun): the fused reduce + all-reduce kernel equals
    yatt_policy_loss bit for bit, also when replayed from a CUDA graph."""
    from paper_2508_07970_b200 import ranks
    x = _inputs(cuda)
    step = Step(x, cuda)
    step()
    peer = ranks.PeerGroup(1, 0)
    try:
        args = (step.stats[0], x["old"], step.tadv, step.stats[3], step.stats[2])
        plain = ops.policy_loss(*args)
        fused = peer.policy_loss(*args)
        v = torch.arange(1, 12, dtype=torch.float64, device=cuda)
        torch.cuda.synchronize()
        assert torch.equal(plain, fused)
        assert torch.equal(peer.allreduce_f64(v), v)
        ws = ops.LossWorkspace(cuda)
        out = torch.empty(8, dtype=torch.float64, device=cuda)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            peer.policy_loss(*args, workspace=ws, sums=out)
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            peer.policy_loss(*args, workspace=ws, sums=out)
        for _ in range(3):
            out.zero_()
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, plain)
        # all-gather (round reports / microbatch words): identity at world 1,
        # up to the 16,384-word capacity, also from a CUDA graph
        for n in (1, 8, 3000, 16384):
            w = torch.arange(n, dtype=torch.int64, device=cuda) * 7 - 5
            assert torch.equal(peer.allgather_i64(w), w)
        w = torch.arange(100, dtype=torch.int64, device=cuda)
        gout = torch.empty_like(w)
        g2 = torch.cuda.CUDAGraph()
        from paper_2508_07970_b200._lib import check, lib
        with torch.cuda.graph(g2):
            check(lib().yatt_peer_allgather_i64(peer.h, w.data_ptr(), 100, gout.data_ptr(),
                                                torch.cuda.current_stream().cuda_stream))
        for k in range(3):
            w.add_(k)
            g2.replay()
            torch.cuda.synchronize()
            assert torch.equal(gout, w)
        with pytest.raises(ConfigError):
            peer.allgather_i64(torch.zeros(16385, dtype=torch.int64, device=cuda))
        assert peer.status() == 0
    finally:
        peer.close()


@pytest.mark.parametrize("V", [32000, 65536, 152064])
def test_fused_loss_grad_replays_bit_exact_from_a_cuda_graph(cuda, V):
    """The fused loss + gradient op (each shape the dispatch picks: 2 CTAs/SM
    + lag, 1 CTA/SM + lag, 1 CTA/SM) captured into a CUDA graph: replays
    reproduce the eager outputs bit for bit (no host sync, no allocation)."""
    rows = 3 * 148 + 5
    pol, ref, tgt = ops.synth_logits(3, 0, rows, V, device=cuda)
    lp, rl, _, _ = ops.token_stats(pol, ref, tgt, None, "k3")
    old = ops.synth_floats(3, 104, 0, rows, "old_delta", base=lp, device=cuda)
    adv = ops.synth_floats(3, 108, 0, rows, "adv", device=cuda)
    cfg = ops.loss_config(0.2, 0.28, 0.0, 0.001, 0.001, "token-mean")
    grad = torch.empty_like(pol)

    def run():
        return ops.policy_loss_grad(pol, tgt, old, adv, rl, None, cfg, "k3", float(rows), grad)
    eager = [t.clone() for t in run()]
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        outs = run()
    for t in outs:
        t.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, outs):
        assert torch.equal(a, b)
