#!/usr/bin/env python3
"""Per-kernel timings of the secondary path kernels at BASELINE shapes, as
achieved algorithmic GB/s vs the measured HBM peak.  One JSON line per op.

  A2  grpo_advantages   configs[1]: 2,048 samples, G=8; configs[4]: 16,384, G=16
  A2' broadcast         8,388,608 tokens
  A3  gae               configs[3]: 2,048 packed seqs, len U[1,8192] (~8.4M tok)
  A3' moments + whiten  same tokens
  A4  policy_loss       8,388,608 tokens, token-mean and seq-mean-token-mean
  A5+A6 filter_compact  configs[4]: 16,384 samples (1,024 x 16), T<=16k+64
  A6  gather_varlen     survivors' 17 B/token payload (~135M tokens total)
  R3  shard_round       16,384 samples, 8 controller shards, one launch
  R10 sort_order_desc   16,384 lengths
Timing: CUDA-graph replay between CUDA events (no host overhead), L2 flushed
before each replay (write, then a read that cleans the dirty lines), median
of 20 after 3 warm-ups, inputs resident.
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_07970_b200 import api, ops  # noqa: E402

dev = torch.device("cuda:0")
PEAK = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())[
    "hbm_gbs"] if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6650.0


_FLUSH = _FLUSH_RD = None


def timeit(fn, iters=20, warm=3):
    """Device time of one call: the call is captured once into a CUDA graph
    (so host-side Python/ctypes overhead is not timed) and replayed between
    CUDA events, with L2 flushed before every replay: a 256 MB write, then a
    256 MB read of a second buffer, so the write-back of the dirty lines the
    write leaves happens before the timed region (otherwise the timed kernel
    pays up to 126 MB of write-back).  Ops that cannot be captured (host syncs
    inside) fall back to eager timing."""
    global _FLUSH, _FLUSH_RD
    if _FLUSH is None:
        _FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        _FLUSH_RD = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    run = fn
    try:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        run = g.replay
    except Exception:  # noqa: BLE001 - host sync inside the op: time it eagerly
        torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        _FLUSH.zero_()
        _FLUSH_RD.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def report(name, ms, alg_bytes, units, unit_name, **extra):
    gbs = alg_bytes / (ms / 1e3) / 1e9
    print(json.dumps({"op": name, "ms": round(ms, 5), "algorithmic_bytes": alg_bytes,
                      "achieved_gbs": round(gbs, 1), "frac_of_measured_hbm": round(gbs / PEAK, 3),
                      f"{unit_name}_per_s": units / (ms / 1e3), **extra}), flush=True)


def main():
    seed = 20250814
    # harness calibration: a plain device copy (torch) at the small kernels' sizes
    for mb in (42, 150):
        src = torch.ones(mb << 17, dtype=torch.float32, device=dev)  # mb/2 MB each way
        dst = torch.empty_like(src)
        ms = timeit(lambda: dst.copy_(src))
        report(f"harness: torch copy_ {mb} MB moved", ms, 2 * src.numel() * 4, src.numel(), "floats")
        del src, dst
    # A2
    for n, G in [(2048, 8), (16384, 16)]:
        r = ops.synth_floats(seed, 105, 0, n, "reward", G, device=dev)
        ms = timeit(lambda: ops.grpo_advantages(r, G))
        report(f"grpo_advantages n={n} G={G}", ms, n * 8, n, "samples")
    ntok = 8388608
    adv = torch.randn(2048, device=dev)
    cu = torch.arange(2049, dtype=torch.int64, device=dev) * 4096
    out = torch.empty(ntok, device=dev)
    ms = timeit(lambda: ops.broadcast_to_tokens(adv, cu, ntok, None, out))
    report("broadcast_to_tokens", ms, ntok * 4 + 2048 * 12, ntok, "tokens")
    # A3
    lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 8192, 8192), 2048, seed)
    cu = torch.zeros(2049, dtype=torch.int64, device=dev)
    cu[1:] = torch.cumsum(torch.tensor(lens, device=dev), 0)
    n = int(cu[-1])
    v = ops.synth_floats(seed, 106, 0, n, "value", device=dev)
    rw = ops.synth_floats(seed, 111, 0, n, "kl", device=dev)
    m = torch.ones(n, dtype=torch.uint8, device=dev)
    ms = timeit(lambda: ops.gae(v, rw, cu, m, 1.0, 0.95))
    report("gae (2048 packed seqs)", ms, n * 17, n, "tokens")
    ms = timeit(lambda: ops.gae(v, rw, cu, m, 1.0, 0.95, return_moments=True))
    report("gae + whitening moments fused (one pass)", ms, n * 17, n, "tokens")

    def gae_then_moments():
        a, _ = ops.gae(v, rw, cu, m, 1.0, 0.95)
        ops.masked_moments(a, m)
    ms = timeit(gae_then_moments)
    report("gae then masked_moments (two passes)", ms, n * 22, n, "tokens")
    mom = ops.masked_moments(v, m)
    ms = timeit(lambda: ops.masked_moments(v, m))
    report("masked_moments", ms, n * 5, n, "tokens")
    y = v.clone()
    ms = timeit(lambda: ops.whiten(y, mom, m))
    report("whiten", ms, n * 9, n, "tokens")
    # A4
    n = ntok
    logp = ops.synth_floats(seed, 107, 0, n, "logp", device=dev)
    old = ops.synth_floats(seed, 104, 0, n, "old_delta", base=logp, device=dev)
    a = ops.synth_floats(seed, 108, 0, n, "adv", device=dev)
    kl = ops.synth_floats(seed, 109, 0, n, "kl", device=dev)
    ent = ops.synth_floats(seed, 110, 0, n, "kl", device=dev)
    mk = torch.ones(n, dtype=torch.uint8, device=dev)
    ws = ops.LossWorkspace(dev)
    sums = torch.empty(8, dtype=torch.float64, device=dev)
    cu = torch.arange(2049, dtype=torch.int64, device=dev) * 4096
    for agg in ["token-mean", "seq-mean-token-mean"]:
        cfg = ops.loss_config(agg_mode=agg)
        ms = timeit(lambda: ops.policy_loss(logp, old, a, kl, ent, mk, cu, cfg, ws, sums))
        report(f"policy_loss {agg}", ms, n * 21, n, "tokens")
    # A5+A6
    G, ns = 16, 16384
    lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 16384, 16384), ns, seed)
    d_lens = torch.tensor(lens, dtype=torch.int64, device=dev) + 64
    rew = ops.synth_floats(seed, 105, 0, ns, "reward", G, device=dev)
    res = {}

    def fc():
        res.update(ops.filter_compact(rew, d_lens, G))
    ms = timeit(fc)
    report("filter_compact (plan)", ms, ns * (4 + 8 + 4 + 8) + ns // G, ns, "samples",
           kept_samples=int(res["counts"][0]), kept_tokens=int(res["counts"][1]))
    old_cu = torch.zeros(ns + 1, dtype=torch.int64, device=dev)
    old_cu[1:] = torch.cumsum(d_lens, 0)
    total = int(old_cu[-1])
    kt = int(res["counts"][1])
    srcs = [torch.empty(total, dtype=t, device=dev) for t in
            (torch.int32, torch.float32, torch.float32, torch.float32, torch.uint8)]
    dsts = [torch.empty(kt, dtype=s.dtype, device=dev) for s in srcs]

    def gather_all():
        for s, d in zip(srcs, dsts):
            ops.gather_varlen(s, old_cu, res["index_map"], res["new_cu"], res["counts"][:1], ns, d)
    ms = timeit(gather_all, iters=10)
    report("gather_varlen 17 B/token payload (5 launches)", ms, kt * 17 * 2, kt, "tokens",
           total_tokens=total)
    ms = timeit(lambda: ops.gather_varlen_multi(srcs, old_cu, res["index_map"], res["new_cu"],
                                                res["counts"][:1], ns, dsts), iters=10)
    report("gather_varlen_multi 17 B/token payload (1 launch)", ms, kt * 17 * 2, kt, "tokens",
           total_tokens=total)
    # R3
    P = 8
    batch = api.RolloutBatch(1, [api.RolloutSample(ns + i, 64) for i in range(ns)])
    params = api.RoundParams(api.LengthDistribution(api.UNIFORM, 1, 16384, 16384),
                             api.RejectionConfig(0.3, True, 16), seed, 16, 4)
    shards = [api.make_shard_state(batch, P, r) for r in range(P)]
    ds = api._DeviceShards(shards, params, dev)
    import ctypes as C
    from paper_2508_07970_b200._lib import check, lib
    off = (C.c_int64 * (P + 1))(*ds.off.tolist())
    pristine = ds.d.clone()

    def rnd():  # restore the round-1 state (D2D copy of 393 KB) then one round
        ds.d.copy_(pristine)
        check(lib().yatt_shard_round(ds.d.data_ptr(), off, P, 0, 1, 1, C.byref(params.c()),
                                     ds.d_rep.data_ptr(), ds.d_mbs.data_ptr(), None))
    ms = timeit(rnd)
    report("shard_round (8 shards, one launch)", ms, ns * 24 * 2, ns, "samples")
    # R10
    l32 = torch.tensor(lens, dtype=torch.int32, device=dev)
    ms = timeit(lambda: ops.sort_order_desc(l32))
    report("sort_order_desc n=16384", ms, ns * 8, ns, "samples")
    # §8f #1 backward into the logits: one prompt group at V = 152,064; V = 32,000
    del srcs, dsts
    torch.cuda.empty_cache()
    for rows, V in [(32768, 152064), (65536, 32000)]:
        pol, ref, tgt = ops.synth_logits(seed, 0, rows, V, device=dev)
        lp, rl, en, kl = ops.token_stats(pol, ref, tgt, None, "k3")
        old = ops.synth_floats(seed, 104, 0, rows, "old_delta", base=lp, device=dev)
        a = ops.synth_floats(seed, 108, 0, rows, "adv", device=dev)
        grad = torch.empty_like(pol)
        for mode in ["k3", "full"]:
            kl_m = ops.token_stats(pol, ref, tgt, None, mode)[3]
            ms = timeit(lambda: ops.logits_grad(pol, ref, tgt, lp, rl, old, a, en, kl_m, None, None,
                                                ops.loss_config(entropy_coef=0.001), mode,
                                                float(rows), grad), iters=10)
            per_row = (6 if mode == "full" else 4) * V + 32
            report(f"logits_grad {mode} (coef + backward) {rows} x {V}", ms, rows * per_row, rows,
                   "tokens")
        # training side fused: loss terms + gradient from the policy logits
        # (HBM: 2V read + 2V written per row; the second read is from L2)
        cfg = ops.loss_config(0.2, 0.28, 0.0, 0.001, 0.001, "token-mean")
        ms = timeit(lambda: ops.policy_loss_grad(pol, tgt, old, a, rl, None, cfg, "k3",
                                                 float(rows), grad), iters=10)
        report(f"policy_loss_grad fused (loss terms + grad) {rows} x {V}", ms,
               rows * (4 * V + 28), rows, "tokens")

        def two_kernel():
            s_ = ops.token_stats(pol, ref, tgt, None, "k3")
            ops.logits_grad(pol, ref, tgt, s_[0], rl, old, a, s_[2], s_[3], None, None, cfg,
                            "k3", float(rows), grad)
        ms = timeit(two_kernel, iters=10)
        report(f"token_stats + logits_grad (two-kernel form) {rows} x {V}", ms,
               rows * (8 * V + 60), rows, "tokens")
        # full-vocabulary KL: policy + reference logits in both passes
        # (HBM: 4V read + 2V written per row; the second read from L2)
        ms = timeit(lambda: ops.policy_loss_grad(pol, tgt, old, a, None, None, cfg, "full",
                                                 float(rows), grad, ref_logits=ref), iters=10)
        report(f"policy_loss_grad fused FULL KL {rows} x {V}", ms, rows * (6 * V + 24), rows,
               "tokens")

        def two_kernel_full():
            s_ = ops.token_stats(pol, ref, tgt, None, "full")
            ops.logits_grad(pol, ref, tgt, s_[0], s_[1], old, a, s_[2], s_[3], None, None, cfg,
                            "full", float(rows), grad)
        ms = timeit(two_kernel_full, iters=10)
        report(f"token_stats + logits_grad FULL KL (two-kernel form) {rows} x {V}", ms,
               rows * (10 * V + 60), rows, "tokens")
        del pol, ref, tgt, grad
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
