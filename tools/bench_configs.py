#!/usr/bin/env python3
"""Measured throughput of the non-headline BASELINE configs (one JSON line each).

  configs[0]  GRPO 16 prompts x 8 responses, T=256, V=32,000: A1 + GRPO + loss
  configs[3]  PPO, 2,048 packed sequences with lengths U[1, 8192] (~8.4M
              tokens), V=152,064: A1 over 32,768-row chunks + GAE + whitening
              (global moments) + loss
  configs[4]  dynamic sampling on 1,024 prompts x 16 responses, T<=16k + 64
              prompt (~135M tokens): dynamic-sampling round (R3), group filter
              + compaction plan (A5/A6), gather of the survivors' 17 B/token
              payload + 4 payload refs per sample (multimodal-shaped), repack
              order (R10) and microbatch aggregates
Timing: CUDA events around the whole pipeline, median of 3 after a warm-up.
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_07970_b200 import api, ops  # noqa: E402

dev = torch.device("cuda:0")
SEED = 20250814


def timeit(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def config1():
    P, R, T, V = 16, 8, 256, 32000
    rows = P * R * T
    pol, ref, tgt = ops.synth_logits(SEED, 0, rows, V, device=dev)
    rew = ops.synth_floats(SEED, 105, 0, P * R, "reward", R, device=dev)
    cu = torch.arange(P * R + 1, dtype=torch.int64, device=dev) * T
    stats = torch.empty((4, rows), device=dev)
    old = ops.synth_floats(SEED, 104, 0, rows, "old_delta", device=dev)
    ws = ops.LossWorkspace(dev)

    def run():
        ops.token_stats(pol, ref, tgt, None, "k3", out=stats)
        tadv = ops.broadcast_to_tokens(ops.grpo_advantages(rew, R), cu, rows)
        ops.policy_loss(stats[0], old, tadv, stats[3], stats[2], None, None, None, ws)
    ms = timeit(run)
    return {"config": "configs[0] GRPO 16x8, T=256, V=32000", "tokens": rows, "ms": ms,
            "tokens_per_s": rows / ms * 1e3,
            "a1_gbs": rows * (4 * V + 21) / ms / 1e6}


def config4():
    V, n_seq, chunk = 152064, 2048, 32768
    lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 8192, 8192), n_seq, SEED)
    cu = torch.zeros(n_seq + 1, dtype=torch.int64, device=dev)
    cu[1:] = torch.cumsum(torch.tensor(lens, device=dev), 0)
    ntok = int(cu[-1])
    bufs = [ops.synth_logits(SEED + k, 0, chunk, V, device=dev) for k in range(2)]
    stats = torch.empty((4, ntok), device=dev)
    values = ops.synth_floats(SEED, 106, 0, ntok, "value", device=dev)
    rewards = (ops.synth_floats(SEED, 111, 0, ntok, "kl", device=dev) * 4 - 0.5).contiguous()
    old = ops.synth_floats(SEED, 104, 0, ntok, "old_delta", device=dev)
    ws = ops.LossWorkspace(dev)
    cfg = ops.loss_config(0.2, 0.2, 3.0, 0.0, 0.0, "token-mean")

    def run():
        for c0 in range(0, ntok, chunk):
            n = min(chunk, ntok - c0)
            pol, ref, tgt = bufs[(c0 // chunk) % 2]
            ops.token_stats(pol[:n], ref[:n], tgt[:n], None, "k3", out=stats[:, c0:c0 + n])
        adv, ret, mom = ops.gae(values, rewards, cu, None, 1.0, 0.95, return_moments=True)
        ops.whiten(adv, mom)  # whitening statistics from the GAE pass itself
        ops.policy_loss(stats[0], old, adv, stats[3], stats[2], None, None, cfg, ws)
    ms = timeit(run, iters=2)
    return {"config": "configs[3] PPO 2048 packed seqs U[1,8192], V=152064, GAE g=1 l=0.95",
            "tokens": ntok, "ms": ms, "tokens_per_s": ntok / ms * 1e3,
            "a1_gbs_effective": ntok * (4 * V + 21) / ms / 1e6}


def config5():
    G, n_prompts = 16, 1024
    n = G * n_prompts
    batch = api.RolloutBatch(1, [api.RolloutSample(n + i, 64) for i in range(n)])
    params = api.RoundParams(api.LengthDistribution(api.UNIFORM, 1, 16384, 16384),
                             api.RejectionConfig(0.3, True, G), SEED, 16, 4)
    ds = api._DeviceShards([api.make_shard_state(batch, 1, 0)], params, dev)
    import ctypes as C
    from paper_2508_07970_b200._lib import check, lib
    off = (C.c_int64 * 2)(0, n)
    pristine = ds.d.clone()
    lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 16384, 16384), n, SEED)
    d_lens = torch.tensor(lens, dtype=torch.int64, device=dev) + 64
    rew = ops.synth_floats(SEED, 105, 0, n, "reward", G, device=dev)
    old_cu = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    old_cu[1:] = torch.cumsum(d_lens, 0)
    total = int(old_cu[-1])
    payload = [torch.empty(total, dtype=t, device=dev) for t in
               (torch.int32, torch.float32, torch.float32, torch.float32, torch.uint8)]
    refs = torch.arange(n * 4, dtype=torch.int64, device=dev).view(n, 4)
    plan = ops.filter_compact(rew, d_lens, G)
    kt = int(plan["counts"][1])
    kept = int(plan["counts"][0])
    outs = [torch.empty(kt, dtype=p.dtype, device=dev) for p in payload]
    rout = torch.empty((n, 4), dtype=torch.int64, device=dev)
    l32 = (d_lens - 64).to(torch.int32)
    p32 = torch.full((n,), 64, dtype=torch.int32, device=dev)

    def run():
        ds.d.copy_(pristine)
        check(lib().yatt_shard_round(ds.d.data_ptr(), off, 1, 0, 1, 1, C.byref(params.c()),
                                     ds.d_rep.data_ptr(), ds.d_mbs.data_ptr(), None))
        pl = ops.filter_compact(rew, d_lens, G)
        ops.gather_varlen_multi(payload, old_cu, pl["index_map"], pl["new_cu"], pl["counts"][:1], n,
                                outs)
        ops.gather_rows(refs, pl["index_map"], pl["counts"][:1], n, rout)
        ops.sort_order_desc(l32)
        ops.microbatch_aggregates(p32, l32, 16)
    ms = timeit(run)
    moved = kt * 17 * 2 + kept * 32 * 2
    return {"config": "configs[4] dynamic sampling 1024x16, T<=16k+64, multimodal refs",
            "samples": n, "tokens": total, "kept_samples": kept, "kept_tokens": kt, "ms": ms,
            "samples_per_s": n / ms * 1e3, "tokens_per_s": total / ms * 1e3,
            "payload_gbs": moved / ms / 1e6}


if __name__ == "__main__":
    for fn in (config1, config4, config5):
        print(json.dumps(fn()), flush=True)
