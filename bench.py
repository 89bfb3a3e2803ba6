#!/usr/bin/env python3
"""Experience-making throughput (logprob + KL + advantage + loss) at V=152k.

Workload (BASELINE.json configs[1], sharded per configs[2]): one step = the
whole GRPO experience batch of 256 prompts x 8 responses, T = 4096 response
tokens each, V = 152,064 (Qwen2.5-7B vocabulary) = 8,388,608 tokens.  Rank r
of N owns prompt groups shard_dataset(256, N, r) (strong scaling: the global
batch is fixed) and, per group (one 32,768-row chunk of bf16 policy +
reference logits resident in HBM):

    A1 token_stats (logp, ref_logp, entropy, k3 KL)        <- dominant kernel
then over all its tokens: A2 GRPO group advantages -> token broadcast ->
A4 clipped-surrogate + KL loss sums, and (N > 1) one NCCL all-reduce of the
8 fp64 loss sums (global token count) — the only cross-rank traffic.

Logits cannot all be resident (2 x 2.55 TB); each rank keeps two distinct
32,768-row chunks (2 x 19.9 GB) resident and streams its groups through them
alternately: every chunk pass reads 19.9 GB from HBM (>> 126 MB L2), so no
L2 flush is needed and none is done.

`--impl reference` times the CPU restatement of the same path (oracle/,
fp64, all host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "experience tokens/sec (logprob+KL+adv+loss) at V=152k; % HBM roofline, 1-8 B200"
PROMPTS, RESPONSES, T, VOCAB = 256, 8, 4096, 152064
CHUNK_ROWS = RESPONSES * T  # one prompt group
SEED = 20250814
FALLBACK_HBM_GBS = 6650.0


def bytes_per_row(vocab: int) -> int:
    # 2 bf16 logit rows + i32 target + u8 mask + 4 fp32 outputs
    return 4 * vocab + 21


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """Per-launch DRAM bytes of token_stats from the committed ncu capture."""
    p = ROOT / "profiles" / "token_stats_ncu.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get("dram_bytes_per_launch"), d.get("rows_per_launch")
        except Exception:
            pass
    return None, None


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, power, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ------------------------------------------------------------- CPU arm ----
_CPU_SAMPLES = {}


def host_cpu() -> dict:
    """nproc + the lscpu-style model / sockets / physical cores of this host
    (the CPU baseline is reported with the box's CPU)."""
    model, phys, cores = None, set(), set()
    try:
        cur = None
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name" and model is None:
                model = v
            elif k == "physical id":
                cur = v
                phys.add(v)
            elif k == "core id":
                cores.add((cur, v))
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model, "sockets": len(phys) or None,
            "physical_cores": len(cores) or None}


def cpu_experience_rate(sample_rows: int | None = None, threads: int | None = None,
                        budget_s: float = 12.0, repeat: bool = True):
    """Oracle (fp64 CPU restatement) of the same per-token path on a bounded
    sample: A1 over `rows` rows of V=152,064 + A2 over their samples + A4."""
    from oracle import oracle as O
    threads = threads or os.cpu_count() or 1
    uniq = 64
    pol_u, ref_u, tgt_u = O.synth_logits(SEED, 0, uniq, VOCAB)

    def prepare(rows):
        if (rows, threads) in _CPU_SAMPLES:
            return _CPU_SAMPLES[(rows, threads)]
        _CPU_SAMPLES.clear()  # one prepared sample at a time (host memory)
        reps = -(-rows // uniq)
        pol = np.ascontiguousarray(np.tile(pol_u, (reps, 1))[:rows])
        ref = np.ascontiguousarray(np.tile(ref_u, (reps, 1))[:rows])
        tgt = np.ascontiguousarray(np.tile(tgt_u, reps)[:rows])
        n_samples = max(1, rows // T) if rows >= T else 1
        rewards = O.synth_floats(SEED, 105, 0, max(n_samples, RESPONSES), "reward", RESPONSES)
        old_delta = O.synth_floats(SEED, 104, 0, rows, "old_delta")

        def once():
            t0 = time.perf_counter()
            st = O.token_stats(pol, ref, tgt, None, "k3", threads=threads)
            adv_s = O.grpo_advantages(rewards, RESPONSES)
            adv_t = np.repeat(adv_s, -(-rows // len(adv_s)))[:rows].astype(np.float32)
            old = (st[0] + old_delta).astype(np.float32)
            O.policy_loss(st[0], old, adv_t, st[3], st[2])
            return time.perf_counter() - t0
        _CPU_SAMPLES[(rows, threads)] = once
        return once

    probe = 128
    dt = prepare(probe)()
    # host memory caps one pass at 16,384 rows (~10 GB of tiled bf16 logits);
    # passes repeat over the same rows until ~budget_s of CPU work is done
    rows = sample_rows or int(min(16384, max(probe, probe * budget_s / max(dt, 1e-6))))
    once = prepare(rows) if rows != probe else None
    passes, total = 0, 0.0
    if once is None:
        passes, total = 1, dt
    while once is not None and (passes == 0 or (repeat and total < 0.8 * budget_s and passes < 32)):
        total += once()
        passes += 1
    return {"value": rows * passes / total, "unit": "tokens/s", "cores": threads, "kind": "port",
            "host": host_cpu(),
            "sample": f"{passes} pass(es) over {rows} rows x V={VOCAB} "
                      f"(A1 fp64 + GRPO adv + loss), {total:.2f} s"}


def _run_json(cmd):
    """One JSON line from a helper binary; an error dict (never an exception)
    if it is missing or fails, so the bench line is always printed."""
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
        return json.loads(res.stdout)
    except Exception as e:  # noqa: BLE001
        return {"error": f"{Path(cmd[0]).name}: {type(e).__name__}: {e}"[:300]}


def _ref_timing():
    exe = Path(__file__).resolve().parent / "oracle" / "_ref" / "ref_timing"
    if not exe.exists():
        return None
    return _run_json([str(exe), "8"])


def integer_path_baseline():
    """the reference's own integer path (compiled from its
    sources into oracle/_ref, `ref_timing`, one host thread per shard) next to
    the same work through the drop-in C++ API on the GPU
    (examples/_build/integer_timing: sim::run_rollout_rounds, every shard in one
    launch per round), on configs[4]'s batch (16,384 samples, 8 controller
    shards, rounds until none pending); the total train units must agree
    bit-exactly.  None when oracle/_ref is absent."""
    exe = Path(__file__).resolve().parent / "oracle" / "_ref" / "ref_timing"
    if not exe.exists():
        return None
    ref = _ref_timing()
    drv = Path(__file__).resolve().parent / "examples" / "_build" / "integer_timing"
    ours = _run_json([str(drv)]) if drv.exists() else None
    units = ours.get("train_units") if ours else None
    rounds = ours.get("rounds") if ours else None
    return {"reference_cpu": ref, "b200": ours, "host": host_cpu(),
            "train_units_bit_exact": (units is not None and units == ref.get("train_units")
                                      and rounds == ref.get("rounds"))}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    vals = []
    for _ in range(args.warmup):
        cpu_experience_rate(sample_rows=256, repeat=False)
    last = None
    for _ in range(args.steps):
        last = cpu_experience_rate(budget_s=args.ref_budget_s)
        vals.append(last["value"])
    v = statistics.median(vals)
    # a full configs[1] step (8.4M tokens) at the sampled rate: each timed
    # "step" here is a bounded sample of it (cpu_baseline.sample)
    full_step_ms = PROMPTS * RESPONSES * T / v * 1e3
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": full_step_ms,
            "ms_per_step_note": "extrapolated: one full configs[1] step at the sampled CPU rate",
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (keyed integer-derived bf16 logits, DESIGN.md)",
            "config": workload_config(args.gpus), "impl": "reference",
            "cpu_baseline": {**last, "value": v},
            "integer_path_reference_cpu": _ref_timing(),
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


def workload_config(n, collective="peer"):
    coll = ("none" if n == 1 else
            "loss reduce + all-reduce fused in one kernel over NVLink peer memory"
            if collective == "peer" else "NCCL all-reduce of the loss sums / token count")
    return {"collective": coll, "workload": "configs[1]/[2]: GRPO Qwen2.5-7B shape, 256 prompts x 8 responses, "
                        "T=4096, V=152064, sharded by prompt group",
            "global_batch": PROMPTS * RESPONSES, "seq_len": T, "vocab": VOCAB,
            "tokens_per_step": PROMPTS * RESPONSES * T, "parallelism": f"dp{n} by prompt group",
            "kl": "k3", "loss": "clipped surrogate eps=0.2 + 0.001 k3, token-mean",
            "l2": "no flush: each chunk pass streams 19.9 GB >> 126 MB L2"}


# ----------------------------------------------------------- GPU arm ------
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2508_07970_b200 import ops
    from paper_2508_07970_b200._lib import lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib()

    # ---- this rank's shard of prompt groups (workload.cpp:183-198 split) ----
    base, rem = divmod(PROMPTS, world)
    g0 = rank * base + min(rank, rem)
    ng = base + (1 if rank < rem else 0)
    n_samples, n_tok = ng * RESPONSES, ng * CHUNK_ROWS

    # ---- resident inputs ----
    bufs = [ops.synth_logits(SEED + k, 0, CHUNK_ROWS, VOCAB, device=dev) for k in range(2)]
    mask = torch.ones((n_tok,), dtype=torch.uint8, device=dev)
    stats = torch.empty((4, n_tok), dtype=torch.float32, device=dev)
    rewards = ops.synth_floats(SEED, 105, g0 * RESPONSES, n_samples, "reward", RESPONSES,
                               device=dev)
    cu = torch.arange(0, n_samples + 1, dtype=torch.int64, device=dev) * T
    tok_adv = torch.empty((n_tok,), dtype=torch.float32, device=dev)
    # old_logp: the rollout policy's log-probs = current logp + keyed jitter
    for g in range(ng):
        pol, ref, tgt = bufs[g % 2]
        sl = slice(g * CHUNK_ROWS, (g + 1) * CHUNK_ROWS)
        ops.token_stats(pol, ref, tgt, mask[sl], "k3", out=stats[:, sl])
    old_logp = ops.synth_floats(SEED, 104, g0 * CHUNK_ROWS, n_tok, "old_delta", base=stats[0],
                                device=dev)
    cfg = ops.loss_config(0.2, 0.2, 0.0, 0.001, 0.0, "token-mean")
    ws = ops.LossWorkspace(dev)
    sums = torch.empty((8,), dtype=torch.float64, device=dev)
    # N > 1: the loss reduction and its all-reduce are ONE kernel over NVLink
    # peer memory (yatt_policy_loss_allreduce); no NCCL call in the step
    peer = None
    if world > 1 and args.collective == "peer":
        from paper_2508_07970_b200 import ranks
        peer = ranks.PeerGroup(world, rank)
    torch.cuda.synchronize()

    st = torch.cuda.current_stream()
    a1_events: list = []

    def step(record=False):
        for g in range(ng):
            pol, ref, tgt = bufs[g % 2]
            sl = slice(g * CHUNK_ROWS, (g + 1) * CHUNK_ROWS)
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
            ops.token_stats(pol, ref, tgt, mask[sl], "k3", out=stats[:, sl])
            if record:
                e1.record(st)
                a1_events.append((e0, e1))
        adv = ops.grpo_advantages(rewards, RESPONSES, 1e-6, True, g0 * RESPONSES)
        ops.broadcast_to_tokens(adv, cu, n_tok, mask, out=tok_adv)
        if peer is not None:
            peer.policy_loss(stats[0], old_logp, tok_adv, stats[3], stats[2], mask, None, cfg, ws,
                             sums)
        else:
            ops.policy_loss(stats[0], old_logp, tok_adv, stats[3], stats[2], mask, None, cfg, ws,
                            sums)
            if world > 1:
                dist.all_reduce(sums)
        return sums

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(st)
    for _ in range(args.steps):
        step(record=True)
    t1.record(st)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    elapsed_ms = t0.elapsed_time(t1)
    t_local_ms = elapsed_ms
    a1_ms = [a.elapsed_time(b) for a, b in a1_events]
    if world > 1:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    total_tokens = PROMPTS * RESPONSES * T  # all ranks, per step
    value = total_tokens * args.steps / (elapsed_ms / 1e3)
    loss = ops.loss_finalize(sums.cpu(), cfg)

    # ---- roofline of the dominant kernel (A1) ----
    peak, peak_src = hbm_peak()
    a1_avg_ms = statistics.mean(a1_ms)
    alg_bytes = CHUNK_ROWS * bytes_per_row(VOCAB)
    achieved = alg_bytes / (a1_avg_ms / 1e3) / 1e9
    traffic, rows_per = ncu_traffic()
    if traffic is not None and rows_per:  # ncu capture size -> this launch size
        traffic = traffic * CHUNK_ROWS / rows_per
    roofline = {"bound": "hbm", "kernel": "token_stats_kernel", "achieved": achieved,
                "peak": peak, "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                "frac_of_8TBs": achieved / 8000.0, "traffic": traffic,
                "algorithmic_bytes_per_launch": alg_bytes, "launch_ms_avg": a1_avg_ms,
                "share_of_step": sum(a1_ms) / t_local_ms}

    # ---- e2e through the public API: pinned host inputs -> device -> loss ----
    e2e = run_e2e(args, dev, ops, cfg, ws, world)
    hidden = None
    if world == 1 and not args.no_hidden_path:
        try:
            hidden = run_hidden_state_path(dev, ops, cfg, ws)
        except Exception as e:  # noqa: BLE001 - informational; the bench line must print
            hidden = {"error": f"{type(e).__name__}: {e}"[:300]}

    cpu = None
    integer = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_experience_rate(budget_s=args.ref_budget_s)
        except Exception as e:  # noqa: BLE001 - the bench line must still print
            cpu = {"error": f"{type(e).__name__}: {e}"[:300]}
        try:
            integer = integer_path_baseline()
        except Exception as e:  # noqa: BLE001
            integer = {"error": f"{type(e).__name__}: {e}"[:300]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic (keyed integer-derived bf16 logits, "
                "binary group rewards; DESIGN.md)", "config": workload_config(world, args.collective),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "integer_path": integer, "hidden_state_path": hidden,
                # per group: token_stats + its fix-up pass; per step: grpo_adv,
                # broadcast, loss partials + final
                "gpu_launches": args.steps * (2 * ng + 4), "clocks": clk,
                "loss": loss}
        emit(line)
    if world > 1:
        dist.barrier()
        if peer is not None:
            peer.close()
        dist.destroy_process_group()
    return 0


def _mem_available_bytes() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def run_e2e(args, dev, ops, cfg, ws, world=1):
    """Same metric through the reference-facing C-ABI call with HOST buffers
    (yatt_grpo_step_host): each step hands pinned host logits (one configs[1]
    prompt group: 8 responses x 4,096 tokens = 32,768 rows, 2 x 9.97 GB bf16), targets,
    mask, the group's rewards and old log-probs to one call that streams them
    H2D (chunked, overlapped with A1), runs A1 -> GRPO -> A4 and returns the
    loss sums to the host.  Every rank runs it on its own GPU and host link
    between barriers; wall-clock around the blocking calls, max over ranks;
    value = tokens of all ranks / that time."""
    import torch
    import torch.distributed as dist
    def pinned(t):  # device -> pinned host without a pageable staging copy
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h
    # the configs[1] group (32,768 rows); halved while two pinned copies would
    # take more than half the host's available memory split over the local
    # ranks (8 ranks on one box must not drive the host out of memory), and
    # again if pinning itself fails
    local = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    avail = _mem_available_bytes()
    rows = CHUNK_ROWS
    while avail and rows > RESPONSES * 512 and 2 * rows * VOCAB * 2 > 0.5 * avail / local:
        rows //= 2
    while True:
        try:
            h_pol = torch.empty((rows, VOCAB), dtype=torch.bfloat16, pin_memory=True)
            h_ref = torch.empty((rows, VOCAB), dtype=torch.bfloat16, pin_memory=True)
            break
        except RuntimeError as e:
            if rows <= RESPONSES * 512:
                raise
            print(f"e2e: pinning 2 x {rows} rows failed ({e}); halving", file=sys.stderr)
            rows //= 2
    pol, ref, tgt = ops.synth_logits(SEED, 0, rows, VOCAB, device=dev)
    h_pol.copy_(pol)
    h_ref.copy_(ref)
    h_tgt = pinned(tgt)
    h_mask = torch.ones((rows,), dtype=torch.uint8).pin_memory()
    h_rew = pinned(ops.synth_floats(SEED, 105, 0, RESPONSES, "reward", RESPONSES, device=dev))
    logp = ops.token_stats(pol, ref, tgt, None, "k3")[0]
    h_old = pinned(ops.synth_floats(SEED, 104, 0, rows, "old_delta", base=logp, device=dev))
    del pol, ref, tgt, logp
    torch.cuda.synchronize()

    def step():
        return ops.grpo_step_host(h_pol, h_ref, h_tgt, h_rew, h_old, RESPONSES, h_mask,
                                  0, cfg, "k3")

    for _ in range(max(1, args.warmup)):
        step()
    k = max(2, args.steps)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(k):
        step()
    ms = (time.perf_counter() - t0) * 1e3 / k
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    h2d = 2 * rows * VOCAB * 2 + rows * (4 + 1 + 4) + RESPONSES * 4
    # the link's own ceiling: plain pinned H2D copies of the same two tensors
    d_pol = torch.empty(h_pol.shape, dtype=h_pol.dtype, device=dev)
    d_ref = torch.empty_like(d_pol)
    copy_ms = []
    for i in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        d_pol.copy_(h_pol, non_blocking=True)
        d_ref.copy_(h_ref, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        copy_ms.append(a.elapsed_time(b))
    del d_pol, d_ref
    link_gbs = 2 * h_pol.numel() * 2 / (min(copy_ms[1:]) / 1e3) / 1e9
    return {"value": world * rows / (ms / 1e3), "unit": "tokens/s",
            "h2d_bytes_per_step": world * h2d, "d2h_bytes_per_step": world * 64,
            "ms_per_step": ms, "h2d_gbs_per_gpu": h2d / (ms / 1e3) / 1e9,
            "h2d_copy_peak_gbs": link_gbs,
            "frac_of_h2d_copy_peak": h2d / (ms / 1e3) / 1e9 / link_gbs,
            "ranks": world,
            "api": "yatt_grpo_step_host (C ABI, host buffers)",
            "sample": f"per rank: one prompt group of {RESPONSES} x {rows // RESPONSES} tokens per step "
                      f"({h2d / 1e9:.2f} GB H2D from pinned memory)"}


def run_hidden_state_path(dev, ops, cfg, ws, steps=3):
    """The same experience metric from HIDDEN STATES (logits never
    materialised): per step one configs[1] prompt group (32,768 rows) through
    the fused tcgen05 LM head + log-softmax twice (policy and reference
    heads, Qwen2.5-7B shape d=3,584 x V=152,064, random-init bf16 weights),
    the k3 KL from the two log-probs, GRPO advantages and the loss.
    Informational (outside the timed region of the headline): what the path
    costs when the logits are produced on the device instead of read."""
    import torch
    rows, d = CHUNK_ROWS, 3584
    g = torch.Generator(device=dev).manual_seed(SEED)
    h = torch.randn(rows, d, device=dev, generator=g).to(torch.bfloat16)
    hr = (h.float() + 0.05 * torch.randn(rows, d, device=dev, generator=g)).to(torch.bfloat16)
    w = (torch.randn(VOCAB, d, device=dev, generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    wr = (w.float() + 0.01 * torch.randn(VOCAB, d, device=dev, generator=g)).to(torch.bfloat16)
    y = torch.randint(0, VOCAB, (rows,), device=dev, generator=g, dtype=torch.int32)
    rewards = ops.synth_floats(SEED, 105, 0, RESPONSES, "reward", RESPONSES, device=dev)
    cu = torch.arange(0, RESPONSES + 1, dtype=torch.int64, device=dev) * T
    tok_adv = torch.empty((rows,), dtype=torch.float32, device=dev)
    sums = torch.empty((8,), dtype=torch.float64, device=dev)
    out_p = torch.empty((3, rows), dtype=torch.float32, device=dev)
    out_r = torch.empty((3, rows), dtype=torch.float32, device=dev)
    old = None

    def step():
        lp, ent, _ = ops.lmhead_token_stats(h, w, y, out=out_p)
        rl, _, _ = ops.lmhead_token_stats(hr, wr, y, out=out_r)
        kl = ops.kl_from_logps(lp, rl, "k3")
        adv = ops.grpo_advantages(rewards, RESPONSES)
        ops.broadcast_to_tokens(adv, cu, rows, None, out=tok_adv)
        ops.policy_loss(lp, old if old is not None else lp, tok_adv, kl, ent, None, None, cfg,
                        ws, sums)

    step()
    old = out_p[0].clone()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    flops = 2 * 2.0 * rows * d * VOCAB  # two heads
    peak, sustained = 1646.0, 1377.5  # MEASURED_PEAKS.json burst / sustained cuBLAS bf16
    try:
        mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        peak, sustained = float(mp["bf16_tflops"]), float(mp["bf16_tflops_sustained"])
    except Exception:  # noqa: BLE001
        pass
    tf = flops / (ms / 1e3) / 1e12
    return {"value": rows / (ms / 1e3), "unit": "tokens/s", "ms_per_group": ms,
            "sample": f"{steps} x one prompt group ({rows} rows), hidden {d}, V={VOCAB}",
            "roofline": {"bound": "tensor", "kernel": "lmhead_lse_pair_kernel (cta_group::2)",
                         "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                         "peak_sustained": sustained, "frac_of_sustained": tf / sustained,
                         "flops": "GEMM only (2 x 2 rows d V); the step's time includes the "
                                  "split combine, KL, GRPO and loss kernels"}}


_JSON_OUT = None


def emit(line: dict) -> None:
    """The one JSON line on the real stdout (everything else goes to stderr)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # Libraries (NCCL, torch) may print banners on stdout; keep stdout for the
    # single JSON line by pointing fd 1 at stderr for the rest of the run.
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hidden-path", action="store_true",
                    help="skip the informational hidden-state (LM head) measurement")
    ap.add_argument("--ref-budget-s", type=float, default=12.0)
    ap.add_argument("--collective", choices=["peer", "nccl"], default="peer",
                    help="N>1 loss/token-count all-reduce: fused into the loss's final "
                         "reduction over NVLink peer memory (default) or NCCL all-reduce")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
