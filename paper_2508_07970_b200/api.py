"""Python mirror of the reference's on-path host API (proj/include/yatt/).

Same names, fields and error behaviour as the C++ drop-in (include/yatt/
*.hpp), over the same C ABI: batched work runs on the B200, the scalar keyed
draw and O(1) helpers are host arithmetic like in the reference.

    workload.hpp  -> RolloutSample, RolloutBatch, LengthDistribution, RejectionConfig,
                     sample_length_keyed, sample_lengths, rejection_process, shard_dataset
    simcore.hpp   -> ShardSampleState, ShardState, RoundParams, MicrobatchAggregate,
                     ShardRoundReport, make_shard_state, shard_round_output,
                     reduce_round_reports, run_rollout_rounds
    balancer.hpp  -> BatchingPlan, sort_and_bucket, padding_waste, waste_bound
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import (ConfigError, InvalidDistribution, LengthDist, MbAggC, RejectionCfg, ReportC,
                   RoundParamsC, RoundsIoC, RoundsViewC, SampleC, check, lib)

CONSTANT, UNIFORM, NORMAL, LOGNORMAL = range(4)
PROMPT_LEN_STREAM, OUTPUT_LEN_STREAM, REJECTION_STREAM = 1, 2, 3
_MASK64 = (1 << 64) - 1


# ------------------------------------------------------------- keyed RNG ---
def splitmix64(x: int) -> int:
    """proj/include/yatt/common.hpp:17-22."""
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


def hash_key(parts) -> int:
    """common.hpp:25-31."""
    h = 0x243F6A8885A308D3
    for p in parts:
        h = splitmix64(h ^ splitmix64(p & _MASK64))
    return h


def uniform_from_key(key: int) -> float:
    """common.hpp:35-37."""
    return (splitmix64(key) >> 11) * 2.0 ** -53


# ---------------------------------------------------------------- workload --
@dataclass
class LengthDistribution:
    kind: int = CONSTANT
    p1: float = 1.0
    p2: float = 0.0
    max_len_tokens: int = 1 << 20

    def validate(self) -> None:
        if self.max_len_tokens < 1:
            raise InvalidDistribution("max_len_tokens must be at least 1")
        if self.kind == CONSTANT and self.p1 < 1:
            raise InvalidDistribution("constant length must be at least 1")
        if self.kind == UNIFORM and self.p1 < 1:
            raise InvalidDistribution("uniform low bound must be at least 1")
        if self.kind == UNIFORM and self.p2 < self.p1:
            raise InvalidDistribution("uniform high bound below low bound")
        if self.kind in (NORMAL, LOGNORMAL) and self.p2 < 0:
            raise InvalidDistribution("stddev must be non-negative")

    def c(self) -> LengthDist:
        return LengthDist(self.kind, self.max_len_tokens, self.p1, self.p2)


@dataclass
class RolloutSample:
    sample_id: int = 0
    prompt_len_tokens: int = 0
    target_out_len_tokens: int = 0
    accepted_round: int = 0
    accepted: bool = False


@dataclass
class RolloutBatch:
    step_index: int = 0
    samples: list = field(default_factory=list)


@dataclass
class RejectionConfig:
    reject_rate: float = 0.0
    per_group: bool = False
    group_size: int = 1

    def c(self) -> RejectionCfg:
        return RejectionCfg(self.reject_rate, int(self.per_group), self.group_size)


@dataclass
class ShardRange:
    begin: int = 0
    end: int = 0

    def size(self) -> int:
        return self.end - self.begin


def _clamp(v: float, max_len: int) -> int:
    r = float(np.rint(v))  # nearbyint, round-half-even
    return 1 if r < 1 else (max_len if r > max_len else int(r))


def sample_length_keyed(dist: LengthDistribution, seed, stream, step, round_, sample_id) -> int:
    """workload.cpp:109-132 (host scalar, like the reference)."""
    key = hash_key([seed, stream, step, round_, sample_id])
    if dist.kind == CONSTANT:
        return _clamp(dist.p1, dist.max_len_tokens)
    if dist.kind == UNIFORM:
        llround = lambda x: int(math.copysign(math.floor(abs(x) + 0.5), x))  # noqa: E731
        lo, hi = llround(dist.p1), llround(dist.p2)
        return _clamp(lo + int(uniform_from_key(key) * float(hi - lo + 1)), dist.max_len_tokens)
    u1 = uniform_from_key(key)
    u2 = uniform_from_key(splitmix64(key ^ 0x5BF0A8B1457E1D23))
    z = math.sqrt(-2.0 * math.log1p(-u1)) * math.cos(6.283185307179586476925286766559 * u2)
    v = dist.p1 + dist.p2 * z
    return _clamp(v if dist.kind == NORMAL else math.exp(v), dist.max_len_tokens)


def sample_lengths(dist: LengthDistribution, n: int, seed: int, device="cuda") -> list[int]:
    """Batched keyed draws for ids 0..n-1 (workload.cpp:134-143): device
    draws, uncertified Normal/LogNormal ones redone with glibc (bit-exact by
    construction, keyed_draw.cuh)."""
    if n <= 0:
        return []
    ids = np.arange(n, dtype=np.uint64)
    out = np.empty(n, dtype=np.int32)
    with torch.cuda.device(device):
        check(lib().yatt_sample_lengths_host(C.byref(dist.c()), seed, OUTPUT_LEN_STREAM, 0, 0,
                                             ids.ctypes.data, n, out.ctypes.data))
    return out.tolist()


def _pack(samples, sample_attr_out="target_out_len_tokens") -> np.ndarray:
    arr = (SampleC * max(len(samples), 1))()
    for i, s in enumerate(samples):
        arr[i] = SampleC(s.sample_id, s.prompt_len_tokens, getattr(s, sample_attr_out),
                         s.accepted_round, int(s.accepted))
    return np.frombuffer(arr, dtype=np.uint8)[: len(samples) * C.sizeof(SampleC)].copy()


def rejection_process(batch: RolloutBatch, round_: int, config: RejectionConfig, seed: int,
                      device="cuda") -> list[bool]:
    """workload.cpp:145-167 on the device."""
    n = len(batch.samples)
    d = torch.from_numpy(_pack(batch.samples)).to(device) if n else \
        torch.empty((C.sizeof(SampleC),), dtype=torch.uint8, device=device)
    out = torch.empty((max(n, 1),), dtype=torch.uint8, device=device)
    check(lib().yatt_rejection_flags(d.data_ptr(), n, batch.step_index, round_,
                                     C.byref(config.c()), seed, out.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream))
    return [bool(x) for x in out[:n].cpu().tolist()]


def shard_dataset(total_samples: int, num_controllers: int, controller_rank: int) -> ShardRange:
    """workload.cpp:183-198 (C ABI, host arithmetic)."""
    b, e = C.c_uint64(), C.c_uint64()
    check(lib().yatt_shard_dataset(total_samples, num_controllers, controller_rank, C.byref(b),
                                   C.byref(e)))
    return ShardRange(b.value, e.value)


# ----------------------------------------------------------------- simcore --
@dataclass
class ShardSampleState:
    sample_id: int = 0
    prompt_len_tokens: int = 0
    out_len_tokens: int = 0
    accepted: bool = False
    accepted_round: int = 0


@dataclass
class ShardState:
    controller_rank: int = 0
    step_index: int = 0
    samples: list = field(default_factory=list)


@dataclass
class RoundParams:
    out_dist: LengthDistribution = field(default_factory=LengthDistribution)
    rejection: RejectionConfig = field(default_factory=RejectionConfig)
    seed: int = 0
    microbatch_size: int = 1
    max_rounds: int = 64

    def c(self) -> RoundParamsC:
        return RoundParamsC(self.out_dist.c(), self.rejection.c(), self.seed,
                            self.microbatch_size, self.max_rounds)


@dataclass
class MicrobatchAggregate:
    controller_rank: int = 0
    mb_index: int = 0
    sample_count: int = 0
    max_out_len_tokens: int = 0
    score_tokens: int = 0


@dataclass
class ShardRoundReport:
    controller_rank: int = 0
    round: int = 0
    active_count: int = 0
    newly_accepted_count: int = 0
    forced_accept_count: int = 0
    pending_count: int = 0
    accepted_score_tokens: int = 0
    accepted_train_units: int = 0
    microbatches: list = field(default_factory=list)


def _report(r: ReportC, mbs) -> ShardRoundReport:
    return ShardRoundReport(r.controller_rank, r.round, r.active_count, r.newly_accepted_count,
                            r.forced_accept_count, r.pending_count, r.accepted_score_tokens,
                            r.accepted_train_units,
                            [MicrobatchAggregate(m.controller_rank, m.mb_index, m.sample_count,
                                                 m.max_out_len_tokens, m.score_tokens)
                             for m in mbs[: r.num_microbatches]])


def make_shard_state(batch: RolloutBatch, num_controllers: int, controller_rank: int) -> ShardState:
    """simcore.cpp:246-266."""
    rng = shard_dataset(len(batch.samples), num_controllers, controller_rank)
    return ShardState(controller_rank, batch.step_index,
                      [ShardSampleState(s.sample_id, s.prompt_len_tokens, s.target_out_len_tokens,
                                        s.accepted, s.accepted_round)
                       for s in batch.samples[rng.begin:rng.end]])


class _DeviceShards:
    """Samples of several shards resident on the device; one launch per round."""

    def __init__(self, shards: list, params: RoundParams, device="cuda"):
        if params.microbatch_size <= 0:
            raise ConfigError("microbatch_size must be positive")
        self.shards, self.params = shards, params
        self.off = np.zeros(len(shards) + 1, dtype=np.int64)
        for i, s in enumerate(shards):
            self.off[i + 1] = self.off[i] + len(s.samples)
        flat = [x for s in shards for x in s.samples]
        self.n = len(flat)
        self.d = torch.from_numpy(_pack(flat, "out_len_tokens")).to(device) if self.n else \
            torch.empty((C.sizeof(SampleC),), dtype=torch.uint8, device=device)
        mb = params.microbatch_size
        self.slots = [-(-len(s.samples) // mb) for s in shards]
        self.d_rep = torch.empty((len(shards) * C.sizeof(ReportC),), dtype=torch.uint8,
                                 device=device)
        self.d_mbs = torch.empty((max(sum(self.slots), 1) * C.sizeof(MbAggC),), dtype=torch.uint8,
                                 device=device)

    def round(self, round_: int, first_rank: int) -> list[ShardRoundReport]:
        off = (C.c_int64 * len(self.off))(*self.off.tolist())
        check(lib().yatt_shard_round(self.d.data_ptr(), off, len(self.shards), first_rank,
                                     self.shards[0].step_index if self.shards else 0, round_,
                                     C.byref(self.params.c()), self.d_rep.data_ptr(),
                                     self.d_mbs.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream))
        reps = (ReportC * len(self.shards)).from_buffer_copy(self.d_rep.cpu().numpy().tobytes())
        mbs = (MbAggC * max(sum(self.slots), 1)).from_buffer_copy(self.d_mbs.cpu().numpy().tobytes())
        out, base = [], 0
        for i, r in enumerate(reps):
            out.append(_report(r, mbs[base: base + self.slots[i]]))
            base += self.slots[i]
        return out

    def samples(self):
        raw = self.d[: self.n * C.sizeof(SampleC)].cpu().numpy().tobytes()
        return (SampleC * max(self.n, 1)).from_buffer_copy(raw.ljust(C.sizeof(SampleC), b"\0"))


_ROUNDS: dict = {}


def _run_rounds(samples, out_attr, offsets, first_rank, step, first_round, limit,
                params: RoundParams, device, peer=None):
    """yatt_rounds_run over host samples (one persistent kernel for every
    round of every shard); returns (reports[round][shard], final state per
    sample: (out_len, accepted, accepted_round), None if accepted before).
    With `peer` (ranks.PeerGroup): yatt_peer_rounds_run — `samples` are this
    rank's controller shard, the reports come back for every rank."""
    if params.microbatch_size <= 0:
        raise ConfigError("microbatch_size must be positive")
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    with torch.cuda.device(idx):
        h = _ROUNDS.get(idx)
        if h is None:
            h = C.c_void_p()
            check(lib().yatt_rounds_create(C.byref(h)))
            _ROUNDS[idx] = h
        n, ns = len(samples), len(offsets) - 1
        io = RoundsIoC()
        check(lib().yatt_rounds_stage(h, n, ns, C.byref(io)))
        acc = np.array([bool(x.accepted) for x in samples], dtype=np.uint8)
        if n:
            ids = np.array([x.sample_id for x in samples], dtype=np.uint64)
            prm = np.array([x.prompt_len_tokens for x in samples], dtype=np.int32)
            C.memmove(io.sample_id, ids.ctypes.data, ids.nbytes)
            C.memmove(io.prompt_len, prm.ctypes.data, prm.nbytes)
            C.memmove(io.accepted, acc.ctypes.data, acc.nbytes)
        if peer is None:
            off = (C.c_int64 * len(offsets))(*offsets)
            check(lib().yatt_rounds_run(h, n, off, ns, first_rank, step, first_round, limit,
                                        C.byref(params.c()), 0, None))
        else:
            check(lib().yatt_peer_rounds_run(peer.h, h, n, step, C.byref(params.c()), 0, None))
        v = RoundsViewC()
        check(lib().yatt_rounds_result(h, C.byref(v)))
        ns = v.num_shards
        reps = (ReportC * (v.rounds * ns)).from_buffer_copy(
            C.string_at(v.reports, C.sizeof(ReportC) * v.rounds * ns))
        mbs = (MbAggC * max(v.num_microbatches, 1)).from_buffer_copy(
            C.string_at(v.microbatches, C.sizeof(MbAggC) * v.num_microbatches).ljust(
                C.sizeof(MbAggC), b"\0"))
        out_len = np.frombuffer(C.string_at(io.out_len, 4 * n), dtype=np.int32) if n else []
        out_round = np.frombuffer(C.string_at(io.accepted_round, 4 * n), dtype=np.int32) if n else []
        out_acc = np.frombuffer(C.string_at(io.accepted_out, n), dtype=np.uint8) if n else []
        final = [None if acc[i] else (int(out_len[i]), bool(out_acc[i]), int(out_round[i]))
                 for i in range(n)]  # None: accepted before the call, untouched
    rounds, base = [], 0
    for r in range(v.rounds):
        row = []
        for s_ in range(ns):
            rep = reps[r * ns + s_]
            row.append(_report(rep, mbs[base: base + rep.num_microbatches]))
            base += rep.num_microbatches
        rounds.append(row)
    return rounds, final


def shard_round_output(state: ShardState, round_: int, params: RoundParams,
                       device="cuda") -> ShardRoundReport:
    """simcore.cpp:157-214 on the device; mutates `state` like the reference."""
    rounds, final = _run_rounds(state.samples, "out_len_tokens", [0, len(state.samples)],
                                state.controller_rank, state.step_index, round_, 1, params,
                                device)
    for s, c in zip(state.samples, final):
        if c is not None:
            s.out_len_tokens, s.accepted, s.accepted_round = c
    return rounds[0][0]


def reduce_round_reports(reports) -> dict:
    """Integer part of StepAssembler::feed_round (simcore.cpp:304-311)."""
    return {"active": sum(r.active_count for r in reports),
            "pending": sum(r.pending_count for r in reports),
            "forced_accepts": sum(r.forced_accept_count for r in reports),
            "train_units": sum(r.accepted_train_units for r in reports),
            "score_tokens": sum(r.accepted_score_tokens for r in reports)}


def run_rollout_rounds(batch: RolloutBatch, num_controllers: int, params: RoundParams,
                       device="cuda") -> list[list[ShardRoundReport]]:
    """The round loop of run_rlhf_step (simcore.cpp:470-494): every round of
    every shard in ONE device call (rollout_rounds.cu); copy_back in rank
    order (simcore.cpp:107-119)."""
    params.out_dist.validate()
    if params.max_rounds < 1:
        raise ConfigError("max_rounds must be at least 1")
    n = len(batch.samples)
    offsets = [shard_dataset(n, num_controllers, r).begin for r in range(num_controllers)] + [n]
    rounds, final = _run_rounds(batch.samples, "target_out_len_tokens", offsets, 0,
                                batch.step_index, 1, 0, params, device)
    for s, c in zip(batch.samples, final):
        if c is not None:
            s.target_out_len_tokens, s.accepted, s.accepted_round = c
    return rounds


def run_rollout_rounds_per_launch(batch: RolloutBatch, num_controllers: int,
                                  params: RoundParams, device="cuda"):
    """Same loop through the device-resident per-round entry point
    (yatt_shard_round: the building block of the multi-rank loop, where each
    round's reports are exchanged between ranks before the continue test)."""
    params.out_dist.validate()
    if params.max_rounds < 1:
        raise ConfigError("max_rounds must be at least 1")
    shards = [make_shard_state(batch, num_controllers, r) for r in range(num_controllers)]
    ds = _DeviceShards(shards, params, device)
    rounds, r = [], 1
    while True:
        reps = ds.round(r, 0)
        rounds.append(reps)
        if reduce_round_reports(reps)["pending"] == 0:
            break
        r += 1
    for s, c in zip(batch.samples, ds.samples()):
        s.target_out_len_tokens, s.accepted, s.accepted_round = c.out_len_tokens, \
            bool(c.accepted), c.accepted_round
    return rounds


# ---------------------------------------------------------------- balancer --
@dataclass
class BatchingPlan:
    batch_size: int = 0
    buckets: list = field(default_factory=list)
    shuffle_seed: int = 0


def sort_and_bucket(lengths, batch_size: int, seed: int) -> BatchingPlan:
    """balancer.cpp:16-41: device sort, host std::shuffle (bit-exact)."""
    n = len(lengths)
    if batch_size <= 0:
        raise ConfigError("batch_size must be positive")
    ln = np.ascontiguousarray(lengths, dtype=np.int32)
    nb = -(-n // batch_size)
    flat = np.zeros(max(n, 1), dtype=np.uint32)
    off = np.zeros(nb + 1, dtype=np.int64)
    check(lib().yatt_sort_and_bucket_host(ln.ctypes.data, n, batch_size, seed, flat.ctypes.data,
                                          off.ctypes.data))
    return BatchingPlan(batch_size, [flat[off[b]:off[b + 1]].tolist() for b in range(nb)], seed)


def padding_waste(plan: BatchingPlan, lengths) -> float:
    real = padded = 0.0
    for b in plan.buckets:
        mx = max((lengths[i] for i in b), default=0)
        real += sum(float(lengths[i]) ** 2 for i in b)
        padded += len(b) * float(mx) ** 2
    return 0.0 if padded == 0 else 1.0 - real / padded


def waste_bound(batch_size: int) -> float:
    if batch_size <= 0:
        raise ConfigError("batch_size must be positive")
    k = (batch_size - 1) / batch_size
    return 1.0 - k * k
