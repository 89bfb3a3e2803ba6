"""Parallel-controller rank plumbing: sharding by prompt group and the tiny
cross-rank exchanges of the experience step.

The reference runs one controller per rank over a contiguous shard
(workload::shard_dataset, proj/src/workload.cpp:183-198) and reduces the
per-rank integer reports on a coordinator over JSON/TCP RPC
(proj/src/demo.cpp:261-274, simcore.cpp:304-311).  Here every rank owns whole
prompt groups and the only traffic is
  * all-reduce(sum) of the 8 fp64 loss sums (global token / sequence count),
  * all-gather of per-rank survivor counts -> exclusive offsets into one
    global packed layout (dynamic sampling),
  * for shards that split a group (P not dividing the group count): an
    all-gather of the boundary groups' (n, mean, M2) moments, merged with
    Chan et al.'s pairwise update so advantages match a single rank.
Transport: a torch.distributed group (NCCL for device tensors, gloo on CPU)
or the C-ABI NCCL communicator (YattComm).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from ._lib import check, lib


def shard_groups(n_groups: int, world: int, rank: int) -> tuple[int, int]:
    """[g_begin, g_end) of the prompt groups owned by `rank` (the reference's
    near-even split applied to groups, so groups never straddle ranks)."""
    if world <= 0:
        from ._lib import ConfigError
        raise ConfigError("num_controllers must be positive")
    base, rem = divmod(n_groups, world)
    b = rank * base + min(rank, rem)
    return b, b + base + (1 if rank < rem else 0)


def merge_moments(a, b):
    """Chan et al. pairwise merge of (n, mean, M2) triples (fp64)."""
    na, ma, qa = a
    nb, mb, qb = b
    if na == 0:
        return (nb, mb, qb)
    if nb == 0:
        return (na, ma, qa)
    n = na + nb
    d = mb - ma
    return (n, ma + d * nb / n, qa + qb + d * d * na * nb / n)


def merged_boundary_moments(local: torch.Tensor, first_group: int, all_boundaries):
    """Fix up the first/last rows of this rank's (n, mean, M2) table with the
    other ranks' partial moments of the same global groups.

    all_boundaries: list over ranks of (first_group, first_row, last_group,
    last_row) as gathered from every rank (all_gather_object / a tiny
    all-gather of 8 doubles)."""
    table = local.clone()
    parts: dict[int, list] = {}
    for fg, frow, lg, lrow in all_boundaries:
        parts.setdefault(fg, []).append(tuple(frow))
        if lg != fg:
            parts.setdefault(lg, []).append(tuple(lrow))
    for k in (0, table.shape[0] - 1):
        g = first_group + k
        acc = (0.0, 0.0, 0.0)
        for p in parts.get(g, []):
            acc = merge_moments(acc, p)
        if parts.get(g):
            table[k] = torch.tensor(acc, dtype=table.dtype, device=table.device)
    return table


class YattComm:
    """The C-ABI NCCL communicator (yatt_comm_*): device buffers, caller's
    current stream.  The 128-byte unique id travels out of band."""

    def __init__(self, world: int, rank: int, unique_id: bytes):
        self.world, self.rank = world, rank
        self.h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        check(lib().yatt_comm_init(world, rank, C.addressof(buf), C.byref(self.h)))

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().yatt_comm_unique_id(C.addressof(buf)))
        return bytes(buf)

    def _st(self):
        return torch.cuda.current_stream().cuda_stream

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        fn = lib().yatt_comm_allreduce_f64 if t.dtype == torch.float64 else \
            lib().yatt_comm_allreduce_i64
        check(fn(self.h, t.data_ptr(), t.numel(), self._st()))
        return t

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.world * t.numel(),), dtype=t.dtype, device=t.device)
        check(lib().yatt_comm_allgather_i64(self.h, t.data_ptr(), out.data_ptr(), t.numel(),
                                            self._st()))
        return out

    def close(self):
        if self.h:
            check(lib().yatt_comm_destroy(self.h))
            self.h = C.c_void_p()


class PeerGroup:
    """The node's ranks joined through NVLink peer memory (yatt_peer_*): one
    kernel does a reduction AND its cross-rank all-reduce (no NCCL call).
    Handles (64-byte CUDA IPC handles) are exchanged with torch.distributed's
    all_gather_object (gloo or nccl group).  Collective: every rank calls the
    same ops in the same order; results are bit-identical on all ranks."""

    HANDLE = 64

    def __init__(self, world: int | None = None, rank: int | None = None):
        world = dist.get_world_size() if world is None else world
        rank = dist.get_rank() if rank is None else rank
        self.world, self.rank = world, rank
        self.h = C.c_void_p()
        mine = (C.c_uint8 * self.HANDLE)()
        check(lib().yatt_peer_create(world, rank, C.byref(self.h), C.addressof(mine)))
        handles = [None] * world
        if world > 1:
            dist.all_gather_object(handles, bytes(mine))
        else:
            handles = [bytes(mine)]
        allh = (C.c_uint8 * (self.HANDLE * world)).from_buffer_copy(b"".join(handles))
        check(lib().yatt_peer_connect(self.h, C.addressof(allh)))

    def _st(self):
        return torch.cuda.current_stream().cuda_stream

    def allreduce_f64(self, t: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        from .ops import _dev, _numel
        _dev(t, torch.float64, "t")
        out = torch.empty_like(t) if out is None else out
        _dev(out, torch.float64, "out")
        _numel(t.numel(), out=out)
        check(lib().yatt_peer_allreduce_f64(self.h, t.data_ptr(), t.numel(), out.data_ptr(),
                                            self._st()))
        return out

    def scan_i64(self, t: torch.Tensor):
        """(exclusive prefix over lower ranks, total over all ranks) of the
        int64 counters t (<= 16) in one kernel."""
        from .ops import _dev
        _dev(t, torch.int64, "t")
        pre, tot = torch.empty_like(t), torch.empty_like(t)
        check(lib().yatt_peer_scan_i64(self.h, t.data_ptr(), t.numel(), pre.data_ptr(),
                                       tot.data_ptr(), self._st()))
        return pre, tot

    def allgather_i64(self, t: torch.Tensor) -> torch.Tensor:
        """Rank-major all-gather of n <= 16,384 int64 words per rank in one
        kernel over peer memory (world * n words, identical on all ranks)."""
        t = t.contiguous().view(torch.int64)
        out = torch.empty((self.world * t.numel(),), dtype=torch.int64, device=t.device)
        check(lib().yatt_peer_allgather_i64(self.h, t.data_ptr(), t.numel(), out.data_ptr(),
                                            self._st()))
        return out

    def policy_loss(self, logp, old_logp, advantages, kl, entropy, mask=None, cu_seqlens=None,
                    config=None, workspace=None, sums=None):
        """ops.policy_loss whose final reduction is also the all-reduce: the
        GLOBAL yatt_loss_sums on every rank."""
        from . import ops
        ops._devs(torch.float32, logp=logp, old_logp=old_logp, advantages=advantages, kl=kl,
                  entropy=entropy)
        if cu_seqlens is not None:
            ops._dev(cu_seqlens, torch.int64, "cu_seqlens")
        ops._numel(logp.numel(), old_logp=old_logp, advantages=advantages, kl=kl,
                   entropy=entropy, mask=mask)
        cfg = config or ops.loss_config()
        ws = workspace or ops.LossWorkspace(logp.device)
        if sums is None:
            sums = torch.empty((8,), dtype=torch.float64, device=logp.device)
        nseq = 0 if cu_seqlens is None else cu_seqlens.numel() - 1
        p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        m = None if mask is None else mask.view(torch.uint8)
        check(lib().yatt_policy_loss_allreduce(self.h, p(logp), p(old_logp), p(advantages), p(kl),
                                               p(entropy), p(m), logp.numel(), p(cu_seqlens),
                                               nseq, C.byref(cfg), sums.data_ptr(), ws.buf.data_ptr(),
                                               ws.buf.numel(), self._st()))
        return sums

    def _straddle_ws(self, n, first_sample_id, group_size, device):
        wsb = lib().yatt_straddle_workspace_bytes(n, first_sample_id, group_size, self.world)
        return torch.empty((wsb,), dtype=torch.uint8, device=device), wsb

    def grpo_advantages(self, rewards, group_size, first_sample_id=0, eps=1e-6, norm_by_std=True):
        """GRPO advantages of this rank's shard (global ids [first_sample_id,
        + n)) whose first / last groups may straddle ranks: boundary moments
        exchanged over peer memory and merged on the device, one call
        (yatt_peer_grpo_advantages)."""
        from .ops import _dev
        _dev(rewards, torch.float32, "rewards")
        adv = torch.empty_like(rewards)
        ws, wsb = self._straddle_ws(rewards.numel(), first_sample_id, group_size, rewards.device)
        check(lib().yatt_peer_grpo_advantages(self.h, rewards.data_ptr(), rewards.numel(),
                                              first_sample_id, group_size, eps, int(norm_by_std),
                                              adv.data_ptr(), ws.data_ptr(), wsb, self._st()))
        return adv

    def filter_compact(self, rewards, seq_lens, group_size, first_sample_id=0):
        """Zero-variance filter + compaction of this rank's shard with exact
        decisions for straddling groups (yatt_peer_filter_compact)."""
        from .ops import _dev, _numel
        _dev(rewards, torch.float32, "rewards")
        _dev(seq_lens, torch.int64, "seq_lens")
        _numel(rewards.numel(), seq_lens=seq_lens)
        n, dev = rewards.numel(), rewards.device
        ng = lib().yatt_grpo_num_local_groups(n, first_sample_id, group_size)
        keep = torch.empty((max(ng, 1),), dtype=torch.uint8, device=dev)
        imap = torch.empty((max(n, 1),), dtype=torch.int32, device=dev)
        new_cu = torch.empty((n + 1,), dtype=torch.int64, device=dev)
        counts = torch.empty((3,), dtype=torch.int64, device=dev)
        ws, wsb = self._straddle_ws(n, first_sample_id, group_size, dev)
        check(lib().yatt_peer_filter_compact(self.h, rewards.data_ptr(), seq_lens.data_ptr(), n,
                                             first_sample_id, group_size, keep.data_ptr(),
                                             imap.data_ptr(), new_cu.data_ptr(), counts.data_ptr(),
                                             ws.data_ptr(), wsb, self._st()))
        return {"keep_groups": keep[:ng], "index_map": imap, "new_cu": new_cu, "counts": counts}

    def allgather_words(self, words: torch.Tensor) -> torch.Tensor:
        """All-gather of any number of int64 words per rank (sizes may differ
        by rank): one gather of the sizes, then the padded payload in chunks
        of YATT_PEER_GATHER_MAX_WORDS.  Returns [world, max_words] (rows
        zero-padded past each rank's size) and the per-rank sizes."""
        dev = words.device
        n = torch.tensor([words.numel()], dtype=torch.int64, device=dev)
        sizes = self.allgather_i64(n).cpu().tolist()
        width = max(max(sizes), 1)
        buf = torch.zeros((width,), dtype=torch.int64, device=dev)
        buf[: words.numel()] = words
        cap = 16384  # YATT_PEER_GATHER_MAX_WORDS
        cols = [self.allgather_i64(buf[c0:c0 + cap]).view(self.world, -1)
                for c0 in range(0, width, cap)]
        return torch.cat(cols, dim=1), sizes

    def run_rollout_rounds(self, samples, step_index: int, params, device="cuda"):
        """Dynamic-sampling rounds of THIS rank's controller shard (the
        reference's sample-level shard_dataset range, workload.cpp:183-198)
        with ONE cross-rank exchange per step instead of one per round
        (yatt_peer_rounds_run): acceptance never depends on the drawn lengths,
        so each rank runs its shard to completion in one persistent kernel;
        the global loop (simcore.cpp:470-490, the coordinator's continue test
        in demo.cpp:468-476) runs max over ranks of those round counts, a
        finished shard reporting zeros, and the reports + microbatch
        aggregates travel once over peer memory.  Returns the global
        reports[round][rank] (== api.run_rollout_rounds of the whole batch
        over `world` controllers) and updates `samples` like the reference's
        copy_back (simcore.cpp:107-119)."""
        from . import api
        params.out_dist.validate()
        rounds, final = api._run_rounds(samples, "target_out_len_tokens", [0, len(samples)],
                                        self.rank, step_index, 1, 0, params, device, peer=self)
        for x, c in zip(samples, final):
            if c is not None:
                x.target_out_len_tokens, x.accepted, x.accepted_round = c
        return rounds

    def status(self) -> int:
        s = C.c_int32()
        check(lib().yatt_peer_status(self.h, C.byref(s)))
        return s.value

    def close(self):
        if self.h:
            check(lib().yatt_peer_destroy(self.h))
            self.h = C.c_void_p()


REPORT_WORDS = 6  # yatt_round_report = 48 bytes = 6 int64 words (binary wire format)
MB_WORDS = 3      # yatt_mb_agg = 24 bytes


def exchange_round_reports(d_reports: torch.Tensor, d_mbs: torch.Tensor, comm=None,
                           peer: "PeerGroup | None" = None):
    """All-gather this rank's round reports (+ microbatch aggregates, fixed
    per-rank capacity) as raw int64 words and reduce them on the device —
    the binary replacement of the reference's JSON `submit_round` RPC and
    coordinator reduce (demo.cpp:32-76, :261-274; simcore.cpp:304-311).
    With `peer` the two all-gathers are peer-memory kernels over NVLink
    (no NCCL call); otherwise NCCL (comm) / torch.distributed.
    Returns (all_reports_words, all_mb_words, reduction[6]) on the device;
    reduction = {active, pending, forced, train_units, score_tokens, continue}."""
    if peer is not None:
        rep = peer.allgather_i64(d_reports.view(torch.int64))
        mbs = peer.allgather_i64(d_mbs.view(torch.int64))
    else:
        rep = allgather_counts(d_reports.view(torch.int64).contiguous(), comm)
        mbs = allgather_counts(d_mbs.view(torch.int64).contiguous(), comm)
    out = torch.empty((6,), dtype=torch.int64, device=d_reports.device)
    check(lib().yatt_reduce_round_reports(rep.data_ptr(), rep.numel() // REPORT_WORDS,
                                          out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return rep, mbs, out


def allreduce_sums(sums: torch.Tensor, comm=None) -> torch.Tensor:
    """Sum the fp64 loss sums over ranks (in place)."""
    if comm is None:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            dist.all_reduce(sums)
        return sums
    return comm.allreduce_(sums)


def allgather_counts(counts: torch.Tensor, comm=None) -> torch.Tensor:
    """Per-rank int64 count vectors, rank-major (world * counts.numel())."""
    if comm is None:
        import torch.distributed as dist
        if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
            return counts.clone()
        out = [torch.empty_like(counts) for _ in range(dist.get_world_size())]
        dist.all_gather(out, counts)
        return torch.cat(out)
    return comm.allgather(counts)
