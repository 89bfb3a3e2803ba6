"""Device ops over torch tensors, each one C-ABI call into libyatt_b200.so.

torch is only plumbing here (device memory, the current stream); the compute
is the sm_100a kernels behind include/yatt_cuda.h.  Every op runs on the
caller's current CUDA stream and does not synchronise unless it returns host
data.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import (ConfigError, LossConfigC, LossSumsC, check, lib)


class _Modes(dict):
    """Name -> ABI enum; unknown names raise ConfigError like the C ABI."""

    def __missing__(self, key):
        raise ConfigError(f"unknown mode {key!r} (expected one of {sorted(self)})")


KL_MODES = _Modes({"k1": 0, "k2": 1, "k3": 2, "low_var_kl": 2, "full": 3})
SYNTH = _Modes({"logp": 0, "old_delta": 1, "adv": 2, "kl": 3, "value": 4, "reward": 5})
AGG_MODES = _Modes({"token-mean": 0, "seq-mean-token-mean": 1, "seq-mean-token-sum": 2})


def _p(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _st() -> int:
    return torch.cuda.current_stream().cuda_stream


def _dev(t: torch.Tensor, dtype: torch.dtype, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _devs(dtype: torch.dtype, **named) -> None:
    """_dev for several (optional) tensors of one dtype."""
    for name, t in named.items():
        if t is not None:
            _dev(t, dtype, name)


def _dense(**named) -> None:
    """CUDA + contiguous, any dtype (byte-level gathers)."""
    for name, t in named.items():
        if t is not None:
            _dev(t, t.dtype, name)


def _numel(n: int, **named) -> None:
    """Per-token / per-sample arrays must hold exactly n elements (the
    kernels read n of each: a shorter tensor would be read out of bounds)."""
    for name, t in named.items():
        if t is not None and t.numel() != n:
            raise ValueError(f"{name} has {t.numel()} elements, expected {n}")


def _mask(mask: torch.Tensor | None) -> torch.Tensor | None:
    if mask is None:
        return None
    if mask.dtype == torch.bool:
        mask = mask.to(torch.uint8)
    return _dev(mask, torch.uint8, "mask")


# ------------------------------------------------------------------ A1 ----
def token_stats(policy_logits: torch.Tensor, ref_logits: torch.Tensor, targets: torch.Tensor,
                mask: torch.Tensor | None = None, kl_mode: str = "k3", out=None):
    """Fused per-token (logp, ref_logp, entropy, kl) over [rows, V] bf16 logits."""
    _dev(policy_logits, torch.bfloat16, "policy_logits")
    _dev(ref_logits, torch.bfloat16, "ref_logits")
    _dev(targets, torch.int32, "targets")
    rows, vocab = policy_logits.shape
    if ref_logits.shape != policy_logits.shape or targets.shape != (rows,):
        raise ValueError("shape mismatch between logits / targets")
    m = _mask(mask)
    _numel(rows, mask=m)
    if out is None:
        out = torch.empty((4, rows), dtype=torch.float32, device=policy_logits.device)
    elif out.shape != (4, rows):
        raise ValueError(f"out must be [4, {rows}], got {list(out.shape)}")
    # the four outputs are written as four dense rows: a column slice of a
    # wider [4, N] buffer is fine (bench.py shards one), a strided row is not
    if not out.is_cuda or out.dtype != torch.float32 or (rows > 1 and out.stride(1) != 1):
        raise ValueError("out must be a CUDA float32 [4, rows] tensor with dense rows")
    check(lib().yatt_token_stats(_p(policy_logits), _p(ref_logits), _p(targets), _p(m), rows,
                                 vocab, KL_MODES[kl_mode], _p(out[0]), _p(out[1]), _p(out[2]),
                                 _p(out[3]), _st()))
    return out[0], out[1], out[2], out[3]


def _host(a, dtype, name: str, shape: tuple | None = None, optional: bool = False):
    """Validate a HOST buffer handed to a *_host C-ABI entry (numpy array or
    CPU torch tensor): dtype, exact shape, C-contiguity.  The library trusts
    the sizes it is given, so a wrong dtype or shape here would be read or
    written out of bounds."""
    if a is None:
        if optional:
            return None
        raise ValueError(f"{name} is required")
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            raise ValueError(f"{name} must be a host (CPU) buffer")
        if a.dtype != dtype[1]:
            raise TypeError(f"{name} must be {dtype[1]}, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        got, ptr = tuple(a.shape), a.data_ptr()
    else:
        a = np.asarray(a) if not isinstance(a, np.ndarray) else a
        if a.dtype != np.dtype(dtype[0]):
            raise TypeError(f"{name} must be {np.dtype(dtype[0])}, got {a.dtype}")
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name} must be C-contiguous")
        got, ptr = tuple(a.shape), a.ctypes.data
    if shape is not None and got != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {got}")
    return ptr


_U16 = (np.uint16, torch.int16)   # bf16 bit patterns (torch: int16 / bfloat16 views)
_I32 = (np.int32, torch.int32)
_U8 = (np.uint8, torch.uint8)
_F32 = (np.float32, torch.float32)


def _logits_shape(policy) -> tuple[int, int]:
    if len(policy.shape) != 2:
        raise ValueError(f"logits must be 2-D [rows, vocab], got shape {tuple(policy.shape)}")
    return int(policy.shape[0]), int(policy.shape[1])


def _as_u16(a):
    return a.view(torch.int16) if isinstance(a, torch.Tensor) and a.dtype == torch.bfloat16 else a


def token_stats_host(policy: np.ndarray, ref: np.ndarray, targets: np.ndarray,
                     mask: np.ndarray | None = None, kl_mode: str = "k3", out: np.ndarray | None = None):
    """Same op on HOST buffers (uint16 bf16 bits): H2D, kernel, D2H inside."""
    policy, ref = _as_u16(policy), _as_u16(ref)
    rows, vocab = _logits_shape(policy)
    if out is None:
        out = np.empty((4, rows), dtype=np.float32)
    pp = _host(policy, _U16, "policy", (rows, vocab))
    pr = _host(ref, _U16, "ref", (rows, vocab))
    pt = _host(targets, _I32, "targets", (rows,))
    mp = _host(mask, _U8, "mask", (rows,), optional=True)
    _host(out, _F32, "out", (4, rows))
    check(lib().yatt_token_stats_host(pp, pr, pt, mp, rows, vocab, KL_MODES[kl_mode],
                                      out[0].ctypes.data, out[1].ctypes.data, out[2].ctypes.data,
                                      out[3].ctypes.data))
    return out


def grpo_step_host(policy, ref, targets, rewards, old_logp, group_size: int, mask=None,
                   first_sample_id: int = 0, config: LossConfigC | None = None,
                   kl_mode: str = "k3", stats_out=None):
    """One GRPO experience step through the C ABI from HOST buffers (numpy or
    CPU torch tensors, pinned for full PCIe speed): returns the 8 loss sums."""
    policy, ref = _as_u16(policy), _as_u16(ref)
    rows, vocab = _logits_shape(policy)
    n = int(rewards.shape[0]) if len(rewards.shape) == 1 else -1
    if n <= 0 or rows % n != 0:
        raise ValueError(f"rewards must be 1-D with rows ({rows}) a multiple of its length")
    args = (_host(policy, _U16, "policy", (rows, vocab)), _host(ref, _U16, "ref", (rows, vocab)),
            _host(targets, _I32, "targets", (rows,)), _host(mask, _U8, "mask", (rows,), True))
    pr = _host(rewards, _F32, "rewards", (n,))
    po = _host(old_logp, _F32, "old_logp", (rows,))
    ps = _host(stats_out, _F32, "stats_out", (4, rows), optional=True)
    sums = LossSumsC()
    check(lib().yatt_grpo_step_host(*args, rows, vocab, pr, n, first_sample_id, group_size, po,
                                    C.byref(config or loss_config()), KL_MODES[kl_mode],
                                    C.byref(sums), ps))
    return [getattr(sums, f) for f, _ in LossSumsC._fields_]


# ------------------------------------------------------------ synthetic ----
def synth_logits(seed: int, row0: int, rows: int, vocab: int, device="cuda", out=None):
    if out is None:
        pol = torch.empty((rows, vocab), dtype=torch.bfloat16, device=device)
        ref = torch.empty_like(pol)
        tgt = torch.empty((rows,), dtype=torch.int32, device=device)
    else:
        pol, ref, tgt = out
    check(lib().yatt_synth_logits(seed, row0, rows, vocab, _p(pol), _p(ref), _p(tgt), _st()))
    return pol, ref, tgt


def synth_floats(seed: int, stream_id: int, i0: int, n: int, kind: str, group_size: int = 1,
                 base: torch.Tensor | None = None, device="cuda") -> torch.Tensor:
    out = torch.empty((n,), dtype=torch.float32, device=device)
    check(lib().yatt_synth_floats(seed, stream_id, i0, n, SYNTH[kind], group_size, _p(base),
                                  _p(out), _st()))
    return out


# ------------------------------------------------------------------ A2 ----
def grpo_group_moments(rewards: torch.Tensor, group_size: int, first_sample_id: int = 0):
    _dev(rewards, torch.float32, "rewards")
    n = rewards.numel()
    ng = lib().yatt_grpo_num_local_groups(n, first_sample_id, group_size)
    out = torch.empty((max(ng, 0), 3), dtype=torch.float64, device=rewards.device)
    check(lib().yatt_grpo_group_moments(_p(rewards), n, first_sample_id, group_size, _p(out),
                                        _st()))
    return out


def grpo_advantages(rewards: torch.Tensor, group_size: int, eps: float = 1e-6,
                    norm_by_std: bool = True, first_sample_id: int = 0,
                    moments: torch.Tensor | None = None) -> torch.Tensor:
    _dev(rewards, torch.float32, "rewards")
    adv = torch.empty_like(rewards)
    check(lib().yatt_grpo_advantages(_p(rewards), rewards.numel(), first_sample_id, group_size,
                                     eps, int(norm_by_std), _p(moments), _p(adv), _st()))
    return adv


def broadcast_to_tokens(sample_vals: torch.Tensor, cu_seqlens: torch.Tensor, n_tokens: int,
                        mask: torch.Tensor | None = None, out: torch.Tensor | None = None):
    _dev(cu_seqlens, torch.int64, "cu_seqlens")
    _devs(torch.float32, sample_vals=sample_vals, out=out)
    if out is None:
        out = torch.empty((n_tokens,), dtype=torch.float32, device=sample_vals.device)
    _numel(n_tokens, out=out, mask=mask)
    if cu_seqlens.numel() < sample_vals.numel() + 1:
        raise ValueError("cu_seqlens needs n_samples + 1 entries")
    check(lib().yatt_broadcast_to_tokens(_p(sample_vals), _p(cu_seqlens), sample_vals.numel(),
                                         _p(_mask(mask)), _p(out), n_tokens, _st()))
    return out


# ------------------------------------------------------------------ A3 ----
def gae(values: torch.Tensor, rewards: torch.Tensor, cu_seqlens: torch.Tensor,
        mask: torch.Tensor | None = None, gamma: float = 1.0, lam: float = 0.95,
        return_moments: bool = False):
    """(advantages, returns) — and with return_moments the masked moments
    {count, sum, sum_sq} (fp64) of the advantages, from the same pass."""
    _dev(values, torch.float32, "values")
    _dev(rewards, torch.float32, "rewards")
    _dev(cu_seqlens, torch.int64, "cu_seqlens")
    n = values.numel()
    _numel(n, rewards=rewards, mask=mask)
    adv = torch.empty_like(values)
    ret = torch.empty_like(values)
    wsb = lib().yatt_gae_workspace_bytes(n)
    ws = torch.empty((max(wsb, 16),), dtype=torch.uint8, device=values.device)
    if return_moments:
        mom = torch.empty((3,), dtype=torch.float64, device=values.device)
        check(lib().yatt_gae_with_moments(_p(values), _p(rewards), _p(_mask(mask)),
                                          _p(cu_seqlens), cu_seqlens.numel() - 1, n, gamma, lam,
                                          _p(adv), _p(ret), _p(mom), _p(ws), wsb, _st()))
        return adv, ret, mom
    check(lib().yatt_gae(_p(values), _p(rewards), _p(_mask(mask)), _p(cu_seqlens),
                         cu_seqlens.numel() - 1, n, gamma, lam, _p(adv), _p(ret), _p(ws), wsb,
                         _st()))
    return adv, ret


def masked_moments(x: torch.Tensor, mask: torch.Tensor | None = None) -> torch.Tensor:
    _dev(x, torch.float32, "x")
    _numel(x.numel(), mask=mask)
    out = torch.empty((3,), dtype=torch.float64, device=x.device)
    wsb = lib().yatt_masked_moments_workspace_bytes()
    ws = torch.empty((wsb,), dtype=torch.uint8, device=x.device)
    check(lib().yatt_masked_moments(_p(x), _p(_mask(mask)), x.numel(), _p(out), _p(ws), wsb, _st()))
    return out


def whiten(x: torch.Tensor, moments: torch.Tensor, mask: torch.Tensor | None = None,
           shift_mean: bool = True) -> torch.Tensor:
    _dev(x, torch.float32, "x")
    _dev(moments, torch.float64, "moments")
    _numel(x.numel(), mask=mask)
    _numel(3, moments=moments)
    check(lib().yatt_whiten(_p(x), _p(_mask(mask)), x.numel(), _p(moments), int(shift_mean), _st()))
    return x


# ------------------------------------------------------------------ A4 ----
def loss_config(clip_low=0.2, clip_high=0.2, clip_ratio_c=0.0, kl_coef=0.001, entropy_coef=0.0,
                agg_mode="token-mean") -> LossConfigC:
    return LossConfigC(clip_low, clip_high, clip_ratio_c, kl_coef, entropy_coef,
                       AGG_MODES[agg_mode] if isinstance(agg_mode, str) else int(agg_mode))


class LossWorkspace:
    def __init__(self, device="cuda"):
        nb = lib().yatt_policy_loss_workspace_bytes(0, 0, 0)
        self.buf = torch.empty((nb,), dtype=torch.uint8, device=device)


def policy_loss(logp, old_logp, advantages, kl, entropy, mask=None, cu_seqlens=None,
                config: LossConfigC | None = None, workspace: LossWorkspace | None = None,
                sums: torch.Tensor | None = None) -> torch.Tensor:
    """Returns the 8 fp64 yatt_loss_sums fields as a device tensor."""
    _devs(torch.float32, logp=logp, old_logp=old_logp, advantages=advantages, kl=kl,
          entropy=entropy)
    if cu_seqlens is not None:
        _dev(cu_seqlens, torch.int64, "cu_seqlens")
    _numel(logp.numel(), old_logp=old_logp, advantages=advantages, kl=kl, entropy=entropy,
           mask=mask)
    cfg = config or loss_config()
    ws = workspace or LossWorkspace(logp.device)
    if sums is None:
        sums = torch.empty((8,), dtype=torch.float64, device=logp.device)
    nseq = 0 if cu_seqlens is None else cu_seqlens.numel() - 1
    check(lib().yatt_policy_loss(_p(logp), _p(old_logp), _p(advantages), _p(kl), _p(entropy),
                                 _p(_mask(mask)), logp.numel(), _p(cu_seqlens), nseq,
                                 C.byref(cfg), _p(sums), _p(ws.buf), ws.buf.numel(), _st()))
    return sums


def loss_finalize(sums, config: LossConfigC | None = None) -> float:
    s = LossSumsC(*[float(v) for v in (sums.tolist() if hasattr(sums, "tolist") else sums)])
    return lib().yatt_loss_finalize(C.byref(s), C.byref(config or loss_config()))


# ------------------------------------------------------------- A5 / A6 ----
def filter_compact(rewards: torch.Tensor, seq_lens: torch.Tensor, group_size: int,
                   first_sample_id: int = 0, all_records: torch.Tensor | None = None,
                   world: int = 1):
    """A5+A6.  first_sample_id / all_records: a shard of a sample-level split
    whose boundary groups straddle ranks (yatt_filter_compact_sharded; the
    records are every rank's filter_boundary_record, gathered in rank order)."""
    _dev(rewards, torch.float32, "rewards")
    _dev(seq_lens, torch.int64, "seq_lens")
    n = rewards.numel()
    _numel(n, seq_lens=seq_lens)
    dev = rewards.device
    ng = lib().yatt_grpo_num_local_groups(n, first_sample_id, group_size)
    keep = torch.empty((max(ng, 1),), dtype=torch.uint8, device=dev)
    imap = torch.empty((max(n, 1),), dtype=torch.int32, device=dev)
    new_cu = torch.empty((n + 1,), dtype=torch.int64, device=dev)
    counts = torch.empty((3,), dtype=torch.int64, device=dev)
    wsb = lib().yatt_filter_compact_workspace_bytes(n)
    ws = torch.empty((wsb,), dtype=torch.uint8, device=dev)
    if first_sample_id == 0 and all_records is None:
        check(lib().yatt_filter_compact(_p(rewards), _p(seq_lens), n, group_size, _p(keep),
                                        _p(imap), _p(new_cu), _p(counts), _p(ws), wsb, _st()))
    else:
        if all_records is not None:
            _dev(all_records, torch.int64, "all_records")
        check(lib().yatt_filter_compact_sharded(_p(rewards), _p(seq_lens), n, first_sample_id,
                                                group_size, _p(all_records), world, _p(keep),
                                                _p(imap), _p(new_cu), _p(counts), _p(ws), wsb,
                                                _st()))
    return {"keep_groups": keep[:ng], "index_map": imap, "new_cu": new_cu, "counts": counts}


def _moments_fit(moments: torch.Tensor, n: int, group_size: int, first_sample_id: int) -> None:
    """The per-group moments table must cover this shard's local groups."""
    ng = lib().yatt_grpo_num_local_groups(n, first_sample_id, group_size)
    if moments.numel() < 3 * ng:
        raise ValueError(f"moments holds {moments.numel()} doubles, the shard's {ng} groups "
                         f"need {3 * ng}")


def filter_boundary_record(rewards: torch.Tensor, group_size: int,
                           first_sample_id: int = 0) -> torch.Tensor:
    _dev(rewards, torch.float32, "rewards")
    rec = torch.empty((6,), dtype=torch.int64, device=rewards.device)
    check(lib().yatt_filter_boundary_record(_p(rewards), rewards.numel(), first_sample_id,
                                            group_size, _p(rec), _st()))
    return rec


def grpo_boundary_record(moments: torch.Tensor, n: int, group_size: int,
                         first_sample_id: int = 0) -> torch.Tensor:
    _dev(moments, torch.float64, "moments")
    _moments_fit(moments, n, group_size, first_sample_id)
    rec = torch.empty((8,), dtype=torch.float64, device=moments.device)
    check(lib().yatt_grpo_boundary_record(_p(moments), n, first_sample_id, group_size, _p(rec),
                                          _st()))
    return rec


def grpo_merge_boundaries(moments: torch.Tensor, n: int, group_size: int, first_sample_id: int,
                          all_records: torch.Tensor) -> torch.Tensor:
    _dev(moments, torch.float64, "moments")
    _dev(all_records, torch.float64, "all_records")
    _moments_fit(moments, n, group_size, first_sample_id)
    if all_records.numel() == 0 or all_records.numel() % 8:
        raise ValueError("all_records must hold 8 doubles per rank")
    check(lib().yatt_grpo_merge_boundaries(_p(moments), n, first_sample_id, group_size,
                                           _p(all_records), all_records.numel() // 8, _st()))
    return moments


def _plan_arrays(old_cu, index_map, new_cu, n_kept, max_kept, dst_offset=None):
    """The compaction plan's device arrays: dtypes, and sizes the gather
    kernels index up to max_kept."""
    _devs(torch.int64, old_cu=old_cu, new_cu=new_cu, n_kept=n_kept, dst_offset=dst_offset)
    _dev(index_map, torch.int32, "index_map")
    if max_kept < 0 or index_map.numel() < max_kept or new_cu.numel() < max_kept + 1:
        raise ValueError(f"index_map / new_cu must cover max_kept = {max_kept} samples")
    if n_kept.numel() < 1 or (dst_offset is not None and dst_offset.numel() < 1):
        raise ValueError("n_kept / dst_offset are one-element device counters")


def gather_varlen(src: torch.Tensor, old_cu: torch.Tensor, index_map: torch.Tensor,
                  new_cu: torch.Tensor, n_kept: torch.Tensor, max_kept: int, dst: torch.Tensor,
                  dst_offset: torch.Tensor | None = None) -> torch.Tensor:
    _dense(src=src, dst=dst)
    _plan_arrays(old_cu, index_map, new_cu, n_kept, max_kept, dst_offset)
    check(lib().yatt_gather_varlen(_p(src), _p(old_cu), _p(index_map), _p(new_cu), _p(n_kept),
                                   max_kept, _p(dst_offset), src.element_size(), _p(dst), _st()))
    return dst


def gather_varlen_multi(srcs, old_cu: torch.Tensor, index_map: torch.Tensor, new_cu: torch.Tensor,
                        n_kept: torch.Tensor, max_kept: int, dsts,
                        dst_offset: torch.Tensor | None = None):
    """gather_varlen over several per-token arrays (<= 8) in one launch."""
    _plan_arrays(old_cu, index_map, new_cu, n_kept, max_kept, dst_offset)
    n = len(srcs)
    if n != len(dsts):
        raise ValueError("srcs and dsts differ in length")
    for i, (a, b) in enumerate(zip(srcs, dsts)):
        _dense(**{f"srcs[{i}]": a, f"dsts[{i}]": b})
        if a.dtype != b.dtype:
            raise TypeError(f"srcs[{i}] and dsts[{i}] differ in dtype")
    h_src = (C.c_void_p * n)(*[t.data_ptr() for t in srcs])
    h_dst = (C.c_void_p * n)(*[t.data_ptr() for t in dsts])
    h_esz = (C.c_int32 * n)(*[t.element_size() for t in srcs])
    check(lib().yatt_gather_varlen_multi(n, h_src, h_dst, h_esz, _p(old_cu), _p(index_map),
                                         _p(new_cu), _p(n_kept), max_kept, _p(dst_offset), _st()))
    return dsts


def gather_rows(src: torch.Tensor, index_map: torch.Tensor, n_kept: torch.Tensor, max_kept: int,
                dst: torch.Tensor, dst_offset: torch.Tensor | None = None) -> torch.Tensor:
    _dense(src=src, dst=dst)
    _devs(torch.int64, n_kept=n_kept, dst_offset=dst_offset)
    _dev(index_map, torch.int32, "index_map")
    if max_kept < 0 or index_map.numel() < max_kept:
        raise ValueError(f"index_map must cover max_kept = {max_kept} rows")
    row_bytes = src[0].numel() * src.element_size() if src.dim() > 1 else src.element_size()
    check(lib().yatt_gather_rows(_p(src), _p(index_map), _p(n_kept), max_kept, row_bytes,
                                 _p(dst_offset), _p(dst), _st()))
    return dst


def microbatch_aggregates(prompt_len: torch.Tensor, out_len: torch.Tensor, microbatch_size: int,
                          controller_rank: int = 0, n: torch.Tensor | None = None,
                          max_n: int | None = None) -> torch.Tensor:
    _devs(torch.int32, prompt_len=prompt_len, out_len=out_len)
    _numel(prompt_len.numel(), out_len=out_len)
    if n is not None:
        _dev(n, torch.int64, "n")
    cap = prompt_len.numel() if max_n is None else max_n
    if cap > prompt_len.numel():
        raise ValueError("max_n exceeds the length arrays")
    nmb = -(-cap // microbatch_size)
    out = torch.zeros((max(nmb, 1), 6), dtype=torch.int32, device=prompt_len.device)  # 24 B rows
    check(lib().yatt_microbatch_aggregates(_p(prompt_len), _p(out_len), _p(n), cap,
                                           microbatch_size, controller_rank, _p(out), _st()))
    return out[:nmb]


def exclusive_offset(counts: torch.Tensor, nranks: int, rank: int, stride: int, field: int):
    _dev(counts, torch.int64, "counts")
    if counts.numel() < nranks * stride or not 0 <= field < stride:
        raise ValueError("counts must hold nranks x stride words and field < stride")
    out = torch.empty((1,), dtype=torch.int64, device=counts.device)
    check(lib().yatt_exclusive_offset(_p(counts), nranks, rank, stride, field, _p(out), _st()))
    return out


# ------------------------------------------------------------------ R10 ---
def sort_order_desc(lengths: torch.Tensor) -> torch.Tensor:
    _dev(lengths, torch.int32, "lengths")
    n = lengths.numel()
    order = torch.empty((n,), dtype=torch.int32, device=lengths.device)
    wsb = lib().yatt_sort_order_workspace_bytes(n)
    ws = torch.empty((wsb,), dtype=torch.uint8, device=lengths.device)
    check(lib().yatt_sort_order_desc(_p(lengths), n, _p(order), _p(ws), wsb, _st()))
    return order


# ------------------------------------- fused LM head + log-softmax (§8f #4) --
def lmhead_token_stats(hidden: torch.Tensor, lm_head: torch.Tensor, targets: torch.Tensor,
                       n_split: int | None = None, out: torch.Tensor | None = None):
    """(logp, entropy, lse) per row of softmax(hidden @ lm_head^T) without
    materialising the logits (tcgen05 GEMM + online LSE epilogue)."""
    _dev(hidden, torch.bfloat16, "hidden")
    _dev(lm_head, torch.bfloat16, "lm_head")
    _dev(targets, torch.int32, "targets")
    rows, d = hidden.shape
    vocab = lm_head.shape[0]
    if n_split is None:
        n_split = 0  # the library picks (yatt_lmhead_token_stats)
    if out is None:
        out = torch.empty((3, rows), dtype=torch.float32, device=hidden.device)
    wsb = lib().yatt_lmhead_workspace_bytes(rows, vocab, n_split)
    ws = torch.empty((max(wsb, 16),), dtype=torch.uint8, device=hidden.device)
    check(lib().yatt_lmhead_token_stats(_p(hidden), _p(lm_head), _p(targets), rows, d, vocab,
                                        n_split, _p(out[0]), _p(out[1]), _p(out[2]), _p(ws),
                                        wsb, _st()))
    return out[0], out[1], out[2]


def kl_from_logps(logp: torch.Tensor, ref_logp: torch.Tensor, kl_mode: str = "k3"):
    _devs(torch.float32, logp=logp, ref_logp=ref_logp)
    _numel(logp.numel(), ref_logp=ref_logp)
    kl = torch.empty_like(logp)
    check(lib().yatt_kl_from_logps(_p(logp), _p(ref_logp), logp.numel(), KL_MODES[kl_mode],
                                   _p(kl), _st()))
    return kl


# --------------------------------------------------- backward (§8f #1) ----
def policy_loss_grad(policy_logits, targets, old_logp, advantages, ref_logp=None, mask=None,
                     config=None, kl_mode="k3", norm: float = 1.0, grad=None, cu_seqlens=None,
                     ref_logits=None):
    """Fused training-side op (yatt_policy_loss_grad): from the policy logits
    alone, the per-token (logp, entropy, kl vs the stored ref_logp) AND
    dL/d(policy logits) (bf16 [rows, V]) of the A4 loss, each row streamed
    twice with the second read from L2.  norm: global valid-token count
    (token-mean) or global sequence count (seq modes; seq-mean-token-mean
    also takes cu_seqlens).  kl_mode "full" reads ref_logits (the
    full-vocabulary KL) instead of ref_logp.  Returns (logp, entropy, kl,
    grad); the loss sums
    follow from policy_loss(logp, old_logp, advantages, kl, entropy, ...)."""
    cfg = config or loss_config()
    _devs(torch.bfloat16, policy_logits=policy_logits, grad=grad, ref_logits=ref_logits)
    _devs(torch.float32, ref_logp=ref_logp, old_logp=old_logp, advantages=advantages)
    if ref_logits is not None and ref_logits.shape != policy_logits.shape:
        raise ValueError("ref_logits must have the shape of policy_logits")
    _dev(targets, torch.int32, "targets")
    if cu_seqlens is not None:
        _dev(cu_seqlens, torch.int64, "cu_seqlens")
    rows, vocab = policy_logits.shape
    _numel(rows, targets=targets, old_logp=old_logp, advantages=advantages, ref_logp=ref_logp,
           mask=mask)
    if grad is not None and grad.shape != policy_logits.shape:
        raise ValueError("grad must have the shape of policy_logits")
    out = torch.empty((3, rows), dtype=torch.float32, device=policy_logits.device)
    if grad is None:
        grad = torch.empty_like(policy_logits)
    wsb = lib().yatt_policy_loss_grad_workspace_bytes(rows, cfg.agg_mode)
    ws = torch.empty((max(wsb, 16),), dtype=torch.uint8, device=policy_logits.device)
    nseq = 0 if cu_seqlens is None else cu_seqlens.numel() - 1
    check(lib().yatt_policy_loss_grad(_p(policy_logits), _p(ref_logits), _p(targets),
                                      _p(_mask(mask)),
                                      _p(ref_logp), _p(old_logp), _p(advantages), rows, vocab,
                                      _p(cu_seqlens), nseq, C.byref(cfg), KL_MODES[kl_mode],
                                      float(norm), _p(out[0]), _p(out[1]), _p(out[2]), _p(grad),
                                      _p(ws), wsb, _st()))
    return out[0], out[1], out[2], grad


def logits_grad(policy_logits, ref_logits, targets, logp, ref_logp, old_logp, advantages,
                entropy, kl, mask=None, cu_seqlens=None, config=None, kl_mode="k3",
                norm: float = 1.0, grad=None):
    """dL/d(policy logits) of the A4 loss (bf16 [rows, V]) + the per-token
    coefficient table (fp32 [rows, 8]: g, h, f, lse_p, lse_q, H, KL, scratch)."""
    cfg = config or loss_config()
    _devs(torch.bfloat16, policy_logits=policy_logits, ref_logits=ref_logits, grad=grad)
    _devs(torch.float32, logp=logp, ref_logp=ref_logp, old_logp=old_logp, advantages=advantages,
          entropy=entropy, kl=kl)
    _dev(targets, torch.int32, "targets")
    rows, vocab = policy_logits.shape
    _numel(rows, targets=targets, logp=logp, ref_logp=ref_logp, old_logp=old_logp,
           advantages=advantages, entropy=entropy, kl=kl, mask=mask)
    if grad is not None and grad.shape != policy_logits.shape:
        raise ValueError("grad must have the shape of policy_logits")
    coef = torch.empty((rows, 8), dtype=torch.float32, device=policy_logits.device)
    m = _mask(mask)
    nseq = 0 if cu_seqlens is None else cu_seqlens.numel() - 1
    check(lib().yatt_policy_grad_coef(_p(policy_logits), _p(ref_logits), _p(targets), _p(logp),
                                      _p(ref_logp), _p(old_logp), _p(advantages), _p(entropy),
                                      _p(kl), _p(m), rows, vocab, _p(cu_seqlens), nseq,
                                      C.byref(cfg), KL_MODES[kl_mode], float(norm), _p(coef),
                                      _st()))
    if grad is None:
        grad = torch.empty_like(policy_logits)
    full = int(KL_MODES[kl_mode] == 3)
    check(lib().yatt_logits_backward(_p(policy_logits), _p(ref_logits) if full else None,
                                     _p(targets), _p(m), rows, vocab, _p(coef), full, _p(grad),
                                     _st()))
    return grad, coef
