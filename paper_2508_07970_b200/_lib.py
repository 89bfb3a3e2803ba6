"""ctypes binding of ``libyatt_b200.so`` (the C ABI in include/yatt_cuda.h).

The library is the product: there is no Python or CPU fallback.  If the
shared object is missing the import of any op raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("YATT_B200_LIB") or
                Path(__file__).resolve().parent / "libyatt_b200.so")

c_i32, c_i64, c_u64, c_f32, c_f64, c_p, c_sz = (C.c_int32, C.c_int64, C.c_uint64, C.c_float,
                                                C.c_double, C.c_void_p, C.c_size_t)

# ---------------------------------------------------------------- errors --
YATT_OK, ERR_CONFIG, ERR_RANK, ERR_DIST, ERR_CUDA, ERR_NCCL, ERR_WORKSPACE = range(7)


class YattError(RuntimeError):
    """yatt::Error (proj/include/yatt/errors.hpp:10-13)."""


class ConfigError(YattError):
    """yatt::ConfigError (errors.hpp:45-48)."""


class RankOutOfRange(YattError):
    """yatt::RankOutOfRange (errors.hpp:25-28)."""


class InvalidDistribution(YattError):
    """yatt::InvalidDistribution (errors.hpp:20-23)."""


_ERR = {ERR_CONFIG: ConfigError, ERR_RANK: RankOutOfRange, ERR_DIST: InvalidDistribution,
        ERR_WORKSPACE: ConfigError}


# ------------------------------------------------------------ POD structs --
class LengthDist(C.Structure):
    _fields_ = [("kind", c_i32), ("max_len_tokens", c_i32), ("p1", c_f64), ("p2", c_f64)]


class RejectionCfg(C.Structure):
    _fields_ = [("reject_rate", c_f64), ("per_group", c_i32), ("group_size", c_i32)]


class RoundParamsC(C.Structure):
    _fields_ = [("out_dist", LengthDist), ("rejection", RejectionCfg), ("seed", c_u64),
                ("microbatch_size", c_i32), ("max_rounds", c_i32)]


class SampleC(C.Structure):
    _fields_ = [("sample_id", c_u64), ("prompt_len_tokens", c_i32), ("out_len_tokens", c_i32),
                ("accepted_round", c_i32), ("accepted", c_i32)]


class MbAggC(C.Structure):
    _fields_ = [("controller_rank", c_i32), ("mb_index", c_i32), ("sample_count", c_i32),
                ("max_out_len_tokens", c_i32), ("score_tokens", c_i64)]


class ReportC(C.Structure):
    _fields_ = [("controller_rank", c_i32), ("round", c_i32), ("active_count", c_i32),
                ("newly_accepted_count", c_i32), ("forced_accept_count", c_i32),
                ("pending_count", c_i32), ("accepted_score_tokens", c_i64),
                ("accepted_train_units", c_i64), ("num_microbatches", c_i64)]


class RoundsIoC(C.Structure):
    _fields_ = [("sample_id", c_p), ("prompt_len", c_p), ("accepted", c_p), ("out_len", c_p),
                ("accepted_round", c_p), ("accepted_out", c_p), ("first_round_len", c_p)]


class RoundsViewC(C.Structure):
    _fields_ = [("reports", c_p), ("rounds", c_i32), ("num_shards", c_i32),
                ("microbatches", c_p), ("num_microbatches", c_i64), ("redrawn_on_host", c_i64),
                ("first_round_lens_valid", c_i32)]


class LossConfigC(C.Structure):
    _fields_ = [("clip_low", c_f32), ("clip_high", c_f32), ("clip_ratio_c", c_f32),
                ("kl_coef", c_f32), ("entropy_coef", c_f32), ("agg_mode", c_i32)]


class LossSumsC(C.Structure):
    _fields_ = [(n, c_f64) for n in ("loss_sum", "pg_sum", "kl_sum", "entropy_sum", "clip_count",
                                     "ratio_sum", "token_count", "seq_count")]


P = C.POINTER
# name -> (restype, argtypes)
SIGNATURES = {
    "yatt_last_error_message": (C.c_char_p, []),
    "yatt_abi_version": (C.c_int, []),
    "yatt_device_info": (C.c_int, [C.c_int, C.c_char_p, C.c_int, P(C.c_int), P(C.c_int),
                                   P(C.c_int)]),
    "yatt_shard_dataset": (C.c_int, [c_u64, c_i32, c_i32, P(c_u64), P(c_u64)]),
    "yatt_sample_lengths_keyed": (C.c_int, [P(LengthDist), c_u64, c_u64, c_u64, c_u64, c_p, c_i64,
                                            c_p, c_p]),
    "yatt_rejection_flags": (C.c_int, [c_p, c_i64, c_i32, c_i32, P(RejectionCfg), c_u64, c_p,
                                       c_p]),
    "yatt_shard_round": (C.c_int, [c_p, P(c_i64), c_i32, c_i32, c_i32, c_i32, P(RoundParamsC), c_p,
                                   c_p, c_p]),
    "yatt_reduce_round_reports": (C.c_int, [c_p, c_i32, c_p, c_p]),
    "yatt_rounds_create": (C.c_int, [P(c_p)]),
    "yatt_rounds_destroy": (None, [c_p]),
    "yatt_rounds_stage": (C.c_int, [c_p, c_i64, c_i32, P(RoundsIoC)]),
    "yatt_rounds_run": (C.c_int, [c_p, c_i64, P(c_i64), c_i32, c_i32, c_i32, c_i32, c_i32,
                                  P(RoundParamsC), c_i32, c_p]),
    "yatt_peer_rounds_run": (C.c_int, [c_p, c_p, c_i64, c_i32, P(RoundParamsC), c_i32, c_p]),
    "yatt_rounds_result": (C.c_int, [c_p, P(RoundsViewC)]),
    "yatt_sample_lengths_host": (C.c_int, [P(LengthDist), c_u64, c_u64, c_u64, c_u64, c_p, c_i64,
                                           c_p]),
    "yatt_set_tie_band": (C.c_int, [c_f64]),
    "yatt_uncertified_draws": (C.c_int, [P(c_i64), c_i32]),
    "yatt_lmhead_workspace_bytes": (c_sz, [c_i64, c_i32, c_i32]),
    "yatt_lmhead_token_stats": (C.c_int, [c_p, c_p, c_p, c_i64, c_i32, c_i32, c_i32, c_p, c_p,
                                          c_p, c_p, c_sz, c_p]),
    "yatt_kl_from_logps": (C.c_int, [c_p, c_p, c_i64, c_i32, c_p, c_p]),
    "yatt_token_stats": (C.c_int, [c_p, c_p, c_p, c_p, c_i64, c_i32, c_i32, c_p, c_p, c_p, c_p,
                                   c_p]),
    "yatt_token_stats_host": (C.c_int, [c_p, c_p, c_p, c_p, c_i64, c_i32, c_i32, c_p, c_p, c_p,
                                        c_p]),
    "yatt_grpo_step_host": (C.c_int, [c_p, c_p, c_p, c_p, c_i64, c_i32, c_p, c_i64, c_u64, c_i32,
                                      c_p, P(LossConfigC), c_i32, c_p, c_p]),
    "yatt_grpo_num_local_groups": (c_i64, [c_i64, c_u64, c_i32]),
    "yatt_grpo_group_moments": (C.c_int, [c_p, c_i64, c_u64, c_i32, c_p, c_p]),
    "yatt_grpo_advantages": (C.c_int, [c_p, c_i64, c_u64, c_i32, c_f32, c_i32, c_p, c_p, c_p]),
    "yatt_broadcast_to_tokens": (C.c_int, [c_p, c_p, c_i64, c_p, c_p, c_i64, c_p]),
    "yatt_gae_workspace_bytes": (c_sz, [c_i64]),
    "yatt_gae_with_moments": (C.c_int, [c_p, c_p, c_p, c_p, c_i64, c_i64, c_f32, c_f32, c_p, c_p,
                                        c_p, c_p, c_sz, c_p]),
    "yatt_gae": (C.c_int, [c_p, c_p, c_p, c_p, c_i64, c_i64, c_f32, c_f32, c_p, c_p, c_p, c_sz,
                           c_p]),
    "yatt_masked_moments_workspace_bytes": (c_sz, []),
    "yatt_masked_moments": (C.c_int, [c_p, c_p, c_i64, c_p, c_p, c_sz, c_p]),
    "yatt_whiten": (C.c_int, [c_p, c_p, c_i64, c_p, c_i32, c_p]),
    "yatt_policy_loss_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32]),
    "yatt_policy_loss": (C.c_int, [c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_p, c_i64,
                                   P(LossConfigC), c_p, c_p, c_sz, c_p]),
    "yatt_loss_finalize": (c_f64, [P(LossSumsC), P(LossConfigC)]),
    "yatt_policy_grad_coef": (C.c_int, [c_p] * 10 + [c_i64, c_i32, c_p, c_i64, P(LossConfigC),
                                                       c_i32, c_f64, c_p, c_p]),
    "yatt_logits_backward": (C.c_int, [c_p, c_p, c_p, c_p, c_i64, c_i32, c_p, c_i32, c_p, c_p]),
    "yatt_policy_loss_grad_workspace_bytes": (c_sz, [c_i64, c_i32]),
    "yatt_policy_loss_grad": (C.c_int, [c_p] * 7 + [c_i64, c_i32, c_p, c_i64, P(LossConfigC),
                                                    c_i32, c_f64] + [c_p] * 5 + [c_sz, c_p]),
    "yatt_filter_compact_workspace_bytes": (c_sz, [c_i64]),
    "yatt_filter_boundary_record": (C.c_int, [c_p, c_i64, c_u64, c_i32, c_p, c_p]),
    "yatt_filter_compact_sharded": (C.c_int, [c_p, c_p, c_i64, c_u64, c_i32, c_p, c_i32, c_p, c_p,
                                              c_p, c_p, c_p, c_sz, c_p]),
    "yatt_grpo_boundary_record": (C.c_int, [c_p, c_i64, c_u64, c_i32, c_p, c_p]),
    "yatt_grpo_merge_boundaries": (C.c_int, [c_p, c_i64, c_u64, c_i32, c_p, c_i32, c_p]),
    "yatt_straddle_workspace_bytes": (c_sz, [c_i64, c_u64, c_i32, c_i32]),
    "yatt_peer_world": (C.c_int, [c_p, P(c_i32), P(c_i32)]),
    "yatt_peer_grpo_advantages": (C.c_int, [c_p, c_p, c_i64, c_u64, c_i32, c_f32, c_i32, c_p, c_p,
                                            c_sz, c_p]),
    "yatt_peer_filter_compact": (C.c_int, [c_p, c_p, c_p, c_i64, c_u64, c_i32, c_p, c_p, c_p, c_p,
                                           c_p, c_sz, c_p]),
    "yatt_filter_compact": (C.c_int, [c_p, c_p, c_i64, c_i32, c_p, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "yatt_gather_varlen": (C.c_int, [c_p, c_p, c_p, c_p, c_p, c_i64, c_p, c_i32, c_p, c_p]),
    "yatt_gather_varlen_multi": (C.c_int, [c_i32, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_p,
                                           c_p]),
    "yatt_gather_rows": (C.c_int, [c_p, c_p, c_p, c_i64, c_i64, c_p, c_p, c_p]),
    "yatt_microbatch_aggregates": (C.c_int, [c_p, c_p, c_p, c_i64, c_i32, c_i32, c_p, c_p]),
    "yatt_exclusive_offset": (C.c_int, [c_p, c_i32, c_i32, c_i32, c_i32, c_p, c_p]),
    "yatt_sort_order_workspace_bytes": (c_sz, [c_i64]),
    "yatt_sort_order_desc": (C.c_int, [c_p, c_i64, c_p, c_p, c_sz, c_p]),
    "yatt_sort_and_bucket_host": (C.c_int, [c_p, c_i64, c_i32, c_u64, c_p, c_p]),
    "yatt_peer_create": (C.c_int, [c_i32, c_i32, P(c_p), c_p]),
    "yatt_peer_connect": (C.c_int, [c_p, c_p]),
    "yatt_peer_destroy": (C.c_int, [c_p]),
    "yatt_peer_status": (C.c_int, [c_p, P(c_i32)]),
    "yatt_peer_allreduce_f64": (C.c_int, [c_p, c_p, c_i32, c_p, c_p]),
    "yatt_peer_scan_i64": (C.c_int, [c_p, c_p, c_i32, c_p, c_p, c_p]),
    "yatt_peer_allgather_i64": (C.c_int, [c_p, c_p, c_i32, c_p, c_p]),
    "yatt_policy_loss_allreduce": (C.c_int, [c_p] * 7 + [c_i64, c_p, c_i64, P(LossConfigC), c_p, c_p,
                                                         c_sz, c_p]),
    "yatt_comm_unique_id": (C.c_int, [c_p]),
    "yatt_comm_init": (C.c_int, [c_i32, c_i32, c_p, P(c_p)]),
    "yatt_comm_destroy": (C.c_int, [c_p]),
    "yatt_comm_allreduce_f64": (C.c_int, [c_p, c_p, c_i64, c_p]),
    "yatt_comm_allreduce_i64": (C.c_int, [c_p, c_p, c_i64, c_p]),
    "yatt_comm_allgather_i64": (C.c_int, [c_p, c_p, c_p, c_i64, c_p]),
    "yatt_synth_logits": (C.c_int, [c_u64, c_i64, c_i64, c_i32, c_p, c_p, c_p, c_p]),
    "yatt_synth_floats": (C.c_int, [c_u64, c_u64, c_i64, c_i64, c_i32, c_i32, c_p, c_p, c_p]),
}

_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2508_07970_b200.build` "
                "(there is no CPU fallback)")
        handle = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    """Map a C-ABI status onto the reference's exception types."""
    if rc == YATT_OK:
        return
    msg = lib().yatt_last_error_message().decode(errors="replace")
    raise _ERR.get(rc, YattError)(msg)
