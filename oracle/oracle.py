"""numpy/ctypes front-end of the CPU oracle (oracle/yatt_oracle.c).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, as the checker / timed CPU baseline.  The
product path (paper_2508_07970_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"
SRC = HERE / "yatt_oracle.c"


def build() -> Path:
    """Compile the C restatement (gcc, -O2, no fast-math: IEEE fp64)."""
    LIB.parent.mkdir(exist_ok=True)
    if LIB.exists() and LIB.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB
    tmp = LIB.with_suffix(".tmp.so")
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-fno-fast-math", str(SRC),
                    "-o", str(tmp), "-lm", "-lpthread"], check=True)
    os.replace(tmp, LIB)
    return LIB


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(LIB))
        _lib.yo_splitmix64.restype = C.c_uint64
        _lib.yo_splitmix64.argtypes = [C.c_uint64]
        _lib.yo_hash_key.restype = C.c_uint64
        _lib.yo_hash_key.argtypes = [C.c_void_p, C.c_int]
        _lib.yo_uniform_from_key.restype = C.c_double
        _lib.yo_uniform_from_key.argtypes = [C.c_uint64]
        _lib.yo_sample_length_keyed.restype = C.c_int
        _lib.yo_sample_length_keyed.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int,
                                                C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                                C.c_uint64]
        _lib.yo_sample_lengths_range.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int] + \
            [C.c_uint64] * 5 + [C.c_int64, C.c_void_p]
        _lib.yo_near_ties.restype = C.c_int64
        _lib.yo_near_ties.argtypes = [C.c_int, C.c_double, C.c_double] + [C.c_uint64] * 5 + \
            [C.c_int64, C.c_double, C.c_void_p, C.c_int64]
        _lib.yo_shard_dataset.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        _lib.yo_rejection_flags.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                            C.c_double, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        _lib.yo_shard_round.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.c_double, C.c_int, C.c_double, C.c_int,
                                        C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_void_p,
                                        C.c_void_p]
        _lib.yo_sort_order_desc.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        _lib.yo_padding_waste.restype = C.c_double
        _lib.yo_padding_waste.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        _lib.yo_synth_logits.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p,
                                         C.c_void_p, C.c_void_p]
        _lib.yo_synth_floats.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int,
                                         C.c_int, C.c_void_p, C.c_void_p]
        _lib.yo_token_stats.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                        C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_int]
        _lib.yo_grpo_advantages.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_float,
                                            C.c_int, C.c_void_p]
        _lib.yo_gae.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                C.c_double, C.c_double, C.c_void_p, C.c_void_p]
        _lib.yo_masked_moments.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        _lib.yo_policy_loss.argtypes = [C.c_void_p] * 6 + [C.c_int64, C.c_void_p, C.c_int64] + \
            [C.c_float] * 5 + [C.c_int, C.c_void_p]
        _lib.yo_filter_compact.restype = C.c_int64
        _lib.yo_filter_compact.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p]
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


SAMPLE_DT = np.dtype([("sample_id", "<u8"), ("prompt_len_tokens", "<i4"),
                      ("out_len_tokens", "<i4"), ("accepted_round", "<i4"), ("accepted", "<i4")])
MB_DT = np.dtype([("controller_rank", "<i4"), ("mb_index", "<i4"), ("sample_count", "<i4"),
                  ("max_out_len_tokens", "<i4"), ("score_tokens", "<i8")])
REPORT_DT = np.dtype([("controller_rank", "<i4"), ("round", "<i4"), ("active_count", "<i4"),
                      ("newly_accepted_count", "<i4"), ("forced_accept_count", "<i4"),
                      ("pending_count", "<i4"), ("accepted_score_tokens", "<i8"),
                      ("accepted_train_units", "<i8"), ("num_microbatches", "<i8")])


# ---------------------------------------------------------------- L0 / R ---
def splitmix64(x: int) -> int:
    return lib().yo_splitmix64(x)


def hash_key(parts) -> int:
    a = np.asarray(parts, dtype=np.uint64)
    return lib().yo_hash_key(a.ctypes.data, len(a))


def uniform_from_key(key: int) -> float:
    return lib().yo_uniform_from_key(key)


def sample_length_keyed(kind, p1, p2, max_len, seed, stream, step, round_, sample_id) -> int:
    return lib().yo_sample_length_keyed(kind, p1, p2, max_len, seed, stream, step, round_,
                                        sample_id)


def sample_lengths_range(kind, p1, p2, max_len, seed, stream, step, round_, id0, n):
    out = np.empty(n, dtype=np.int32)
    lib().yo_sample_lengths_range(kind, p1, p2, max_len, seed, stream, step, round_, id0, n,
                                  out.ctypes.data)
    return out


def near_ties(kind, p1, p2, seed, stream, step, round_, id0, n, band, cap=4096):
    """ids whose glibc pre-rounding value lies within band of a .5 tie."""
    out = np.empty(cap, dtype=np.uint64)
    found = lib().yo_near_ties(kind, p1, p2, seed, stream, step, round_, id0, n, band,
                               out.ctypes.data, cap)
    return out[:min(found, cap)], found


def shard_dataset(total: int, p: int, r: int):
    b, e = C.c_uint64(), C.c_uint64()
    rc = lib().yo_shard_dataset(total, p, r, C.byref(b), C.byref(e))
    return rc, b.value, e.value


def rejection_flags(ids, accepted, step, round_, rate, per_group, G, seed) -> np.ndarray:
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    acc = np.ascontiguousarray(accepted, dtype=np.uint8)
    out = np.zeros(len(ids), dtype=np.uint8)
    rc = lib().yo_rejection_flags(_ptr(ids), _ptr(acc), len(ids), step, round_, rate,
                                  int(per_group), G, seed, _ptr(out))
    if rc:
        raise ValueError("ConfigError")
    return out


def shard_round(samples: np.ndarray, rank, step, round_, dist, rate, per_group, G, seed, mb,
                max_rounds):
    """samples: SAMPLE_DT array, mutated in place.  dist = (kind, p1, p2, max_len)."""
    n = len(samples)
    mbs = np.zeros(max(-(-n // mb), 1), dtype=MB_DT)
    rep = np.zeros(1, dtype=REPORT_DT)
    kind, p1, p2, max_len = dist
    rc = lib().yo_shard_round(_ptr(samples), n, rank, step, round_, kind, p1, p2, max_len, rate,
                              int(per_group), G, seed, mb, max_rounds, _ptr(rep), _ptr(mbs))
    if rc:
        raise ValueError("ConfigError")
    return rep[0], mbs[: int(rep[0]["num_microbatches"])]


def sort_order_desc(lengths) -> np.ndarray:
    ln = np.ascontiguousarray(lengths, dtype=np.int32)
    out = np.zeros(len(ln), dtype=np.uint32)
    lib().yo_sort_order_desc(_ptr(ln), len(ln), _ptr(out))
    return out


def padding_waste(flat, offsets, lengths) -> float:
    f = np.ascontiguousarray(flat, dtype=np.uint32)
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    ln = np.ascontiguousarray(lengths, dtype=np.int32)
    return lib().yo_padding_waste(_ptr(f), _ptr(o), len(o) - 1, _ptr(ln))


# ------------------------------------------------------------- synthetic ---
def synth_logits(seed, row0, rows, vocab):
    pol = np.empty((rows, vocab), dtype=np.uint16)
    ref = np.empty((rows, vocab), dtype=np.uint16)
    tgt = np.empty((rows,), dtype=np.int32)
    lib().yo_synth_logits(seed, row0, rows, vocab, _ptr(pol), _ptr(ref), _ptr(tgt))
    return pol, ref, tgt


SYNTH = {"logp": 0, "old_delta": 1, "adv": 2, "kl": 3, "value": 4, "reward": 5}


def synth_floats(seed, stream_id, i0, n, kind, group_size=1, base=None) -> np.ndarray:
    out = np.empty((n,), dtype=np.float32)
    b = None if base is None else np.ascontiguousarray(base, dtype=np.float32)
    lib().yo_synth_floats(seed, stream_id, i0, n, SYNTH[kind], group_size, _ptr(b), _ptr(out))
    return out


# -------------------------------------------------------------- float path --
KL_MODES = {"k1": 0, "k2": 1, "k3": 2, "full": 3}


def token_stats(pol, ref, tgt, mask=None, kl_mode="k3", threads=None):
    rows, vocab = pol.shape
    out = np.zeros((4, rows), dtype=np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    lib().yo_token_stats(_ptr(pol), _ptr(ref), _ptr(np.ascontiguousarray(tgt, dtype=np.int32)),
                         _ptr(m), rows, vocab, KL_MODES[kl_mode], _ptr(out[0]), _ptr(out[1]),
                         _ptr(out[2]), _ptr(out[3]), threads or os.cpu_count() or 1)
    return out


def grpo_advantages(rewards, group_size, eps=1e-6, norm_by_std=True, first_sample_id=0):
    r = np.ascontiguousarray(rewards, dtype=np.float32)
    out = np.zeros(len(r), dtype=np.float64)
    lib().yo_grpo_advantages(_ptr(r), len(r), first_sample_id, group_size, eps, int(norm_by_std),
                             _ptr(out))
    return out


def gae(values, rewards, cu, mask=None, gamma=1.0, lam=0.95):
    v = np.ascontiguousarray(values, dtype=np.float32)
    r = np.ascontiguousarray(rewards, dtype=np.float32)
    c = np.ascontiguousarray(cu, dtype=np.int64)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    adv = np.zeros(len(v), dtype=np.float64)
    ret = np.zeros(len(v), dtype=np.float64)
    lib().yo_gae(_ptr(v), _ptr(r), _ptr(m), _ptr(c), len(c) - 1, float(np.float32(gamma)),
                 float(np.float32(lam)), _ptr(adv), _ptr(ret))
    return adv, ret


def masked_moments(x, mask=None):
    xv = np.ascontiguousarray(x, dtype=np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    out = np.zeros(3, dtype=np.float64)
    lib().yo_masked_moments(_ptr(xv), _ptr(m), len(xv), _ptr(out))
    return out


def policy_loss(logp, old_logp, adv, kl, ent, mask=None, cu=None, clip_low=0.2, clip_high=0.2,
                clip_ratio_c=0.0, kl_coef=0.001, entropy_coef=0.0, agg_mode=0):
    f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    c = None if cu is None else np.ascontiguousarray(cu, dtype=np.int64)
    sums = np.zeros(8, dtype=np.float64)
    arrs = [f(logp), f(old_logp), f(adv), f(kl), f(ent)]
    lib().yo_policy_loss(*[_ptr(a) for a in arrs], _ptr(m), len(arrs[0]), _ptr(c),
                         0 if c is None else len(c) - 1, clip_low, clip_high, clip_ratio_c,
                         kl_coef, entropy_coef, agg_mode, _ptr(sums))
    return sums


def filter_compact(rewards, lens, group_size):
    r = np.ascontiguousarray(rewards, dtype=np.float32)
    ln = np.ascontiguousarray(lens, dtype=np.int64)
    n = len(r)
    ng = -(-n // group_size)  # a trailing partial group is a group of its own
    keep = np.zeros(max(ng, 1), dtype=np.uint8)
    imap = np.zeros(max(n, 1), dtype=np.int32)
    new_cu = np.zeros(n + 1, dtype=np.int64)
    counts = np.zeros(3, dtype=np.int64)
    k = lib().yo_filter_compact(_ptr(r), _ptr(ln), n, group_size, _ptr(keep), _ptr(imap),
                                _ptr(new_cu), _ptr(counts))
    return {"keep_groups": keep[:ng], "index_map": imap[:k], "new_cu": new_cu[: k + 1],
            "counts": counts}


def max_rel_error(actual, expected) -> float:
    """proj/src/distattn.cpp:234-244: max |a-e| / (|e| + 1e-12)."""
    a = np.asarray(actual, dtype=np.float64).ravel()
    e = np.asarray(expected, dtype=np.float64).ravel()
    if a.shape != e.shape:
        raise ValueError("tensor size mismatch")
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - e) / (np.abs(e) + 1e-12)))


def logits_backward(pol, ref, tgt, logp, ref_logp, old_logp, adv, mask=None, cu=None,
                    clip_low=0.2, clip_high=0.2, clip_ratio_c=0.0, kl_coef=0.001,
                    entropy_coef=0.0, agg_mode=0, kl_mode="k3", norm=1.0):
    """fp64 dL/dx [rows, V] (+ per-row g, h, f, lse) — see yatt_oracle.c."""
    L = lib()
    if not getattr(L, "_bwd_ready", False):
        L.yo_logits_backward.argtypes = [C.c_void_p] * 4 + [C.c_int64, C.c_int32] + \
            [C.c_void_p] * 5 + [C.c_int64] + [C.c_float] * 5 + [C.c_int, C.c_int, C.c_double,
                                                               C.c_void_p, C.c_void_p]
        L._bwd_ready = True
    rows, V = pol.shape
    f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    grad = np.zeros((rows, V), dtype=np.float64)
    coef = np.zeros((rows, 4), dtype=np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    c = None if cu is None else np.ascontiguousarray(cu, dtype=np.int64)
    args = [f(logp), f(ref_logp), f(old_logp), f(adv)]
    L.yo_logits_backward(_ptr(pol), _ptr(ref), _ptr(np.ascontiguousarray(tgt, dtype=np.int32)),
                         _ptr(m), rows, V, *[_ptr(a) for a in args], _ptr(c),
                         0 if c is None else len(c) - 1, clip_low, clip_high, clip_ratio_c,
                         kl_coef, entropy_coef, agg_mode, KL_MODES[kl_mode], norm, _ptr(grad),
                         _ptr(coef))
    return grad, coef
