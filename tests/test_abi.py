"""The C-ABI library loads without a GPU and exports every declared symbol;
host-only entry points behave like the reference (no compute calls here)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2508_07970_b200 import ConfigError, RankOutOfRange, api
from paper_2508_07970_b200._lib import LIB_PATH, SIGNATURES, lib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "yatt_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(yatt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    h = lib()
    missing = [s for s in declared_symbols() if not hasattr(h, s)]
    assert not missing, missing
    assert set(declared_symbols()) <= set(SIGNATURES) | {"yatt_abi_version"}
    assert h.yatt_abi_version() == 3


def test_cpp_dropin_api_is_exported():
    out = subprocess.run(["nm", "-DC", str(LIB_PATH)], capture_output=True, text=True).stdout
    for sym in ["yatt::workload::rejection_process(", "yatt::workload::shard_dataset(",
                "yatt::workload::sample_length_keyed(", "yatt::sim::shard_round_output(",
                "yatt::sim::make_shard_state(", "yatt::sim::run_rollout_rounds(",
                "yatt::balancer::sort_and_bucket(", "yatt::balancer::padding_waste(",
                "yatt::experience::token_logprob_stats(", "yatt::experience::policy_loss(",
                "yatt::experience::gae(", "yatt::experience::grpo_advantages(",
                "yatt::experience::dynamic_sampling_filter(",
                "yatt::experience::policy_logits_grad(", "yatt::experience::lmhead_token_stats(",
                "yatt::experience::gather_payload(", "yatt::experience::PeerGroup::PeerGroup(",
                "yatt::experience::PeerGroup::policy_loss("]:
        assert sym in out, sym


def test_library_links_sm100a_code_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB_PATH)], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_shard_dataset_host_entry_point():
    # workload_test.cpp:166-197 known answers
    assert [api.shard_dataset(10, 3, r).size() for r in range(3)] == [4, 3, 3]
    assert api.shard_dataset(100, 1, 0) == api.ShardRange(0, 100)
    cursor = 0
    for r in range(7):
        s = api.shard_dataset(1037, 7, r)
        assert s.begin == cursor
        cursor = s.end
    assert cursor == 1037
    with pytest.raises(RankOutOfRange):
        api.shard_dataset(10, 3, 3)
    with pytest.raises(RankOutOfRange):
        api.shard_dataset(10, 3, -1)
    with pytest.raises(ConfigError):
        api.shard_dataset(10, 0, 0)


def test_loss_finalize_host_entry_point():
    from paper_2508_07970_b200 import ops
    cfg = ops.loss_config(agg_mode="token-mean")
    assert ops.loss_finalize([6.0, 0, 0, 0, 0, 0, 3.0, 0.0], cfg) == 2.0
    cfg1 = ops.loss_config(agg_mode="seq-mean-token-mean")
    assert ops.loss_finalize([1.5, 0, 0, 0, 0, 0, 9.0, 3.0], cfg1) == 0.5
    assert ops.loss_finalize([1.5, 0, 0, 0, 0, 0, 0.0, 0.0], cfg1) == 0.0


def test_errors_are_typed_and_messages_thread_local():
    # A config error raised by validation before any device work.
    h = lib()
    rc = h.yatt_shard_dataset(5, 0, 0, None, None)
    assert rc == 1
    assert b"num_controllers" in h.yatt_last_error_message()
    assert h.yatt_shard_dataset(5, 2, 9, None, None) == 2


def test_misaligned_pointers_are_config_errors_before_any_launch():
    """Alignment contract (yatt_cuda.h "Conventions"): checked before any CUDA
    call, so fake addresses never reach the device and this runs on CPU."""
    from paper_2508_07970_b200._lib import check
    A, M = 0x10000, 0x10001  # aligned / misaligned fake device addresses
    calls = [
        ("gae", lambda: lib().yatt_gae(A, A, None, A, 1, 1, 1.0, 1.0, A + 2, A, A, 64, None)),
        ("coef", lambda: lib().yatt_logits_backward(A, None, A, None, 1, 8, A + 4, 0, A, None)),
        ("mbs", lambda: lib().yatt_microbatch_aggregates(A, A, None, 1, 1, 0, A + 4, None)),
        ("sums", lambda: lib().yatt_policy_loss(A, A, A, A, A, None, 1, None, 0, None, A + 4, A, 64,
                                                None)),
        ("order", lambda: lib().yatt_sort_order_desc(A, 1, M, A, 64, None)),
        ("new_cu", lambda: lib().yatt_filter_compact(A, A, 1, 1, A, A, A + 4, A, A, 64, None)),
        ("out", lambda: lib().yatt_token_stats(A, A, A, None, 1, 8, 2, A, A, A + 1, A, None)),
        ("ws", lambda: lib().yatt_lmhead_token_stats(A, A, A, 1, 64, 8, 1, A, A, A, A + 8, 64,
                                                     None)),
        ("d_record", lambda: lib().yatt_grpo_boundary_record(A, 8, 0, 8, A + 4, None)),
        ("d_all_records", lambda: lib().yatt_grpo_merge_boundaries(A, 8, 0, 8, A + 4, 2, None)),
        ("d_rewards", lambda: lib().yatt_filter_boundary_record(M, 8, 0, 8, A, None)),
        ("d_ws", lambda: lib().yatt_peer_grpo_advantages(None, A, 8, 0, 8, 1e-6, 1, A, A + 4, 4096,
                                                         None)),
        ("d_new_cu", lambda: lib().yatt_peer_filter_compact(None, A, A, 8, 0, 8, A, A, A + 4, A, A,
                                                            4096, None)),
    ]
    for what, fn in calls:
        with pytest.raises(ConfigError, match="aligned"):
            check(fn())


def test_peer_group_argument_errors_before_any_cuda_call():
    """yatt_peer_* validate world / rank / pointers before touching CUDA."""
    from paper_2508_07970_b200._lib import check
    h = C.c_void_p()
    buf = (C.c_uint8 * 64)()
    with pytest.raises(ConfigError):
        check(lib().yatt_peer_create(0, 0, C.byref(h), C.addressof(buf)))
    with pytest.raises(ConfigError):
        check(lib().yatt_peer_create(9, 0, C.byref(h), C.addressof(buf)))
    with pytest.raises(RankOutOfRange):
        check(lib().yatt_peer_create(2, 2, C.byref(h), C.addressof(buf)))
    with pytest.raises(ConfigError):
        check(lib().yatt_peer_connect(None, C.addressof(buf)))
    with pytest.raises(ConfigError, match="create"):
        check(lib().yatt_peer_allreduce_f64(None, 0x10000, 4, 0x10000, None))
    with pytest.raises(ConfigError):
        check(lib().yatt_peer_scan_i64(None, 0x10000, 17, None, None, None))
    assert lib().yatt_peer_destroy(None) == 0


def test_host_entry_points_validate_buffers_before_the_call():
    """ops.*_host check dtype / shape / contiguity of every host buffer
    (including the caller's `out` / `stats_out`) before the C-ABI call, which
    trusts the sizes it is given (no compute happens here: every case raises
    first)."""
    import numpy as np
    from paper_2508_07970_b200 import ops
    rows, V = 4, 16
    pol = np.zeros((rows, V), np.uint16)
    tgt = np.zeros(rows, np.int32)
    with pytest.raises(TypeError):
        ops.token_stats_host(pol, pol, tgt.astype(np.int64))
    with pytest.raises(TypeError):
        ops.token_stats_host(pol.astype(np.float16), pol, tgt)
    with pytest.raises(ValueError):
        ops.token_stats_host(pol, pol[:, :8].copy(), tgt)
    with pytest.raises(ValueError):
        ops.token_stats_host(pol, pol, tgt, out=np.empty((4, rows - 1), np.float32))
    with pytest.raises(TypeError):
        ops.token_stats_host(pol, pol, tgt, out=np.empty((4, rows), np.float16))
    with pytest.raises(ValueError):
        ops.token_stats_host(pol, pol, tgt, mask=np.ones(rows + 1, np.uint8))
    with pytest.raises(ValueError):
        ops.token_stats_host(np.asfortranarray(pol), pol, tgt)
    rew, old = np.zeros(2, np.float32), np.zeros(rows, np.float32)
    with pytest.raises(ValueError):
        ops.grpo_step_host(pol, pol, tgt, rew, old, 2, stats_out=np.empty((4, 2), np.float32))
    with pytest.raises(TypeError):
        ops.grpo_step_host(pol, pol, tgt, rew.astype(np.float64), old, 2)
    with pytest.raises(ValueError):
        ops.grpo_step_host(pol, pol, tgt, np.zeros(3, np.float32), old, 3)
