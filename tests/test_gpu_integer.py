"""Integer path on the B200, bit-exact against the reference's golden vectors
(tests/golden, from oracle/_ref) and the pinned CPU oracle.

Reads like the reference's own tests (proj/tests/workload_test.cpp,
simcore_test.cpp, balancer_test.cpp) through the Python mirror of its API.
"""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2508_07970_b200 import ConfigError, api, ops

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"


def load(name):
    return json.loads((GOLD / name).read_text())


# ------------------------------------------------------------- R6 lengths ---
def _device_lengths(dist, seed, stream, step, rnd, ids, cuda):
    import ctypes as C
    from paper_2508_07970_b200._lib import check, lib
    d_ids = torch.as_tensor(np.asarray(ids, dtype=np.int64), device=cuda)
    out = torch.empty(len(ids), dtype=torch.int32, device=cuda)
    check(lib().yatt_sample_lengths_keyed(C.byref(dist.c()), seed, stream, step, rnd,
                                          d_ids.data_ptr(), len(ids), out.data_ptr(), None))
    return out.cpu().numpy()


def test_keyed_lengths_match_reference(cuda):
    g = load("lengths.json")
    for case in g["cases"]:
        d = case["dist"]
        dist = api.LengthDistribution(d["kind"], d["p1"], d["p2"], d["max_len"])
        got = _device_lengths(dist, g["seed"], g["stream"], g["step"], g["round"],
                              range(g["n"]), cuda)
        assert got.tolist() == case["lengths"], case["name"]


def _host_lengths(dist, seed, stream, step, rnd, ids):
    import ctypes as C
    from paper_2508_07970_b200._lib import check, lib
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    out = np.empty(len(ids), dtype=np.int32)
    check(lib().yatt_sample_lengths_host(C.byref(dist.c()), seed, stream, step, rnd,
                                         ids.ctypes.data, len(ids), out.ctypes.data))
    return out


def _uncertified(reset=True):
    import ctypes as C
    from paper_2508_07970_b200._lib import check, lib
    c = C.c_int64()
    check(lib().yatt_uncertified_draws(C.byref(c), int(reset)))
    return c.value


@pytest.mark.parametrize("kind,p1,p2,mx", [(api.NORMAL, 2048, 512, 4096),
                                           (api.LOGNORMAL, 5.0, 0.5, 4096),
                                           (api.UNIFORM, 1, 16384, 16384)])
def test_keyed_lengths_bulk_vs_oracle(cuda, kind, p1, p2, mx):
    """10^7 draws through the host-facing entry (device draws + glibc re-draw
    of the uncertified ones) == glibc for every id (keyed_draw.cuh)."""
    n = 10_000_000
    dist = api.LengthDistribution(kind, p1, p2, mx)
    got = _host_lengths(dist, 20250814, 2, 7, 1, np.arange(n, dtype=np.uint64))
    exp = O.sample_lengths_range(kind, p1, p2, mx, 20250814, 2, 7, 1, 0, n)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("kind,p1,p2", [(api.NORMAL, 2048, 512), (api.LOGNORMAL, 5.0, 0.5),
                                        (api.NORMAL, 300.5, 80)])
def test_keyed_lengths_adversarial_near_ties(cuda, kind, p1, p2):
    """Keys whose glibc value lands within 1e-9 (relative) of a .5 rounding
    tie, found by exhaustive search over 2x10^7 ids: the draws the device
    cannot certify.  The host-facing entry returns glibc's length for every
    one of them; the device-resident entry flags every one (counter)."""
    ids, found = O.near_ties(kind, p1, p2, 20250814, 2, 7, 1, 0, 20_000_000, 1e-9)
    assert found >= 1 and found == len(ids)
    dist = api.LengthDistribution(kind, p1, p2, 1 << 20)
    exp = [O.sample_length_keyed(kind, p1, p2, 1 << 20, 20250814, 2, 7, 1, int(i)) for i in ids]
    assert _host_lengths(dist, 20250814, 2, 7, 1, ids).tolist() == exp
    _uncertified(reset=True)
    _device_lengths(dist, 20250814, 2, 7, 1, ids.astype(np.int64), cuda)
    assert _uncertified(reset=True) == len(ids)


def test_forced_redraw_path_is_exact(cuda):
    """Widen the certification band so ~10% of Normal / LogNormal draws take
    the glibc re-draw + re-run path of the rounds engine: every golden
    rollout and 10^6 bulk draws stay bit-exact."""
    import ctypes as C
    from paper_2508_07970_b200._lib import check, lib
    check(lib().yatt_set_tie_band(C.c_double(0.05)))
    try:
        for name in ["normal", "lognormal_p3"]:
            case = load(f"rollout_{name}.json")
            params = _params(case)
            for run in case["runs"]:
                batch = _make_batch(case, run)
                rounds = api.run_rollout_rounds(batch, run["controllers"], params)
                assert [[_as_golden(r) for r in rnd] for rnd in rounds] == run["rounds"]
                assert [s.target_out_len_tokens for s in batch.samples] == run["final_out_len"]
        n = 1_000_000
        for kind, p1, p2 in [(api.NORMAL, 2048, 512), (api.LOGNORMAL, 5.0, 0.5)]:
            dist = api.LengthDistribution(kind, p1, p2, 4096)
            got = _host_lengths(dist, 3, 2, 0, 2, np.arange(n, dtype=np.uint64))
            assert np.array_equal(got, O.sample_lengths_range(kind, p1, p2, 4096, 3, 2, 0, 2, 0, n))
    finally:
        check(lib().yatt_set_tie_band(C.c_double(1e-9)))


def test_sample_lengths_statistics(cuda):
    # workload_test.cpp:28-57 known-answer style
    lengths = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 1024, 2048), 100000, 7)
    assert abs(np.mean(lengths) - 512.5) <= 0.02 * 512.5
    assert min(lengths) >= 1 and max(lengths) <= 1024


# ---------------------------------------------------------- R5 rejection ---
def test_rejection_matches_reference(cuda):
    g = load("rejection.json")
    batch = api.RolloutBatch(g["step"], [api.RolloutSample(g["id0"] + i, accepted=bool(a))
                                         for i, a in enumerate(g["accepted"])])
    for c in g["cases"]:
        cfg = api.RejectionConfig(c["rate"], bool(c["per_group"]), c["group_size"])
        got = api.rejection_process(batch, c["round"], cfg, 20250814)
        assert [int(x) for x in got] == c["flags"]


def test_rejection_invalid_config_throws(cuda):
    batch = api.RolloutBatch(0, [api.RolloutSample(i) for i in range(4)])
    with pytest.raises(ConfigError):
        api.rejection_process(batch, 1, api.RejectionConfig(1.0, False, 1), 1)
    with pytest.raises(ConfigError):
        api.rejection_process(batch, 1, api.RejectionConfig(0.5, True, 0), 1)


def test_group_mode_flags_whole_groups(cuda):
    # workload_test.cpp:110-119
    batch = api.RolloutBatch(0, [api.RolloutSample(i) for i in range(512)])
    rej = api.rejection_process(batch, 1, api.RejectionConfig(0.5, True, 8), 21)
    for g in range(0, 512, 8):
        assert len(set(rej[g:g + 8])) == 1


# ------------------------------------------------------- R3/R4 rollouts ---
def _make_batch(case, run):
    n = case["n"]
    return api.RolloutBatch(case["step"], [
        api.RolloutSample(case["step"] * n + i, run["prompt_len"][i]) for i in range(n)])


def _params(case):
    d = case["out_dist"]
    return api.RoundParams(api.LengthDistribution(d["kind"], d["p1"], d["p2"], d["max_len"]),
                           api.RejectionConfig(case["reject_rate"], bool(case["per_group"]),
                                               case["group_size"]),
                           case["seed"], case["mb"], case["max_rounds"])


def _as_golden(rep):
    return {"report": [rep.controller_rank, rep.round, rep.active_count, rep.newly_accepted_count,
                       rep.forced_accept_count, rep.pending_count, rep.accepted_score_tokens,
                       rep.accepted_train_units],
            "mbs": [x for m in rep.microbatches for x in (m.controller_rank, m.mb_index,
                                                          m.sample_count, m.max_out_len_tokens,
                                                          m.score_tokens)]}


@pytest.mark.parametrize("engine", ["rounds_engine", "per_launch"])
@pytest.mark.parametrize("name", ["config1", "config5", "normal", "lognormal_p3"])
def test_rollout_rounds_match_reference(cuda, name, engine):
    """Every round of every controller shard == the reference's per-shard
    shard_round_output loop, for P = 1/2/4/8 and misaligned P = 3: through the
    one-call rounds engine (rollout_rounds.cu) and through one device-resident
    launch per round (yatt_shard_round, the multi-rank building block)."""
    case = load(f"rollout_{name}.json")
    params = _params(case)
    run_fn = api.run_rollout_rounds if engine == "rounds_engine" else \
        api.run_rollout_rounds_per_launch
    for run in case["runs"]:
        batch = _make_batch(case, run)
        rounds = run_fn(batch, run["controllers"], params)
        assert [[_as_golden(r) for r in rnd] for rnd in rounds] == run["rounds"]
        assert [s.target_out_len_tokens for s in batch.samples] == run["final_out_len"]
        assert [int(s.accepted) for s in batch.samples] == run["final_accepted"]
        assert [s.accepted_round for s in batch.samples] == run["final_accepted_round"]


def test_feed_round_reduce_on_device(cuda):
    """yatt_reduce_round_reports == the integer sums of feed_round
    (simcore.cpp:304-311) over the golden per-round reports."""
    import ctypes as C
    from paper_2508_07970_b200._lib import ReportC, check, lib
    case = load("rollout_config5.json")
    for run in case["runs"]:
        for rnd in run["rounds"]:
            arr = (ReportC * len(rnd))()
            for i, r in enumerate(rnd):
                rk, ro, act, acc, forced, pend, score, units = r["report"]
                arr[i] = ReportC(rk, ro, act, acc, forced, pend, score, units, 0)
            d = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(cuda)
            out = torch.empty(6, dtype=torch.int64, device=cuda)
            check(lib().yatt_reduce_round_reports(d.data_ptr(), len(rnd), out.data_ptr(), None))
            pend = sum(r["report"][5] for r in rnd)
            assert out.cpu().tolist() == [sum(r["report"][2] for r in rnd), pend,
                                          sum(r["report"][4] for r in rnd),
                                          sum(r["report"][7] for r in rnd),
                                          sum(r["report"][6] for r in rnd), int(pend > 0)]


def test_shard_round_output_single_shard_api(cuda):
    case = load("rollout_config1.json")
    run = [r for r in case["runs"] if r["controllers"] == 2][0]
    batch = _make_batch(case, run)
    params = _params(case)
    shards = [api.make_shard_state(batch, 2, r) for r in range(2)]
    for rnd, golden in enumerate(run["rounds"], start=1):
        reps = [api.shard_round_output(s, rnd, params) for s in shards]
        assert [_as_golden(r) for r in reps] == golden


def test_shard_reports_integer_invariants(cuda):
    # simcore_test.cpp:322-340
    batch = api.RolloutBatch(0, [api.RolloutSample(i, 50) for i in range(10)])
    shard = api.make_shard_state(batch, 1, 0)
    params = api.RoundParams(api.LengthDistribution(api.NORMAL, 300, 80, 1024),
                             api.RejectionConfig(0.5, False, 1), 3, 16, 64)
    rep = api.shard_round_output(shard, 1, params)
    assert rep.active_count == 10
    assert rep.newly_accepted_count + rep.pending_count == 10
    assert sum(m.score_tokens for m in rep.microbatches) == \
        sum(s.prompt_len_tokens + s.out_len_tokens for s in shard.samples)
    with pytest.raises(ConfigError):
        api.shard_round_output(shard, 1, api.RoundParams(microbatch_size=0))


def test_max_rounds_forces_acceptance(cuda):
    # simcore_test.cpp:205-217
    batch = api.RolloutBatch(0, [api.RolloutSample(i, 64) for i in range(16)])
    params = api.RoundParams(api.LengthDistribution(api.CONSTANT, 100, 0, 1024),
                             api.RejectionConfig(0.9, False, 1), 3, 16, 3)
    rounds = api.run_rollout_rounds(batch, 1, params)
    assert len(rounds) == 3
    assert sum(r.forced_accept_count for rnd in rounds for r in rnd) >= 1
    assert all(s.accepted and s.accepted_round <= 3 for s in batch.samples)


def test_reference_unit_tests_pass_against_b200_library(cuda):
    """The reference's own workload_test.cpp + balancer_test.cpp, compiled
    unchanged against include/yatt + libyatt_b200.so (oracle/Makefile)."""
    exe = ROOT / "oracle" / "_ref" / "reftests_b200"
    assert exe.exists(), "build with `make -C oracle ref` (done by __graft_entry__.build)"
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "0 failed" in res.stdout


def test_reference_step_tests_pass_against_b200_library(cuda):
    """The reference's simcore_test.cpp (18 TESTs: exact prep/train charges,
    rejection rounds + swap law, max_rounds, TraceIsIndependentOfController-
    Count :219, probe == first round :246, ShardReportsAreIntegerOnly :322,
    invalid contexts) compiled unchanged at the real call site: run_rlhf_step
    from dropin/run_rlhf_step.cpp (all rounds of all shards in one device
    call), shard_round_output / make_shard_state from libyatt_b200.so, the
    reference's own timing layer (oracle/Makefile simcore_b200)."""
    exe = ROOT / "oracle" / "_ref" / "simcore_b200"
    assert exe.exists(), "build with `make -C oracle ref` (done by __graft_entry__.build)"
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "18 tests, 0 failed" in res.stdout


def test_reference_runner_traces_byte_identical(cuda, tmp_path):
    """The reference's own runner end to end (runner.cpp run_scenario ->
    make_step_batch -> run_rlhf_step, :152-166, :240-241) over its built-in
    scenarios table1 (50 steps), sweep and demo: trace.csv, summary.json and
    scenario.json from the drop-in build (oracle/_ref/runner_b200: every
    round of every shard on the B200) are byte-identical to the reference's
    own (runner_ref) — acceptance criterion 11 (acceptance_test.cpp:609-628)
    across implementations."""
    exes = {k: ROOT / "oracle" / "_ref" / f"runner_{k}" for k in ("ref", "b200")}
    for exe in exes.values():
        assert exe.exists(), "build with `make -C oracle ref` (done by __graft_entry__.build)"
    outs = {}
    for k, exe in exes.items():
        out = tmp_path / k
        res = subprocess.run([str(exe), str(out)], capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
        outs[k] = out
    files = sorted(p.relative_to(outs["ref"]) for p in outs["ref"].rglob("*") if p.is_file())
    assert len(files) == 9, files
    for f in files:
        a, b = (outs["ref"] / f).read_bytes(), (outs["b200"] / f).read_bytes()
        assert a == b, f"{f} differs"


def test_reference_acceptance_suite_passes_against_b200_library(cuda):
    """The reference's scenario-level suites compiled unchanged — its 11
    acceptance criteria (acceptance_test.cpp: :64 rollout totals across
    rejection rates, :130 swap-count law, :371 balancer waste and bias, :609
    byte-identical traces, ...) plus runner_test, controller_test and
    scenario_test, 38 TESTs — with the on-path functions (run_rlhf_step ->
    every round of every shard, sort_and_bucket, sample_length_keyed, ...)
    from the drop-in (oracle/Makefile accept_b200).  Each criterion's report
    line equals the reference-only build's (accept_ref) once wall-clock
    seconds are masked."""
    import re
    outs = {}
    for k in ("ref", "b200"):
        exe = ROOT / "oracle" / "_ref" / f"accept_{k}"
        assert exe.exists(), "build with `make -C oracle ref` (done by __graft_entry__.build)"
        res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
        assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
        assert "38 tests, 0 failed" in res.stdout
        outs[k] = [re.sub(r"\d+\.\d+ s\b", "<t> s", ln) for ln in res.stdout.splitlines()
                   if ln.startswith("[CRITERION")]
    assert len(outs["b200"]) == 11 and all("] PASS - " in ln for ln in outs["b200"]), outs["b200"]
    assert outs["b200"] == outs["ref"]


# ---------------------------------------------------------------- R10 ----
def test_sort_order_matches_oracle(cuda):
    rng = np.random.default_rng(0)
    for n in [0, 1, 7, 4096, 4097, 100_000]:
        lengths = rng.integers(-5, 300, size=n).astype(np.int32)  # heavy ties, negatives
        got = ops.sort_order_desc(torch.as_tensor(lengths, device=cuda)).cpu().numpy()
        assert got.astype(np.uint32).tolist() == O.sort_order_desc(lengths).tolist()


def test_sort_and_bucket_matches_reference(cuda):
    """Device sort + host std::shuffle == balancer::sort_and_bucket exactly."""
    for c in load("buckets.json")["cases"]:
        plan = api.sort_and_bucket(c["lengths"], c["B"], c["seed"])
        flat = [i for b in plan.buckets for i in b]
        assert flat == c["flat"]
        assert [0] + np.cumsum([len(b) for b in plan.buckets]).tolist() == c["offsets"]
        assert api.padding_waste(plan, c["lengths"]) == pytest.approx(c["waste"], abs=1e-15)
    with pytest.raises(ConfigError):
        api.sort_and_bucket([1, 2, 3], 0, 1)
    assert api.waste_bound(16) == 0.12109375


# ------------------------------------------------------------ A5 / A6 ----
def _config5_batch(cuda, token_scale=16384, n_prompts=1024, G=16, seed=20250814):
    n = n_prompts * G
    dist = api.LengthDistribution(api.UNIFORM, 1, token_scale, token_scale)
    resp = _device_lengths(dist, seed, 2, 1, 1, range(n), cuda).astype(np.int64)
    lens = resp + 64  # prompt 64 (configs[4])
    rewards = ops.synth_floats(seed, 105, 0, n, "reward", G, device=cuda)
    return n, G, lens, rewards


@pytest.mark.parametrize("token_scale", [512, 16384])
def test_filter_compact_matches_oracle(cuda, token_scale):
    n, G, lens, rewards = _config5_batch(cuda, token_scale)
    d_lens = torch.as_tensor(lens, device=cuda)
    out = ops.filter_compact(rewards, d_lens, G)
    exp = O.filter_compact(rewards.cpu().numpy(), lens, G)
    k = int(exp["counts"][0])
    assert out["counts"].cpu().numpy().tolist() == exp["counts"].tolist()
    assert out["keep_groups"].cpu().numpy().tolist() == exp["keep_groups"].tolist()
    assert out["index_map"][:k].cpu().numpy().tolist() == exp["index_map"].tolist()
    assert out["new_cu"][:k + 1].cpu().numpy().tolist() == exp["new_cu"].tolist()
    assert 0 < k < n  # both kinds of group present

    # gather the per-token payload (token ids i32, logp f32, mask u8)
    old_cu = torch.zeros(n + 1, dtype=torch.int64, device=cuda)
    old_cu[1:] = torch.cumsum(d_lens, 0)
    total = int(old_cu[-1])
    tok = torch.randint(0, 152064, (total,), dtype=torch.int32, device=cuda)
    lp = torch.randn(total, device=cuda)
    mk = (torch.arange(total, device=cuda) % 3 != 0).to(torch.uint8)
    kept_tokens = int(exp["counts"][1])
    np_old_cu = old_cu.cpu().numpy()
    idx = np.concatenate([np.arange(np_old_cu[s], np_old_cu[s + 1]) for s in exp["index_map"]])
    for src in (tok, lp, mk):
        dst = torch.empty(kept_tokens, dtype=src.dtype, device=cuda)
        ops.gather_varlen(src, old_cu, out["index_map"], out["new_cu"], out["counts"][:1], n, dst)
        assert torch.equal(dst.cpu(), src.cpu()[torch.from_numpy(idx)])

    # multimodal payload refs: 4 x int64 per sample, remapped by the index map
    refs = torch.arange(n * 4, dtype=torch.int64, device=cuda).view(n, 4)
    rdst = torch.empty((k, 4), dtype=torch.int64, device=cuda)
    ops.gather_rows(refs, out["index_map"], out["counts"][:1], n, rdst)
    assert torch.equal(rdst.cpu(), refs.cpu()[torch.from_numpy(exp["index_map"]).long()])


def test_filter_compact_edge_cases(cuda):
    G = 4
    lens = torch.full((8,), 3, dtype=torch.int64, device=cuda)
    # all groups zero-variance -> nothing kept
    r = torch.ones(8, device=cuda)
    out = ops.filter_compact(r, lens, G)
    assert out["counts"].cpu().tolist() == [0, 0, 0]
    assert int(out["new_cu"][0]) == 0
    # all kept
    r = torch.tensor([0, 1, 0, 0, 1, 1, 0, 1], dtype=torch.float32, device=cuda)
    out = ops.filter_compact(r, lens, G)
    assert out["counts"].cpu().tolist() == [8, 24, 2]
    # empty batch
    e = ops.filter_compact(torch.empty(0, device=cuda), torch.empty(0, dtype=torch.int64,
                                                                      device=cuda), G)
    assert e["counts"].cpu().tolist() == [0, 0, 0]
    # a trailing partial group (n % G != 0) is a group of its own
    # (group = sample_id / G, workload.cpp:158-160); a lone sample is zero-variance
    for r_list in ([1, 1, 1, 1, 2, 3], [1, 2, 1, 1, 5, 5, 5], [0, 1, 0, 0, 7],
                   [3, 3, 3, 3, 1, 2, 2, 2, 9]):
        r = torch.tensor(r_list, dtype=torch.float32, device=cuda)
        ln = torch.arange(1, len(r_list) + 1, dtype=torch.int64, device=cuda)
        out = ops.filter_compact(r, ln, G)
        exp = O.filter_compact(r.cpu().numpy(), ln.cpu().numpy(), G)
        k = int(exp["counts"][0])
        assert out["counts"].cpu().tolist() == exp["counts"].tolist(), r_list
        assert np.array_equal(out["keep_groups"].cpu().numpy(), exp["keep_groups"]), r_list
        assert np.array_equal(out["index_map"][:k].cpu().numpy(), exp["index_map"]), r_list
        assert np.array_equal(out["new_cu"][:k + 1].cpu().numpy(), exp["new_cu"]), r_list
    with pytest.raises(ConfigError):
        ops.filter_compact(torch.ones(6, device=cuda), torch.ones(6, dtype=torch.int64,
                                                                 device=cuda), 0)


def test_microbatch_aggregates_over_survivors(cuda):
    n, G, lens, rewards = _config5_batch(cuda, 512, 64)
    out = ops.filter_compact(rewards, torch.as_tensor(lens, device=cuda), G)
    k = int(out["counts"][0])
    imap = out["index_map"][:k].long()
    plen = torch.full((n,), 64, dtype=torch.int32, device=cuda)
    olen = torch.as_tensor(lens - 64, dtype=torch.int32, device=cuda)
    p_k, o_k = plen[imap].contiguous(), olen[imap].contiguous()
    mbs = ops.microbatch_aggregates(p_k, o_k, 16, controller_rank=3).cpu().numpy()
    o = o_k.cpu().numpy()
    for j in range(-(-k // 16)):
        sl = slice(16 * j, min(k, 16 * j + 16))
        score = int(mbs[j, 4]) | (int(mbs[j, 5]) << 32)
        assert mbs[j, :4].tolist() == [3, j, sl.stop - sl.start, int(o[sl].max())]
        assert score == int(64 * (sl.stop - sl.start) + o[sl].sum())


def test_global_compaction_across_emulated_ranks(cuda):
    """P ranks compact their group-aligned shards; all-gathered counts ->
    exclusive offsets -> one global packed layout identical to P = 1."""
    n, G, lens, rewards = _config5_batch(cuda, 256, 128)
    d_lens = torch.as_tensor(lens, device=cuda)
    single = ops.filter_compact(rewards, d_lens, G)
    kt = int(single["counts"][1])
    P = 4
    outs, counts = [], []
    for r in range(P):
        s = api.shard_dataset(n // G, P, r)
        sl = slice(s.begin * G, s.end * G)
        o = ops.filter_compact(rewards[sl].contiguous(), d_lens[sl].contiguous(), G)
        outs.append((sl, o))
        counts.append(o["counts"])
    gathered = torch.cat(counts)  # stands in for yatt_comm_allgather_i64
    payload = torch.arange(int(d_lens.sum()), dtype=torch.int32, device=cuda)
    cu_all = torch.zeros(n + 1, dtype=torch.int64, device=cuda)
    cu_all[1:] = torch.cumsum(d_lens, 0)
    dst = torch.full((kt,), -1, dtype=torch.int32, device=cuda)
    for r, (sl, o) in enumerate(outs):
        off = ops.exclusive_offset(gathered, P, r, 3, 1)
        local_cu = (cu_all[sl.start:sl.stop + 1] - cu_all[sl.start]).contiguous()
        src = payload[int(cu_all[sl.start]):int(cu_all[sl.stop])].contiguous()
        ops.gather_varlen(src, local_cu, o["index_map"], o["new_cu"], o["counts"][:1],
                          sl.stop - sl.start, dst, off)
    ref = torch.empty(kt, dtype=torch.int32, device=cuda)
    ops.gather_varlen(payload, cu_all, single["index_map"], single["new_cu"],
                      single["counts"][:1], n, ref)
    assert torch.equal(dst, ref)


@pytest.mark.parametrize("esz", [1, 2, 4, 8])
def test_gather_varlen_every_relative_alignment(cuda, esz):
    """Byte-exact gather for every (src, dst) misalignment mod 16 and lengths
    around the 16-byte / 512-byte / 8-KB copy granules; a dst_offset shifts
    the destination base too."""
    rng = np.random.default_rng(esz)
    lens = np.concatenate([np.arange(0, 40), [511, 512, 513, 2047, 2048, 2049, 8191, 8193, 70001],
                           rng.integers(0, 3000, size=200)]).astype(np.int64)
    n = len(lens)
    old_cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    total = int(old_cu[-1])
    src = torch.randint(0, 256, (total * esz + 64,), dtype=torch.uint8, device=cuda)
    keep = rng.random(n) < 0.7
    idx = np.nonzero(keep)[0].astype(np.int32)
    kl = lens[idx]
    new_cu = np.concatenate([[0], np.cumsum(kl)]).astype(np.int64)
    for src_shift, off in [(0, 0), (esz, 3), (3 * esz, 1), (7 * esz, 5)]:
        s = src[src_shift: src_shift + total * esz]
        dst = torch.zeros(((int(new_cu[-1]) + off) * esz + 32,), dtype=torch.uint8, device=cuda)
        d_off = torch.tensor([off], dtype=torch.int64, device=cuda)
        nk = torch.tensor([len(idx)], dtype=torch.int64, device=cuda)
        from paper_2508_07970_b200._lib import check, lib
        d_old, d_idx, d_new = (torch.as_tensor(a, device=cuda) for a in (old_cu, idx, new_cu))
        check(lib().yatt_gather_varlen(
            s.data_ptr(), d_old.data_ptr(), d_idx.data_ptr(), d_new.data_ptr(), nk.data_ptr(), n,
            d_off.data_ptr(), esz, dst.data_ptr(), torch.cuda.current_stream().cuda_stream))
        hs = s.cpu().numpy()
        want = np.concatenate([hs[old_cu[i] * esz: old_cu[i + 1] * esz] for i in idx])
        got = dst.cpu().numpy()
        assert np.array_equal(got[off * esz: off * esz + len(want)], want)
        assert not got[: off * esz].any() and not got[off * esz + len(want):].any()


@pytest.mark.parametrize("row_bytes,shift", [(32, 0), (24, 8), (12, 4), (7, 1), (48, 16)])
def test_gather_rows_widths(cuda, row_bytes, shift):
    n = 1000
    buf = torch.randint(0, 256, (n * row_bytes + shift,), dtype=torch.uint8, device=cuda)
    src = buf[shift:]
    idx = np.nonzero(np.random.default_rng(row_bytes).random(n) < 0.6)[0].astype(np.int32)
    out = torch.zeros((len(idx) * row_bytes,), dtype=torch.uint8, device=cuda)
    from paper_2508_07970_b200._lib import check, lib
    nk = torch.tensor([len(idx)], dtype=torch.int64, device=cuda)
    d_idx = torch.as_tensor(idx, device=cuda)
    check(lib().yatt_gather_rows(src.data_ptr(), d_idx.data_ptr(),
                                 nk.data_ptr(), n, row_bytes, None, out.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream))
    want = src.cpu().numpy().reshape(n, row_bytes)[idx].reshape(-1)
    assert np.array_equal(out.cpu().numpy(), want)


def test_gather_varlen_multi_matches_single(cuda):
    """The fused five-array gather (17 B/token payload) == five single gathers."""
    rng = np.random.default_rng(11)
    n, G = 4096, 16
    lens = torch.as_tensor(rng.integers(1, 700, size=n), device=cuda)
    rw = ops.synth_floats(3, 105, 0, n, "reward", G, device=cuda)
    plan = ops.filter_compact(rw, lens, G)
    old_cu = torch.zeros(n + 1, dtype=torch.int64, device=cuda)
    old_cu[1:] = torch.cumsum(lens, 0)
    tot, kt = int(old_cu[-1]), int(plan["counts"][1])
    srcs = [torch.randint(-2**31, 2**31 - 1, (tot,), dtype=torch.int32, device=cuda),
            torch.randn(tot, device=cuda), torch.randn(tot, device=cuda),
            torch.randn(tot, device=cuda),
            torch.randint(0, 2, (tot,), dtype=torch.uint8, device=cuda)]
    off = torch.tensor([5], dtype=torch.int64, device=cuda)
    fused = [torch.zeros(kt + 5, dtype=t.dtype, device=cuda) for t in srcs]
    single = [torch.zeros(kt + 5, dtype=t.dtype, device=cuda) for t in srcs]
    ops.gather_varlen_multi(srcs, old_cu, plan["index_map"], plan["new_cu"], plan["counts"][:1], n,
                            fused, off)
    for s_, d_ in zip(srcs, single):
        ops.gather_varlen(s_, old_cu, plan["index_map"], plan["new_cu"], plan["counts"][:1], n, d_,
                          off)
    for a, b in zip(fused, single):
        assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))
    with pytest.raises(ConfigError):
        ops.gather_varlen_multi(srcs * 2, old_cu, plan["index_map"], plan["new_cu"],
                                plan["counts"][:1], n, fused * 2)


# ----------------------------------------------- groups straddling ranks ----
@pytest.mark.parametrize("P", [3, 7])
def test_straddling_groups_emulated_ranks(cuda, P):
    """The reference's SAMPLE-level shard_dataset (workload.cpp:183-198) over
    configs[4]'s 1,024 x 16 samples at P = 3 / 7 splits groups across ranks.
    Each emulated rank writes its boundary records, the records are stacked
    in rank order (what the all-gather delivers), and every rank's sharded
    filter + GRPO merge run on its own slice: the global compaction layout is
    byte-identical to one rank's and the advantages match to 1e-12."""
    n, G, lens_np, rew = _config5_batch(cuda, token_scale=512)
    lens = torch.as_tensor(lens_np, device=cuda)
    single = ops.filter_compact(rew, lens, G)
    adv_one = ops.grpo_advantages(rew, G)
    shards = [api.shard_dataset(n, P, r) for r in range(P)]
    assert any(s.begin % G for s in shards)  # some group really straddles
    frecs = torch.stack([ops.filter_boundary_record(rew[s.begin:s.end].contiguous(), G, s.begin)
                         for s in shards]).view(-1)
    moms = [ops.grpo_group_moments(rew[s.begin:s.end].contiguous(), G, s.begin) for s in shards]
    grecs = torch.stack([ops.grpo_boundary_record(m, s.size(), G, s.begin)
                         for m, s in zip(moms, shards)]).view(-1)
    cu = torch.zeros(n + 1, dtype=torch.int64, device=cuda)
    cu[1:] = torch.cumsum(lens, 0)
    payload = torch.arange(int(cu[-1]), dtype=torch.int32, device=cuda)
    kt = int(single["counts"][1])
    dst = torch.full((kt,), -1, dtype=torch.int32, device=cuda)
    off = torch.zeros(3, dtype=torch.int64, device=cuda)
    kept_groups = 0
    for s, m in zip(shards, moms):
        sl = slice(s.begin, s.end)
        loc = ops.filter_compact(rew[sl].contiguous(), lens[sl].contiguous(), G, s.begin, frecs, P)
        lcu = (cu[s.begin:s.end + 1] - cu[s.begin]).contiguous()
        ops.gather_varlen(payload[int(cu[s.begin]):int(cu[s.end])].contiguous(), lcu,
                          loc["index_map"], loc["new_cu"], loc["counts"][:1], s.size(), dst,
                          off[1:2].clone())
        off += loc["counts"]
        kept_groups += int(loc["counts"][2])
        ops.grpo_merge_boundaries(m, s.size(), G, s.begin, grecs)
        adv = ops.grpo_advantages(rew[sl].contiguous(), G, first_sample_id=s.begin, moments=m)
        assert torch.allclose(adv.double(), adv_one[sl].double(), rtol=1e-12, atol=1e-12)
    ref = torch.empty(kt, dtype=torch.int32, device=cuda)
    ops.gather_varlen(payload, cu, single["index_map"], single["new_cu"], single["counts"][:1], n,
                      ref)
    assert off.tolist() == single["counts"].tolist()
    assert kept_groups == int(single["counts"][2])
    assert torch.equal(dst, ref)


def test_straddle_python_layer_validates_shapes(cuda):
    """The Python straddle helpers refuse tables that do not cover the shard
    (the C ABI would read / write moments rows 0 .. ng-1 of them)."""
    r = torch.zeros(20, device=cuda)
    mom = ops.grpo_group_moments(r, 8, 4)           # ids 4..23: 3 local groups
    assert mom.shape == (3, 3)
    with pytest.raises(ValueError, match="groups"):
        ops.grpo_boundary_record(mom[:2].contiguous(), 20, 8, 4)
    rec = ops.grpo_boundary_record(mom, 20, 8, 4)
    with pytest.raises(ValueError, match="8 doubles"):
        ops.grpo_merge_boundaries(mom, 20, 8, 4, rec[:5].contiguous())
    with pytest.raises(TypeError):
        ops.grpo_merge_boundaries(mom.float(), 20, 8, 4, rec)
    ops.grpo_merge_boundaries(mom, 20, 8, 4, rec)     # one rank: its own record
    torch.cuda.synchronize()
