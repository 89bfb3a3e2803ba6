"""World-8 check of the NVLink peer-memory collectives on a box with fewer GPUs.

The driver's scaling run goes to 8 ranks, one per GPU; gpurun offers at most 4
GPUs, and NCCL refuses two ranks on one GPU.  This script oversubscribes:
rank r runs on GPU r % ngpus with gloo for the plumbing (handle exchange,
barriers), so the world-8 code of yatt_peer_* runs for real: 8 mapped IPC
buffers, 8-way rank-order sums, the epoch-parity slot banks, the scan.  Two
processes on one GPU time-slice (no MPS), so nothing here is timed.

Checks (vs single-process results, fixed rank order => bit-exact where the
math is exact):
  * allreduce_f64 of integer-valued doubles, 50 back-to-back calls;
  * scan_i64: exclusive prefix + total of per-rank counters;
  * policy_loss over 8 prompt-group shards == the full batch on one rank
    (max rel 1e-12: fp64 reassociation only);
  * the same under CUDA-graph replay;
  * groups straddling ranks (sample-level shard_dataset; world 3 / 7):
    GRPO advantages and the filter + compaction layout == one rank's;
  * global compaction: per-rank zero-variance filter + survivor counts scanned
    over peer memory -> one packed layout == the single-process compaction;
  * the all-gather (9,000 words per rank) and a full dynamic-sampling round
    loop whose reports travel only over peer memory == the single-process
    rounds (api.run_rollout_rounds).
Run: torchrun --nproc-per-node 8 tools/peer_world8.py   -> "peer world8 ok".
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2508_07970_b200 import ops, ranks  # noqa: E402

P, R, T, V, SEED = 16, 8, 64, 4096, 20250814


def loss_inputs(g0, g1, dev):
    rows = (g1 - g0) * R * T
    pol, ref, tgt = ops.synth_logits(SEED, g0 * R * T, rows, V, device=dev)
    logp, rlogp, ent, kl = ops.token_stats(pol, ref, tgt, None, "k3")
    rewards = ops.synth_floats(SEED, 105, g0 * R, (g1 - g0) * R, "reward", R, device=dev)
    adv = ops.grpo_advantages(rewards, R, 1e-6, True, g0 * R)
    cu = torch.arange((g1 - g0) * R + 1, dtype=torch.int64, device=dev) * T
    tadv = ops.broadcast_to_tokens(adv, cu, rows)
    old = ops.synth_floats(SEED, 104, g0 * R * T, rows, "old_delta", base=logp, device=dev)
    return logp, old, tadv, kl, ent


def main():
    dist.init_process_group("gloo")
    world, rank = dist.get_world_size(), dist.get_rank()
    ngpu = torch.cuda.device_count()
    torch.cuda.set_device(rank % ngpu)
    dev = torch.device("cuda", rank % ngpu)
    peer = ranks.PeerGroup(world, rank)

    tri = world * (world + 1) / 2
    y = peer.allreduce_f64(torch.arange(1, 9, dtype=torch.float64, device=dev) * (rank + 1))
    assert torch.equal(y, torch.arange(1, 9, dtype=torch.float64, device=dev) * tri), y
    outs = []
    for k in range(50):
        x = torch.full((5,), float(k * world + rank), dtype=torch.float64, device=dev)
        outs.append(peer.allreduce_f64(x))
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        assert torch.all(o == float(sum(k * world + r for r in range(world)))), (rank, k, o)

    cnt = torch.tensor([rank + 1, 2 * rank, 7], dtype=torch.int64, device=dev)
    pre, tot = peer.scan_i64(cnt)
    assert pre.tolist() == [sum(r + 1 for r in range(rank)), sum(2 * r for r in range(rank)),
                            7 * rank], pre
    assert tot.tolist() == [tri, world * (world - 1), 7 * world], tot

    g0, g1 = ranks.shard_groups(P, world, rank)
    li = loss_inputs(g0, g1, dev)
    fused = peer.policy_loss(*li)
    full = ops.policy_loss(*loss_inputs(0, P, dev))
    torch.cuda.synchronize()
    rel = ((fused - full).abs() / (full.abs() + 1e-12)).max().item()
    assert rel <= 1e-12, (rank, rel, fused.tolist(), full.tolist())

    ws = ops.LossWorkspace(dev)
    gs = torch.empty(8, dtype=torch.float64, device=dev)
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        peer.policy_loss(*li, workspace=ws, sums=gs)
    torch.cuda.current_stream().wait_stream(s_)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        peer.policy_loss(*li, workspace=ws, sums=gs)
    for _ in range(3):
        gs.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(gs, fused), (rank, gs.tolist(), fused.tolist())
    # global dynamic-sampling compaction: per-rank filter + survivor counts
    # scanned over peer memory (one kernel) give each rank its offsets into
    # ONE packed layout, byte-identical to the single-process compaction
    rewards_all = ops.synth_floats(SEED, 105, 0, P * R, "reward", R, device=dev)
    lens_all = torch.full((P * R,), T, dtype=torch.int64, device=dev) + \
        torch.arange(P * R, dtype=torch.int64, device=dev) % 7
    single = ops.filter_compact(rewards_all, lens_all, R)
    loc = ops.filter_compact(rewards_all[g0 * R:g1 * R].contiguous(),
                             lens_all[g0 * R:g1 * R].contiguous(), R)
    pre_c, tot_c = peer.scan_i64(loc["counts"])
    assert tot_c.tolist() == single["counts"].tolist(), (tot_c, single["counts"])
    cu_all = torch.zeros(P * R + 1, dtype=torch.int64, device=dev)
    cu_all[1:] = torch.cumsum(lens_all, 0)
    payload = torch.arange(int(cu_all[-1]), dtype=torch.int32, device=dev)
    kt = int(single["counts"][1])
    dst = torch.zeros(kt, dtype=torch.int32, device=dev)
    local_cu = (cu_all[g0 * R:g1 * R + 1] - cu_all[g0 * R]).contiguous()
    src = payload[int(cu_all[g0 * R]):int(cu_all[g1 * R])].contiguous()
    ops.gather_varlen(src, local_cu, loc["index_map"], loc["new_cu"], loc["counts"][:1],
                      (g1 - g0) * R, dst, pre_c[1:2].contiguous())
    ref_dst = torch.empty(kt, dtype=torch.int32, device=dev)
    ops.gather_varlen(payload, cu_all, single["index_map"], single["new_cu"],
                      single["counts"][:1], P * R, ref_dst)
    torch.cuda.synchronize()
    mine = dst.cpu()
    dist.all_reduce(mine)  # ranks wrote disjoint ranges of zero-initialised buffers
    assert torch.equal(mine, ref_dst.cpu()), rank

    # all-gather + the dynamic-sampling round loop with reports exchanged over
    # peer memory only == the single-process rounds
    big = torch.arange(9000, dtype=torch.int64, device=dev) + 1000003 * rank
    gb = peer.allgather_i64(big).view(world, 9000)
    for q in range(world):
        assert torch.equal(gb[q], torch.arange(9000, dtype=torch.int64, device=dev) + 1000003 * q)
    import ctypes as C
    from paper_2508_07970_b200 import api
    from paper_2508_07970_b200._lib import ReportC, check, lib
    params = api.RoundParams(api.LengthDistribution(api.UNIFORM, 1, 4096, 4096),
                             api.RejectionConfig(0.3, True, 8), SEED, 8, 5)
    mk = lambda: api.RolloutBatch(0, [api.RolloutSample(i, 64 + i % 13) for i in range(2048)])  # noqa
    ref_rounds = api.run_rollout_rounds(mk(), world, params)
    shard = api.make_shard_state(mk(), world, rank)
    ds = api._DeviceShards([shard], params, dev)
    off = (C.c_int64 * 2)(0, len(shard.samples))
    rnd = 0
    while True:
        rnd += 1
        check(lib().yatt_shard_round(ds.d.data_ptr(), off, 1, rank, 0, rnd, C.byref(params.c()),
                                     ds.d_rep.data_ptr(), ds.d_mbs.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream))
        reps, mbs, red = ranks.exchange_round_reports(ds.d_rep, ds.d_mbs, peer=peer)
        all_reps = (ReportC * world).from_buffer_copy(reps.cpu().numpy().tobytes())
        got = [(r.controller_rank, r.active_count, r.pending_count, r.accepted_train_units)
               for r in all_reps]
        exp = [(r.controller_rank, r.active_count, r.pending_count, r.accepted_train_units)
               for r in ref_rounds[rnd - 1]]
        assert got == exp, (rank, rnd, got, exp)
        if int(red[5]) == 0:
            break
    assert rnd == len(ref_rounds)
    # the same step with ONE exchange: every rank runs its shard's rounds to
    # completion in one persistent kernel, the reports travel once
    # (PeerGroup.run_rollout_rounds) — every field and microbatch of every
    # round == the single-process rounds, and the shard's final states too
    ref_batch = mk()
    ref_rounds = api.run_rollout_rounds(ref_batch, world, params)
    sr0 = api.shard_dataset(2048, world, rank)
    mine_s = mk().samples[sr0.begin:sr0.end]
    got_rounds = peer.run_rollout_rounds(mine_s, 0, params, dev)
    assert got_rounds == ref_rounds, (rank, len(got_rounds), len(ref_rounds))
    assert [(x.target_out_len_tokens, x.accepted, x.accepted_round) for x in mine_s] == \
        [(x.target_out_len_tokens, x.accepted, x.accepted_round)
         for x in ref_batch.samples[sr0.begin:sr0.end]], rank
    # a later step whose shards finish in different rounds (high rejection,
    # one rank's shard already accepted): zero reports pad the finished ones
    params_hi = api.RoundParams(api.LengthDistribution(api.NORMAL, 900, 300, 4096),
                                api.RejectionConfig(0.6, False, 1), SEED + 1, 4, 6)
    mk2 = lambda: api.RolloutBatch(3, [api.RolloutSample(3 * 512 + i, 32, accepted=(  # noqa
        api.shard_dataset(512, world, 0).begin <= i < api.shard_dataset(512, world, 0).end))
        for i in range(512)])
    ref_b2 = mk2()
    ref_r2 = api.run_rollout_rounds(ref_b2, world, params_hi)
    sr2 = api.shard_dataset(512, world, rank)
    mine2 = mk2().samples[sr2.begin:sr2.end]
    assert peer.run_rollout_rounds(mine2, 3, params_hi, dev) == ref_r2, rank
    assert [x.target_out_len_tokens for x in mine2] == \
        [x.target_out_len_tokens for x in ref_b2.samples[sr2.begin:sr2.end]], rank
    # groups straddling ranks: the reference's SAMPLE-level shard_dataset
    # (workload.cpp:183-198) of N = 16 x 8 samples; at world 3 / 7 groups of 8
    # split across ranks.  Advantages == one rank's (fp64 moments merged on
    # the device), filter + compaction layout byte-identical.
    n_all = P * R
    from paper_2508_07970_b200 import api
    sr = api.shard_dataset(n_all, world, rank)
    b, e = sr.begin, sr.end
    rew_all = ops.synth_floats(SEED, 105, 0, n_all, "reward", R, device=dev)
    mine = rew_all[b:e].contiguous()
    adv = peer.grpo_advantages(mine, R, b)
    adv_one = ops.grpo_advantages(rew_all, R)
    torch.cuda.synchronize()
    assert torch.allclose(adv.double(), adv_one[b:e].double(), rtol=1e-12, atol=1e-12), rank
    got = torch.zeros(n_all, dtype=torch.float32)
    got[b:e] = adv.cpu()
    dist.all_reduce(got)
    assert torch.equal(got, adv_one.cpu()), "straddle advantages"
    lens_all = torch.full((n_all,), T, dtype=torch.int64, device=dev) + \
        torch.arange(n_all, dtype=torch.int64, device=dev) % 5
    single2 = ops.filter_compact(rew_all, lens_all, R)
    loc2 = peer.filter_compact(mine, lens_all[b:e].contiguous(), R, b)
    pre2, tot2 = peer.scan_i64(loc2["counts"])
    assert tot2.tolist() == single2["counts"].tolist(), (tot2, single2["counts"])
    cu2 = torch.zeros(n_all + 1, dtype=torch.int64, device=dev)
    cu2[1:] = torch.cumsum(lens_all, 0)
    pay2 = torch.arange(int(cu2[-1]), dtype=torch.int32, device=dev)
    kt2 = int(single2["counts"][1])
    dst2 = torch.zeros(kt2, dtype=torch.int32, device=dev)
    lcu = (cu2[b:e + 1] - cu2[b]).contiguous()
    ops.gather_varlen(pay2[int(cu2[b]):int(cu2[e])].contiguous(), lcu, loc2["index_map"],
                      loc2["new_cu"], loc2["counts"][:1], e - b, dst2, pre2[1:2].contiguous())
    ref2 = torch.empty(kt2, dtype=torch.int32, device=dev)
    ops.gather_varlen(pay2, cu2, single2["index_map"], single2["new_cu"], single2["counts"][:1],
                      n_all, ref2)
    torch.cuda.synchronize()
    m2 = dst2.cpu()
    dist.all_reduce(m2)
    assert torch.equal(m2, ref2.cpu()), "straddle compaction"

    assert peer.status() == 0
    dist.barrier()
    peer.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(f"peer world{world} ok on {ngpu} GPUs")


if __name__ == "__main__":
    main()
