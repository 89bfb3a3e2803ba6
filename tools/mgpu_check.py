"""Multi-GPU check of the rank-level path (run under torchrun, N >= 2).

Each rank owns prompt groups shard_groups(16, N, r) of a config-1-shaped
GRPO batch (16 prompts x 8 responses, T=256, V=32000) and runs
A1 -> A2 -> broadcast -> A4 on its own GPU; the loss sums are all-reduced
through the C-ABI NCCL communicator (yatt_comm_*).  Dynamic-sampling
compaction uses yatt_comm_allgather_i64 + yatt_exclusive_offset to write one
global packed layout.  Both must equal the single-GPU result bit for bit
(sums: up to fp64 reassociation).  Prints "mgpu ok" on success.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2508_07970_b200 import ops, ranks  # noqa: E402

P, R, T, V, SEED = 16, 8, 256, 32000, 20250814


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


def step(g0, g1, dev):
    rows = (g1 - g0) * R * T
    pol, ref, tgt = ops.synth_logits(SEED, g0 * R * T, rows, V, device=dev)
    logp, rlogp, ent, kl = ops.token_stats(pol, ref, tgt, None, "k3")
    rewards = ops.synth_floats(SEED, 105, g0 * R, (g1 - g0) * R, "reward", R, device=dev)
    adv = ops.grpo_advantages(rewards, R, 1e-6, True, g0 * R)
    cu = torch.arange((g1 - g0) * R + 1, dtype=torch.int64, device=dev) * T
    tadv = ops.broadcast_to_tokens(adv, cu, rows)
    old = ops.synth_floats(SEED, 104, g0 * R * T, rows, "old_delta", base=logp, device=dev)
    return ops.policy_loss(logp, old, tadv, kl, ent), rewards


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    uid = [ranks.YattComm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = ranks.YattComm(world, rank, uid[0])

    # collectives sanity
    x = torch.full((5,), float(rank + 1), dtype=torch.float64, device=dev)
    comm.allreduce_(x)
    assert torch.all(x == world * (world + 1) / 2)
    c = torch.tensor([rank, 10 * rank], dtype=torch.int64, device=dev)
    g = comm.allgather(c)
    assert g.tolist() == [v for r in range(world) for v in (r, 10 * r)]

    # sharded GRPO experience step vs the full batch on one GPU
    g0, g1 = ranks.shard_groups(P, world, rank)
    sums, _ = step(g0, g1, dev)
    comm.allreduce_(sums)
    full, rewards_all = step(0, P, dev)
    torch.cuda.synchronize()
    rel = ((sums - full).abs() / (full.abs() + 1e-12)).max().item()
    assert rel <= 1e-12, (rank, rel, sums.tolist(), full.tolist())

    # global compaction across ranks
    lens_all = torch.full((P * R,), T, dtype=torch.int64, device=dev) + \
        torch.arange(P * R, dtype=torch.int64, device=dev) % 7
    single = ops.filter_compact(rewards_all, lens_all, R)
    loc = ops.filter_compact(rewards_all[g0 * R:g1 * R].contiguous(),
                             lens_all[g0 * R:g1 * R].contiguous(), R)
    counts = comm.allgather(loc["counts"])
    off = ops.exclusive_offset(counts, world, rank, 3, 1)
    cu_all = torch.zeros(P * R + 1, dtype=torch.int64, device=dev)
    cu_all[1:] = torch.cumsum(lens_all, 0)
    payload = torch.arange(int(cu_all[-1]), dtype=torch.int32, device=dev)
    kt = int(single["counts"][1])
    dst = torch.zeros(kt, dtype=torch.int32, device=dev)
    local_cu = (cu_all[g0 * R:g1 * R + 1] - cu_all[g0 * R]).contiguous()
    src = payload[int(cu_all[g0 * R]):int(cu_all[g1 * R])].contiguous()
    ops.gather_varlen(src, local_cu, loc["index_map"], loc["new_cu"], loc["counts"][:1],
                      (g1 - g0) * R, dst, off)
    dist.all_reduce(dst)  # ranks wrote disjoint ranges into zero-initialised buffers
    ref = torch.empty(kt, dtype=torch.int32, device=dev)
    ops.gather_varlen(payload, cu_all, single["index_map"], single["new_cu"],
                      single["counts"][:1], P * R, ref)
    assert torch.equal(dst, ref)

    # dynamic-sampling rounds across real ranks: each rank runs its own shard,
    # reports travel as 48-byte structs over NCCL, the feed_round reduce runs
    # on the device; must equal the single-process loop over all shards
    import ctypes as C
    from paper_2508_07970_b200 import api
    from paper_2508_07970_b200._lib import ReportC, check, lib
    n_all = 2048
    params = api.RoundParams(api.LengthDistribution(api.UNIFORM, 1, 4096, 4096),
                             api.RejectionConfig(0.3, True, 8), SEED, 8, 5)
    mk = lambda: api.RolloutBatch(0, [api.RolloutSample(i, 64 + i % 13) for i in range(n_all)])  # noqa
    ref_rounds = api.run_rollout_rounds(mk(), world, params)
    peer = ranks.PeerGroup(world, rank)  # NVLink peer-memory collectives (below too)
    shard = api.make_shard_state(mk(), world, rank)
    ds = api._DeviceShards([shard], params, dev)
    off = (C.c_int64 * 2)(0, len(shard.samples))
    rnd = 0
    while True:
        rnd += 1
        check(lib().yatt_shard_round(ds.d.data_ptr(), off, 1, rank, 0, rnd, C.byref(params.c()),
                                     ds.d_rep.data_ptr(), ds.d_mbs.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream))
        reps, mbs, red = ranks.exchange_round_reports(ds.d_rep, ds.d_mbs, comm)
        # the same exchange as two peer-memory all-gather kernels: identical words
        preps, pmbs, pred = ranks.exchange_round_reports(ds.d_rep, ds.d_mbs, peer=peer)
        assert torch.equal(preps, reps) and torch.equal(pmbs, mbs) and torch.equal(pred, red)
        all_reps = (ReportC * world).from_buffer_copy(reps.cpu().numpy().tobytes())
        got = [(r.controller_rank, r.active_count, r.pending_count, r.accepted_train_units)
               for r in all_reps]
        exp = [(r.controller_rank, r.active_count, r.pending_count, r.accepted_train_units)
               for r in ref_rounds[rnd - 1]]
        assert got == exp, (rank, rnd, got, exp)
        assert int(red[1]) == sum(r.pending_count for r in ref_rounds[rnd - 1])
        if int(red[5]) == 0:  # continue flag decided on the device
            break
    assert rnd == len(ref_rounds)

    # loss reduction + all-reduce fused in one kernel over NVLink peer memory
    tri = world * (world + 1) / 2
    y = peer.allreduce_f64(torch.arange(1, 9, dtype=torch.float64, device=dev) * (rank + 1))
    assert torch.equal(y, torch.arange(1, 9, dtype=torch.float64, device=dev) * tri)
    outs = []
    for k in range(200):  # back-to-back: exercises the epoch-parity slot banks
        x = torch.full((3,), float(k * world + rank), dtype=torch.float64, device=dev)
        outs.append(peer.allreduce_f64(x))
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        assert torch.all(o == float(sum(k * world + r for r in range(world)))), (rank, k, o)
    li = loss_inputs(g0, g1, dev)
    fused = peer.policy_loss(*li)
    full, _ = step(0, P, dev)
    torch.cuda.synchronize()
    rel = ((fused - full).abs() / (full.abs() + 1e-12)).max().item()
    assert rel <= 1e-12, (rank, rel, fused.tolist(), full.tolist())
    # under CUDA-graph replay (the epoch lives on the device)
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
    for _ in range(5):
        gs.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(gs, fused), (rank, gs.tolist(), fused.tolist())
    # dynamic-sampling offsets in one kernel: == NCCL all-gather + exclusive_offset
    pre, tot = peer.scan_i64(loc["counts"])
    assert int(pre[1]) == int(ops.exclusive_offset(counts, world, rank, 3, 1)[0])
    assert tot.tolist() == counts.view(world, 3).sum(0).tolist()
    big = torch.arange(12000, dtype=torch.int64, device=dev) + 1000003 * rank
    gb = peer.allgather_i64(big).view(world, 12000)
    for q in range(world):
        assert torch.equal(gb[q], torch.arange(12000, dtype=torch.int64, device=dev) + 1000003 * q)
    assert peer.status() == 0
    # latency of the 8-double all-reduce: fused peer kernel vs NCCL (device time)
    x8 = torch.ones(8, dtype=torch.float64, device=dev)
    o8 = torch.empty_like(x8)
    res = {}
    r8 = torch.ones(8, dtype=torch.int64, device=dev)
    for name, fn in [("peer", lambda: peer.allreduce_f64(x8, o8)), ("nccl", lambda: comm.allreduce_(x8)),
                     ("peer_gather", lambda: peer.allgather_i64(r8)),
                     ("nccl_gather", lambda: comm.allgather(r8))]:
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(1000):
            fn()
        b.record()
        torch.cuda.synchronize()
        res[name] = a.elapsed_time(b)  # ms per 1000 = us per call
    if rank == 0:
        print(f"allreduce 8 x f64 per call: peer kernel {res['peer']:.2f} us, "
              f"NCCL {res['nccl']:.2f} us (world={world})")
        print(f"allgather 8 x i64 per rank per call: peer kernel {res['peer_gather']:.2f} us, "
              f"NCCL {res['nccl_gather']:.2f} us (world={world})")
    dist.barrier()
    peer.close()
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(f"mgpu ok world={world}")


if __name__ == "__main__":
    main()
