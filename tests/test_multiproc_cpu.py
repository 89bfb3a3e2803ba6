"""N>1 host-side logic on CPU: world_size-2 gloo processes run the per-rank
experience step (CPU oracle standing in for the kernels) over their prompt-
group shards and reduce exactly like bench.py / ranks.py do on NCCL.

Checks: (1) all-reduced loss sums == single-process sums, (2) all-gathered
survivor counts -> exclusive offsets give the single-process packed layout,
(3) groups split across ranks (misaligned shard) get single-rank advantages
after the boundary-moment merge.  Mirrors the reference's controller-count
invariance test (proj/tests/simcore_test.cpp:219-244)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

P, R, T, V, SEED = 8, 4, 16, 512, 20250814


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _full_batch():
    rows = P * R * T
    pol, ref, tgt = O.synth_logits(SEED, 0, rows, V)
    rewards = O.synth_floats(SEED, 105, 0, P * R, "reward", R)
    old_delta = O.synth_floats(SEED, 104, 0, rows, "old_delta")
    return pol, ref, tgt, rewards, old_delta


def _rank_sums(g0, g1):
    pol, ref, tgt, rewards, old_delta = _full_batch()
    sl = slice(g0 * R * T, g1 * R * T)
    st = O.token_stats(pol[sl], ref[sl], tgt[sl], None, "k3", threads=1)
    adv = O.grpo_advantages(rewards[g0 * R:g1 * R], R, 1e-6, True, g0 * R)
    tadv = np.repeat(adv, T).astype(np.float32)
    old = (st[0] + old_delta[sl]).astype(np.float32)
    return O.policy_loss(st[0], old, tadv, st[3], st[2])


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_07970_b200 import ranks
    g0, g1 = ranks.shard_groups(P, world, rank)
    sums = torch.from_numpy(_rank_sums(g0, g1))
    ranks.allreduce_sums(sums)
    # dynamic sampling: local compaction, global offsets
    _, _, _, rewards, _ = _full_batch()
    lens = np.full(P * R, T, dtype=np.int64)
    loc = O.filter_compact(rewards[g0 * R:g1 * R], lens[g0 * R:g1 * R], R)
    counts = ranks.allgather_counts(torch.from_numpy(loc["counts"]))
    tok_off = int(counts.view(world, 3)[:rank, 1].sum())
    smp_off = int(counts.view(world, 3)[:rank, 0].sum())
    packed = (loc["new_cu"][:-1] + tok_off).tolist()
    gidx = (loc["index_map"] + g0 * R + 0 * smp_off).tolist()
    gathered = [None] * world
    dist.all_gather_object(gathered, (smp_off, packed, gidx))
    # misaligned shard of samples (not groups): boundary-moment merge
    n = P * R
    b = rank * (n // world) + (3 if rank else 0)  # split inside a group
    e = (rank + 1) * (n // world) + (3 if rank + 1 < world else 0)
    r = rewards[b:e]
    first = b // R
    local = torch.zeros((((e - 1) // R) - first + 1, 3), dtype=torch.float64)
    for k in range(local.shape[0]):
        g = first + k
        lo, hi = max(g * R, b), min((g + 1) * R, e)
        x = r[lo - b:hi - b].astype(np.float64)
        mean = x.sum() / len(x)
        local[k] = torch.tensor([len(x), mean, ((x - mean) ** 2).sum()])
    bnd = [None] * world
    dist.all_gather_object(bnd, (first, local[0].tolist(), first + local.shape[0] - 1,
                                 local[-1].tolist()))
    merged = ranks.merged_boundary_moments(local, first, bnd)
    if rank == 0:
        out.put(("sums", sums.numpy().tolist()))
        out.put(("packed", gathered))
    out.put(("moments", rank, b, merged.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_step_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=300) for _ in range(2 + world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = {m[0]: m for m in msgs if m[0] != "moments"}
    single = _rank_sums(0, P)
    assert np.allclose(got["sums"][1], single, rtol=1e-12, atol=0)

    _, _, _, rewards, _ = _full_batch()
    full = O.filter_compact(rewards, np.full(P * R, T, dtype=np.int64), R)
    packed = [x for (_, pk, _) in got["packed"][1] for x in pk]
    gidx = [x for (_, _, gi) in got["packed"][1] for x in gi]
    assert packed == full["new_cu"][:-1].tolist()
    assert gidx == full["index_map"].tolist()

    full_mom = {}
    for g in range(P):
        x = rewards[g * R:(g + 1) * R].astype(np.float64)
        full_mom[g] = (len(x), x.mean(), ((x - x.mean()) ** 2).sum())
    for m in msgs:
        if m[0] != "moments":
            continue
        _, rank, b, table = m
        for k, row in enumerate(table):
            exp = full_mom[b // R + k]
            assert np.allclose(row, exp, rtol=1e-12, atol=1e-12)
