#!/usr/bin/env python3
"""Multi-rank dynamic-sampling step (configs[4]: 1,024 prompts x 16 = 16,384
samples, 4 rounds max, 30% per-group rejection), the batch's controller
shards on `world` ranks, two ways:

  per-round: the reference's protocol (demo.cpp:468-476) on the device — each
             round every rank runs its shard (yatt_shard_round), the reports
             are all-gathered over peer memory and reduced, the host reads
             the continue flag;
  one-exchange: PeerGroup.run_rollout_rounds — each rank's rounds in one
             persistent kernel, the reports travel once.

Median wall time per step (max over ranks; the Python batches are built
before the timed region; both paths include their host packing).
torchrun --nproc-per-node N tools/rounds_multirank_timing.py"""
import ctypes as C
import json
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2508_07970_b200 import api, ranks  # noqa: E402
from paper_2508_07970_b200._lib import check, lib  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    dev = torch.device("cuda", rank % ngpu)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    peer = ranks.PeerGroup(world, rank)
    n, G = 16384, 16
    params = api.RoundParams(api.LengthDistribution(api.UNIFORM, 1, 16384, 16384),
                             api.RejectionConfig(0.3, True, G), 20250814, 16, 4)
    mk = lambda: api.RolloutBatch(1, [api.RolloutSample(n + i, 64) for i in range(n)])  # noqa
    sr = api.shard_dataset(n, world, rank)

    def per_round(batch):
        shard = api.make_shard_state(batch, world, rank)
        ds = api._DeviceShards([shard], params, dev)
        off = (C.c_int64 * 2)(0, len(shard.samples))
        rnd = 0
        while True:
            rnd += 1
            check(lib().yatt_shard_round(ds.d.data_ptr(), off, 1, rank, 1, rnd,
                                         C.byref(params.c()), ds.d_rep.data_ptr(),
                                         ds.d_mbs.data_ptr(), torch.cuda.current_stream().cuda_stream))
            _, _, red = ranks.exchange_round_reports(ds.d_rep, ds.d_mbs, peer=peer)
            if int(red[5]) == 0 or rnd >= params.max_rounds:
                return rnd

    def one_exchange(batch):
        return len(peer.run_rollout_rounds(batch.samples[sr.begin:sr.end], 1, params, dev))

    out = {}
    for name, fn in (("per_round", per_round), ("one_exchange", one_exchange)):
        batches = [mk() for _ in range(18)]  # built outside the timed region
        for b in batches[:3]:
            fn(b)
        ts = []
        for b in batches[3:]:
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rounds = fn(b)
            torch.cuda.synchronize()
            t = torch.tensor([time.perf_counter() - t0])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ts.append(float(t) * 1e3)
        out[name] = {"ms_median": statistics.median(ts), "rounds": rounds}
    if rank == 0:
        print(json.dumps({"world": world, "gpus": ngpu, "samples": n, **out}), flush=True)
    peer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
