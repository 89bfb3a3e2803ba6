"""A peer that never arrives must not hang the others: rank 0 calls the
peer all-reduce and all-gather, rank 1 never does.  After ~10 s the kernels
give up, write NaN / -1 and set the status word (yatt_peer_status == 1);
rank 0 then reports and both exit.  World 2 on one GPU, gloo plumbing.
Run: torchrun --nproc-per-node 2 tools/peer_timeout_check.py -> "peer timeout ok"."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2508_07970_b200 import ranks  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(0)
    peer = ranks.PeerGroup(2, rank)
    dist.barrier()
    if rank == 0:
        t0 = time.time()
        y = peer.allreduce_f64(torch.ones(4, dtype=torch.float64, device="cuda"))
        g = peer.allgather_i64(torch.arange(5, dtype=torch.int64, device="cuda"))
        torch.cuda.synchronize()
        dt = time.time() - t0
        assert torch.isnan(y).all(), y
        assert torch.all(g == -1), g
        assert peer.status() == 1
        print(f"peer timeout ok: both calls returned after {dt:.1f} s with NaN / -1, status 1",
              flush=True)
    dist.barrier()  # rank 1 waits here (gloo, host side) without calling the kernel
    peer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
