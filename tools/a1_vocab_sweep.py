"""A1 throughput across vocabularies (8,192 .. 152,064) and row counts, CUDA
events, L2 flushed between launches: the per-row overhead at small V."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_07970_b200 import ops
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for rows, V in [(32768, 32000), (16384, 32000), (8192, 152064), (32768, 152064), (65536, 8192), (32768, 128256)]:
    pol, ref, tgt = ops.synth_logits(1, 0, rows, V, device=dev)
    out = torch.empty((4, rows), device=dev)
    for _ in range(3): ops.token_stats(pol, ref, tgt, None, "k3", out=out)
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ops.token_stats(pol, ref, tgt, None, "k3", out=out); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort(); ms = ts[len(ts)//2]
    print(rows, V, round(ms, 3), "ms", round(rows * (4 * V + 21) / ms / 1e6), "GB/s")
    del pol, ref, tgt
