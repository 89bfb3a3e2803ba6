"""Sustained A1 throughput (power-capped steady state, like inside bench.py).

Streams 2 alternating resident 32,768-row chunks (V=152,064, 19.9 GB each)
through token_stats for `secs` seconds, times every launch with CUDA events
and reports the mean over the last 2/3 of the run, with nvidia-smi clocks.
Load an experiment build with YATT_B200_LIB=path/to/variant.so.
Prints one JSON line.
"""
import json
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import ClockSampler, bytes_per_row  # noqa: E402
from paper_2508_07970_b200 import ops  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
rows, V = 32768, 152064
bufs = [ops.synth_logits(20250814 + k, 0, rows, V) for k in range(2)]
mask = torch.ones(rows, dtype=torch.uint8, device="cuda")
outs = [torch.empty((4, rows), dtype=torch.float32, device="cuda") for _ in range(2)]
for k in range(2):
    ops.token_stats(*bufs[k], mask, "k3", out=outs[k])
torch.cuda.synchronize()
check = [float(outs[0][i].double().mean()) for i in range(4)]
clk = ClockSampler(0)
clk.start()
evs = []
t0 = time.time()
i = 0
while time.time() - t0 < secs:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ops.token_stats(*bufs[i % 2], mask, "k3", out=outs[i % 2])
    b.record()
    evs.append((a, b))
    i += 1
    if i % 64 == 0:
        torch.cuda.synchronize()
torch.cuda.synchronize()
c = clk.stop()
ms = [a.elapsed_time(b) for a, b in evs]
tail = ms[len(ms) // 3:]
avg = statistics.mean(tail)
gbs = rows * bytes_per_row(V) / (avg / 1e3) / 1e9
print(json.dumps({"lib": os.environ.get("YATT_B200_LIB", "default"), "launches": len(ms),
                  "ms_avg_tail": avg, "gbs": gbs, "tok_per_s": rows / (avg / 1e3),
                  "first_ms": ms[:3], "clocks": c, "checksum": check}), flush=True)
