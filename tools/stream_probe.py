"""Power-cap probe: how fast does a PLAIN HBM read stream run when sustained
on this power-capped B200, next to A1 (tools/a1_sustained.py) on the same
buffers?  Streams the same 2 x 2 bf16 tensors (32,768 x 152,064 each, 19.9 GB
per step) through torch.sum (fp32 accumulate: minimal math per byte) for
`secs` seconds, times every step with CUDA events, reports the mean over the
last 2/3 with nvidia-smi clocks / power.  If the plain stream sustains much
more than A1, A1's arithmetic costs bandwidth under the power cap; if it
settles near A1, HBM + the cap set the ceiling.  One JSON line."""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2508_07970_b200 import ops  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
rows, V = 32768, 152064
bufs = [ops.synth_logits(20250814 + k, 0, rows, V)[:2] for k in range(2)]
nbytes = 2 * rows * V * 2
for k in range(2):
    torch.sum(bufs[k][0], dtype=torch.float32)
torch.cuda.synchronize()
clk = ClockSampler(0)
clk.start()
evs = []
t0 = time.time()
i = 0
while time.time() - t0 < secs:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    p, r = bufs[i % 2]
    torch.sum(p, dtype=torch.float32)
    torch.sum(r, dtype=torch.float32)
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
print(json.dumps({"probe": "torch.sum over both tensors (read-only stream)", "steps": len(ms),
                  "ms_avg_tail": avg, "gbs": nbytes / (avg / 1e3) / 1e9,
                  "first_ms": ms[:3], "clocks": c}), flush=True)
