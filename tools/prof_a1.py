"""Profiling driver: the A1 token_stats kernel on one 8192-row chunk at
V=152,064 (4.98 GB of bf16 logits, >> L2), launched 4 times.  Used as
`ncu --set full -k regex:token_stats -s 2 -c 1 python tools/prof_a1.py`."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_07970_b200 import ops  # noqa: E402

ROWS = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
V = int(sys.argv[2]) if len(sys.argv) > 2 else 152064
KL = sys.argv[3] if len(sys.argv) > 3 else "k3"
pol, ref, tgt = ops.synth_logits(20250814, 0, ROWS, V)
mask = torch.ones(ROWS, dtype=torch.uint8, device="cuda")
out = torch.empty((4, ROWS), dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for i in range(4):
    ev[i].record()
    ops.token_stats(pol, ref, tgt, mask, KL, out=out)
ev[4].record()
torch.cuda.synchronize()
ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
gbs = ROWS * (4 * V + 21) / (min(ms[1:]) / 1e3) / 1e9
print(f"token_stats rows={ROWS} V={V} kl={KL} ms={ms} best={gbs:.1f} GB/s")
