"""Profiling driver: logits_backward on 8192 rows x V=152,064 (k3 or full),
4 launches.  `ncu --set full -k regex:logits_backward -s 2 -c 1 python tools/prof_bwd.py`."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_07970_b200 import ops  # noqa: E402

ROWS = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
MODE = sys.argv[2] if len(sys.argv) > 2 else "k3"
V = 152064
pol, ref, tgt = ops.synth_logits(20250814, 0, ROWS, V)
lp, rl, en, kl = ops.token_stats(pol, ref, tgt, None, MODE)
old = ops.synth_floats(1, 104, 0, ROWS, "old_delta", base=lp)
a = ops.synth_floats(1, 108, 0, ROWS, "adv")
grad = torch.empty_like(pol)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for i in range(4):
    ev[i].record()
    ops.logits_grad(pol, ref, tgt, lp, rl, old, a, en, kl, None, None,
                    ops.loss_config(entropy_coef=0.001), MODE, float(ROWS), grad)
ev[4].record()
torch.cuda.synchronize()
ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
per_row = (6 if MODE == "full" else 4) * V + 32
print(f"logits_grad rows={ROWS} mode={MODE} ms={ms} best={ROWS * per_row / min(ms[1:]) / 1e6:.1f} GB/s")
