"""ncu driver: the fused loss + gradient kernel at the Qwen2.5-7B head
(8,192 rows x V=152,064; PROF_ROWS / PROF_V override) — DRAM bytes show
whether pass 2 hits L2."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os  # noqa: E402
import torch  # noqa: E402
from paper_2508_07970_b200 import ops  # noqa: E402

rows, V = int(os.environ.get("PROF_ROWS", 8192)), int(os.environ.get("PROF_V", 152064))
pol, ref, tgt = ops.synth_logits(1, 0, rows, V)
lp, rl, en, kl = ops.token_stats(pol, ref, tgt, None, "k3")
old = ops.synth_floats(1, 104, 0, rows, "old_delta", base=lp)
adv = ops.synth_floats(1, 108, 0, rows, "adv")
grad = torch.empty_like(pol)
cfg = ops.loss_config(0.2, 0.28, 0.0, 0.001, 0.001, "token-mean")
mode = os.environ.get("KL_MODE", "k3")  # k3 | full
for _ in range(2):
    ops.policy_loss_grad(pol, tgt, old, adv, rl if mode != "full" else None, None, cfg, mode,
                         float(rows), grad, ref_logits=ref if mode == "full" else None)
torch.cuda.synchronize()
print("ok")
