#!/usr/bin/env python3
"""The fused loss + gradient kernel (policy_loss_grad.cu) by shape:
SHAPES entries "<pipe>[order][l|n]" — YATT_FUSED_PIPE 0 (the default
dispatch), 1 (large: 1 CTA/SM) or 2 (small: 2 CTAs/SM); YATT_FUSED_ORDER 0
(forward pass 2) / 1 (reverse, the default); "l" / "n" forces the one-row lag
on / off; k3 and full KL at 32,768 x
152,064 (a configs[1] prompt group).  Device time as tools/bench_kernels.py
(CUDA graph, L2 flushed), achieved algorithmic GB/s vs the measured peak, and
every shape's outputs against the first shape's.  GRIDS="148,128,..." also
sweeps the CTA count (YATT_FUSED_GRID) per shape; MODES="full" limits modes.""" 
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

from bench_kernels import PEAK, timeit  # noqa: E402
from paper_2508_07970_b200 import ops  # noqa: E402

rows = int(os.environ.get("ROWS", 32768))
V = int(os.environ.get("VOCAB", 152064))
shapes = os.environ.get("SHAPES", "0,1n,1l,2n,2l").split(",")
seed = 20250814
pol, ref, tgt = ops.synth_logits(seed, 0, rows, V)
lp, rl, en, kl = ops.token_stats(pol, ref, tgt, None, "k3")
old = ops.synth_floats(seed, 104, 0, rows, "old_delta", base=lp)
adv = ops.synth_floats(seed, 108, 0, rows, "adv")
mask = (torch.arange(rows, device=pol.device) % 97 != 5).to(torch.uint8)
cfg = ops.loss_config(0.2, 0.28, 0.0, 0.001, 0.001, "token-mean")
grad = torch.empty_like(pol)
grids = [g for g in os.environ.get("GRIDS", "").split(",") if g]
for mode in os.environ.get("MODES", "k3,full").split(","):
    base = None
    for sh in [f"{s}@{g}" for s in shapes for g in grids] if grids else shapes:
        if "@" in sh:
            sh, g = sh.split("@")
            os.environ["YATT_FUSED_GRID"] = g
        else:
            os.environ.pop("YATT_FUSED_GRID", None)
        os.environ["YATT_FUSED_PIPE"] = sh[0]  # 0 = the default dispatch by vocabulary
        os.environ.pop("YATT_FUSED_LAG", None)
        if "l" in sh or "n" in sh:  # force the lag on ("l") / off ("n")
            os.environ["YATT_FUSED_LAG"] = "1" if "l" in sh else "0"
        os.environ["YATT_FUSED_ORDER"] = sh[1:].replace("l", "").replace("n", "") or "1"

        def run(m=None):
            return ops.policy_loss_grad(pol, tgt, old, adv, rl if mode != "full" else None, m, cfg,
                                        mode, float(rows), grad,
                                        ref_logits=ref if mode == "full" else None)
        outs = run(mask)
        torch.cuda.synchronize()
        res = [t.clone() for t in outs[:3]] + [grad.clone()]  # vs the first shape
        diff = None
        if base is None:
            base = res
        else:
            d = [float(((a.float() - b.float()).abs() / (b.float().abs() + 1e-6)).max())
                 for a, b in zip(res[:3], base[:3])]
            gd = (res[3].float() - base[3].float()).abs().max().item()
            diff = {"logp_ent_kl_maxrel": d, "grad_maxabs": gd,
                    "grad_neq": int((res[3] != base[3]).sum())}
        ms = timeit(lambda: run(None), iters=10)
        per_row = (6 if mode == "full" else 4) * V + (24 if mode == "full" else 28)
        gbs = rows * per_row / (ms / 1e3) / 1e9
        print(json.dumps({"mode": mode, "shape": sh, "grid": os.environ.get("YATT_FUSED_GRID"),
                          "rows": rows, "V": V, "ms": round(ms, 4),
                          "achieved_gbs": round(gbs, 1), "frac": round(gbs / PEAK, 3),
                          "vs_first_shape": diff}), flush=True)
