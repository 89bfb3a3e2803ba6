#!/usr/bin/env python3
"""A1 at small vocabularies: the warp-per-row kernel (YATT_A1_ROWWARP_VMAX >=
V) vs the ring kernels, k3 and full KL; CUDA events, L2 flushed between
launches, median of 10.  One JSON line per (V, kernel, mode)."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_07970_b200 import ops  # noqa: E402

PEAK = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for V in [int(v) for v in os.environ.get("VOCABS", "4096,8192,16384,32000,50264").split(",")]:
    rows = (2 << 30) // (4 * V) // 8 * 8  # ~2 GB of logits per launch
    pol, ref, tgt = ops.synth_logits(1, 0, rows, V, device=dev)
    out = torch.empty((4, rows), device=dev)
    for mode in ("k3", "full"):
        base = None
        for kern, vmax in (("ring", "0"), ("rowwarp", "1000000")):
            os.environ["YATT_A1_ROWWARP_VMAX"] = vmax
            for _ in range(3):
                ops.token_stats(pol, ref, tgt, None, mode, out=out)
            torch.cuda.synchronize()
            res = out.clone()
            ts = []
            for _ in range(10):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ops.token_stats(pol, ref, tgt, None, mode, out=out)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            ms = ts[len(ts) // 2]
            gbs = rows * (4 * V + 21) / (ms / 1e3) / 1e9
            diff = None
            if base is None:
                base = res
            else:
                diff = float(((res - base).abs() / (base.abs() + 1e-6)).max())
            print(json.dumps({"V": V, "rows": rows, "mode": mode, "kernel": kern, "ms": round(ms, 4),
                              "gbs": round(gbs, 1), "frac": round(gbs / PEAK, 3),
                              "max_rel_vs_ring": diff}), flush=True)
    del pol, ref, tgt, out
