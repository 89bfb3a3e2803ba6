"""A1 (and the backward) at vocabularies not divisible by 8 (GPT-2's 50,257,
151,937) next to the nearest aligned size: the aligned-superset staging of
the TMA path.  One line per shape: ms and algorithmic GB/s."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_07970_b200 import ops
dev = torch.device("cuda:0")
for rows, V in [(16384, 50257), (16384, 50264), (4096, 151937)]:
    g = torch.Generator(device=dev).manual_seed(1)
    pol = (torch.randn(rows, V, device=dev, generator=g) * 2).to(torch.bfloat16)
    ref = (pol.float() + 0.1 * torch.randn(rows, V, device=dev, generator=g)).to(torch.bfloat16)
    tgt = torch.randint(0, V, (rows,), device=dev, generator=g, dtype=torch.int32)
    out = torch.empty((4, rows), device=dev)
    for _ in range(2): ops.token_stats(pol, ref, tgt, None, "k3", out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): ops.token_stats(pol, ref, tgt, None, "k3", out=out)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(rows, V, round(ms, 3), "ms", round(rows * (4 * V + 21) / ms / 1e6), "GB/s")

# backward into the logits at the same odd vocabularies (k3: 4V B/row)
for rows, V in [(16384, 50257), (16384, 50264)]:
    g = torch.Generator(device=dev).manual_seed(2)
    pol = (torch.randn(rows, V, device=dev, generator=g) * 2).to(torch.bfloat16)
    tgt = torch.randint(0, V, (rows,), device=dev, generator=g, dtype=torch.int32)
    lp, rl, en, kl = ops.token_stats(pol, pol, tgt, None, "k3")
    adv = torch.randn(rows, device=dev, generator=g)
    grad = torch.empty_like(pol)
    f = lambda: ops.logits_grad(pol, pol, tgt, lp, rl, lp, adv, en, kl, None, None, None, "k3",  # noqa: E731
                                float(rows), grad)
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        f()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print("backward", rows, V, round(ms, 3), "ms", round(rows * (4 * V + 32) / ms / 1e6), "GB/s")
