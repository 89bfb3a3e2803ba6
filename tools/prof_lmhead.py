"""Profiling driver: fused LM-head kernel, 8192 rows x d=3584 x V=152064, 3 launches."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2508_07970_b200 import ops  # noqa: E402
rows, d, V = 8192, 3584, 152064
h = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
w = (torch.randn(V, d, device="cuda") * 0.03).to(torch.bfloat16)
y = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
for _ in range(3):
    ops.lmhead_token_stats(h, w, y)
torch.cuda.synchronize()
print("ok")
