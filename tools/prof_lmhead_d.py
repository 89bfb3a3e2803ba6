"""ncu driver: the fused LM head (cta_group::2 pair kernel) at a large hidden
size (argv: rows d V; default 8,192 x 8,192 x 128,256)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2508_07970_b200 import ops  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
V = int(sys.argv[3]) if len(sys.argv) > 3 else 128256
g = torch.Generator(device="cuda").manual_seed(0)
h = torch.randn(rows, d, device="cuda", generator=g).to(torch.bfloat16)
w = (torch.randn(V, d, device="cuda", generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
y = torch.randint(0, V, (rows,), device="cuda", generator=g, dtype=torch.int32)
for _ in range(2):
    ops.lmhead_token_stats(h, w, y, n_split=int(sys.argv[4]) if len(sys.argv) > 4 else 2)
torch.cuda.synchronize()
print("ok")
