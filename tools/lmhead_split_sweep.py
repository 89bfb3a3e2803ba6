"""n_split sweep of the fused LM head at several heads (argv: d V rows...)."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_07970_b200 import ops  # noqa: E402


def timeit(fn, iters=6):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


d, V = int(sys.argv[1]), int(sys.argv[2])
for rows in [int(x) for x in sys.argv[3:]]:
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.randn(rows, d, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(V, d, device="cuda", generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    y = torch.randint(0, V, (rows,), device="cuda", generator=g, dtype=torch.int32)
    for ns in [int(x) for x in __import__('os').environ.get('NS', '1,2,4,8,19,38,75,150').split(',')]:
        ms = timeit(lambda: ops.lmhead_token_stats(h, w, y, n_split=ns))
        print(json.dumps({"d": d, "V": V, "rows": rows, "n_split": ns, "ms": round(ms, 3),
                          "tflops": round(2.0 * rows * d * V / ms / 1e9, 1)}), flush=True)
