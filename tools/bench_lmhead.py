"""§8f #4 benchmark: fused tcgen05 LM-head + online log-softmax vs the unfused
path (cuBLAS bf16 GEMM writing [rows, V] logits + the A1-style streaming
read); default Qwen2.5-7B head d=3584, V=152,064 (argv: rows [d V]).  TFLOP/s vs the measured cuBLAS
bf16 peak (MEASURED_PEAKS.json).  One JSON line per measurement."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_07970_b200 import ops  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (
    ROOT / "MEASURED_PEAKS.json").exists() else {"bf16_tflops": 1590.0,
                                                  "bf16_tflops_sustained": 1400.0}


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
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


rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d = int(sys.argv[2]) if len(sys.argv) > 2 else 3584      # Qwen2.5-7B hidden
V = int(sys.argv[3]) if len(sys.argv) > 3 else 152064    # Qwen2.5 vocabulary
g = torch.Generator(device="cuda").manual_seed(0)
h = torch.randn(rows, d, device="cuda", generator=g).to(torch.bfloat16)
w = (torch.randn(V, d, device="cuda", generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
y = torch.randint(0, V, (rows,), device="cuda", generator=g, dtype=torch.int32)
flops = 2.0 * rows * d * V

ms = timeit(lambda: ops.lmhead_token_stats(h, w, y))
print(json.dumps({"op": "fused lmhead_token_stats (tcgen05)", "rows": rows, "d": d, "V": V,
                  "ms": ms, "tflops": flops / ms / 1e9,
                  "frac_of_measured_bf16": flops / ms / 1e9 / peaks["bf16_tflops"]}), flush=True)

logits = torch.empty((rows, V), dtype=torch.bfloat16, device="cuda")
ms_gemm = timeit(lambda: torch.matmul(h, w.t(), out=logits))
print(json.dumps({"op": "cuBLAS bf16 GEMM (logits materialised)", "rows": rows, "d": d, "V": V,
                  "ms": ms_gemm,
                  "tflops": flops / ms_gemm / 1e9}), flush=True)
# the unfused path: GEMM + streaming log-softmax statistics over the logits
# (token_stats reads two tensors; the single-model read is half of that)
ms_a1 = timeit(lambda: ops.token_stats(logits, logits, y))
print(json.dumps({"op": "unfused: GEMM + token_stats", "ms": ms_gemm + ms_a1 / 2,
                  "fused_speedup": (ms_gemm + ms_a1 / 2) / ms,
                  "logits_bytes_avoided": rows * V * 2}), flush=True)
