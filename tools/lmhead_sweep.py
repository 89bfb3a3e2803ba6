"""Sweep n_split for the fused LM-head kernel (Qwen2.5-7B head) and compare
precision with cuBLAS (bf16 in, fp32 out) against an fp64 reference."""
import json, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2508_07970_b200 import ops

def timeit(fn, iters=8):
    for _ in range(2): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)

d, V = 3584, 152064
for rows in (8192, 32768):
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.randn(rows, d, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(V, d, device="cuda", generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    y = torch.randint(0, V, (rows,), device="cuda", generator=g, dtype=torch.int32)
    for ns in (1, 2, 4, 8, 16, 32):
        ms = timeit(lambda: ops.lmhead_token_stats(h, w, y, n_split=ns))
        print(json.dumps({"rows": rows, "n_split": ns, "ms": round(ms, 3),
                          "tflops": round(2.0 * rows * d * V / ms / 1e9, 1)}), flush=True)
# precision: our entropy vs cuBLAS fp32-out vs fp64 on a K=3584 slice
rows, V2 = 512, 2304
h = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
w = (torch.randn(V2, d, device="cuda") * (2.0 / d ** 0.5)).to(torch.bfloat16)
y = torch.randint(0, V2, (rows,), device="cuda", dtype=torch.int32)
ent = ops.lmhead_token_stats(h, w, y, n_split=1)[1].double().cpu().numpy()
ref = h.double().cpu().numpy() @ w.double().cpu().numpy().T
def entropy(l):
    lp = l - (l.max(1, keepdims=True) + np.log(np.exp(l - l.max(1, keepdims=True)).sum(1, keepdims=True)))
    return -(np.exp(lp) * lp).sum(1)
e64 = entropy(ref)
out = {"ours": float(np.max(np.abs(ent - e64) / e64))}
try:
    l32 = torch.mm(h, w.t(), out_dtype=torch.float32).double().cpu().numpy()
    out["cublas_bf16_fp32out"] = float(np.max(np.abs(entropy(l32) - e64) / e64))
except Exception as ex:
    out["cublas_bf16_fp32out"] = repr(ex)[:80]
torch.backends.cuda.matmul.allow_tf32 = False
l32s = (h.float() @ w.float().t()).double().cpu().numpy()
out["fp32_simt"] = float(np.max(np.abs(entropy(l32s) - e64) / e64))
print(json.dumps({"entropy_max_rel_err": out}), flush=True)
