"""TEST INFRASTRUCTURE: golden vectors that pin the float oracle's per-token
log-softmax quantities (A1) to the reference's own fp64 softmax
(yatt::distattn::reference_attention, proj/src/distattn.cpp:79-123), via
oracle/softmax_pin.cpp (built by `make -C oracle _ref/softmax_pin` from the
reference's sources).

    python oracle/softmax_golden.py      # writes tests/golden/softmax_pin.json

`inputs(case)` regenerates each case's bf16 logits and targets (the keyed
synthetic rows of SURVEY.md §8d plus hand-built edge rows), so the JSON
holds only the reference's outputs."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
# run as a script: the repo root, not oracle/, resolves `oracle` (the package)
sys.path[:] = [p for p in sys.path if Path(p or ".").resolve() != HERE]
sys.path.insert(0, str(HERE.parent))

CASES = [
    {"name": "keyed_v2048", "seed": 20250814, "rows": 6, "V": 2048},
    {"name": "keyed_v1000_odd", "seed": 7, "rows": 4, "V": 1000},
    {"name": "edge_v512", "seed": 0, "rows": 5, "V": 512},
]


def _bf16_bits(f32):
    """Round-to-nearest-even fp32 -> bf16 bit patterns (uint16)."""
    u = np.ascontiguousarray(f32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def inputs(case):
    """(policy bits, reference bits, targets) of a case."""
    from oracle import oracle as O
    if case["name"].startswith("keyed"):
        return O.synth_logits(case["seed"], 0, case["rows"], case["V"])
    V = case["V"]
    j = np.arange(V, dtype=np.float32)
    rows_p = [
        np.zeros(V, np.float32),                        # uniform: H = ln V
        np.where(j == 17, 60.0, 0.0).astype(np.float32),  # one dominant logit
        np.where(j == 3, -60.0, 1.0).astype(np.float32),  # target far below the rest
        (j % 7 - 3.0).astype(np.float32) * 4.0,         # wide spread, ties
        np.full(V, -30.0, np.float32) + (j % 3),        # large negative offset
    ]
    rows_q = [
        (j % 5).astype(np.float32) * 0.5,
        np.zeros(V, np.float32),
        np.where(j == 3, 2.0, 0.5).astype(np.float32),
        (3.0 - j % 7).astype(np.float32) * 4.0,
        np.full(V, 25.0, np.float32) - (j % 11) * 0.25,
    ]
    tgt = np.array([5, 17, 3, 100, 511], dtype=np.int32)
    return _bf16_bits(np.stack(rows_p)), _bf16_bits(np.stack(rows_q)), tgt


LMHEAD_CASES = [
    {"name": "lmhead_d64_v1024", "seed": 3, "rows": 4, "d": 64, "V": 1024},
    {"name": "lmhead_d256_v520", "seed": 4, "rows": 3, "d": 256, "V": 520},
]


def lmhead_inputs(case):
    """(hidden bits [rows, d], W bits [V, d], targets) of an LM-head case."""
    rng = np.random.default_rng(case["seed"])
    d, V = case["d"], case["V"]
    h = _bf16_bits(rng.standard_normal((case["rows"], d)).astype(np.float32))
    w = _bf16_bits((rng.standard_normal((V, d)) * (2.0 / d ** 0.5)).astype(np.float32))
    tgt = rng.integers(0, V, case["rows"]).astype(np.int32)
    return h, w, tgt


def run_reference_lmhead(h, w, tgt):
    exe = HERE / "_ref" / "softmax_pin"
    rows, d = h.shape
    payload = (np.array([rows, d, w.shape[0]], dtype=np.int32).tobytes() + to_f64(h).tobytes()
               + to_f64(w).tobytes() + np.ascontiguousarray(tgt, dtype=np.int32).tobytes())
    res = subprocess.run([str(exe), "lmhead"], input=payload, capture_output=True, check=True)
    out = []
    for line in res.stdout.decode().split("\n"):
        if line.strip():
            _, py, *ew = line.split()
            out.append({"p_y": float(py), "E_p_W": [float(v) for v in ew]})
    return out


def to_f64(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def run_reference(pol, ref, tgt):
    exe = HERE / "_ref" / "softmax_pin"
    rows, V = pol.shape
    payload = (np.array([rows, V], dtype=np.int32).tobytes() + to_f64(pol).tobytes()
               + to_f64(ref).tobytes() + np.ascontiguousarray(tgt, dtype=np.int32).tobytes())
    res = subprocess.run([str(exe)], input=payload, capture_output=True, check=True)
    out = {}
    for line in res.stdout.decode().split("\n"):
        if line.strip():
            r, t, *c = line.split()
            out[(int(r), int(t))] = [float(v) for v in c]
    return [{"pol": out[(r, 0)], "ref": out[(r, 1)]} for r in range(rows)]


def main():
    golden = []
    for case in CASES:
        pol, ref, tgt = inputs(case)
        golden.append({**case, "targets": tgt.tolist(), "rows_out": run_reference(pol, ref, tgt)})
    lm = []
    for case in LMHEAD_CASES:
        h, w, tgt = lmhead_inputs(case)
        lm.append({**case, "targets": tgt.tolist(), "rows_out": run_reference_lmhead(h, w, tgt)})
    dst = HERE.parent / "tests" / "golden" / "softmax_pin.json"
    dst.write_text(json.dumps({"source": "yatt::distattn::reference_attention "
                                         "(proj/src/distattn.cpp:79-123) via oracle/softmax_pin.cpp",
                               "columns": "per head: (E_p[x], p_y, E_p[z], 1); pol head x = policy, "
                                          "z = reference; ref head swapped",
                               "cases": golden,
                               "lmhead_columns": "per token row: p_y and E_p[W] (softmax over "
                                                 "h . W_j, q = sqrt(d) h, k_j = W_j)",
                               "lmhead_cases": lm}, indent=1))
    print(f"wrote {dst}")


if __name__ == "__main__":
    main()
