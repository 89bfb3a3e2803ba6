#!/usr/bin/env python3
"""Static SASS instruction-class counts of the shipped kernels
(cuobjdump -sass paper_2508_07970_b200/libyatt_b200.so) -> profiles/.

  python tools/sass_classes.py [out.md]

For each hot-path kernel: total static instructions and the classes that
prove the design — UBLKCP (TMA bulk copy), UTMALDG (TMA tensor load), SYNCS
(mbarrier), MUFU.EX2, FFMA2/FADD2/FMUL2 (packed fp32), HMNMX2 (bf16x2 max),
F2FP (fp32 -> bf16x2 pack), LDS/STG widths, UTCHMMA/LDTM (tcgen05 MMA / TMEM
load), DFMA (fp64), and STL/LDL (local-memory spills; 0 expected)."""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2508_07970_b200" / "libyatt_b200.so"
KERNELS = [  # (label, mangled-name substring)
    ("A1 token_stats k3 (large vocab)", "token_stats_cu_308a9ff918token_stats_kernelILb0ELb0E"),
    ("A1 token_stats full KL (large vocab)", "token_stats_cu_308a9ff918token_stats_kernelILb1ELb0E"),
    ("A1 token_stats k3 (small vocab)", "token_stats_small_cu_0a19fc3018token_stats_kernelILb0ELb0E"),
    ("A1 token_stats_rowwarp k3 (V <= 36,864)", "token_stats_rowwarp_kernelILb0E"),
    ("8f#1 policy_loss_grad_pipe k3 (reverse pass 2)", "policy_loss_grad_pipe_kernelILb0ELi1E"),
    ("8f#1 policy_loss_grad_pipe full KL (reverse pass 2)", "policy_loss_grad_pipe_kernelILb1ELi1E"),
    ("8f#1 logits_backward k3", "logits_backward_kernelILb0E"),
    ("8f#4 lmhead_lse single CTA (tcgen05)", "lmhead_lse_kernelILi1E"),
    ("8f#4 lmhead_lse_pair (tcgen05 cta_group::2)", "lmhead_lse_pair_kernel"),
    ("A3 gae_warp (16-B loads)", "gae_warp_kernelILb1ELb0E"),
    ("A3 gae_warp (scalar loads, unaligned views)", "gae_warp_kernelILb0ELb0E"),
    ("A4 loss_token", "loss_token_kernelILb0E"),
]
CLASSES = ["UBLKCP", "UTMALDG", "SYNCS", "MUFU.EX2", "FFMA2", "FADD2", "FMUL2", "HMNMX2",
           "VHMNMX", "F2FP", "LDS.128", "LDS", "STG.E.EF.128", "STG.E.128", "STG", "LDG",
           "UTCHMMA", "UTCBAR", "LDTM", "DFMA", "STL", "LDL"]


def main():
    out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r2_sass_classes.md"
    txt = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)[1:]
    rows = []
    for label, sub in KERNELS:
        body = next((f for f in funcs if sub in f.split("\n")[0]), None)
        if body is None:
            rows.append((label, None, {}))
            continue
        ops = collections.Counter()
        total = 0
        for line in body.split("\n"):
            m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if not m:
                continue
            op = m.group(2)
            total += 1
            for c in CLASSES:
                if op == c or op.startswith(c + "."):
                    ops[c] += 1
                    break
        rows.append((label, total, ops))
    lines = ["# Static SASS instruction classes of the shipped kernels", "",
             f"`python tools/sass_classes.py` over `cuobjdump -sass {LIB.relative_to(ROOT)}` "
             "(sm_100a).  Static counts (instructions in the kernel body, not executions).", "",
             "| kernel | total | " + " | ".join(CLASSES) + " |",
             "|---|---|" + "---|" * len(CLASSES)]
    for label, total, ops in rows:
        if total is None:
            lines.append(f"| {label} | (not found) |" + " |" * len(CLASSES))
            continue
        lines.append(f"| {label} | {total} | " + " | ".join(str(ops.get(c, 0)) for c in CLASSES)
                     + " |")
    out.write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
