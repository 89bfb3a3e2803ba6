#!/usr/bin/env python3
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

  python tools/summarize_ncu.py launches <launches.csv> <out.md>
      per-kernel share of a `--metrics gpu__time_duration.sum` launch list
  python tools/summarize_ncu.py full <report.ncu-rep> <rows_per_launch> <vocab> <out-prefix>
      key metrics of a `--set full` capture of token_stats -> <out-prefix>.md and
      profiles/token_stats_ncu.json (per-launch DRAM traffic used by bench.py)
"""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "lts__t_bytes.sum"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def launches(csv_path, out_md):
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("yattb::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {t / 1e6:.3f} | {100 * t / tot:.2f}% |")
    Path(out_md).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, rows, vocab, prefix):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rs = list(csv.reader(out.splitlines()))
    h, u = rs[0], rs[1]
    vals = {}
    for r in rs[2:]:
        for k in KEYS:
            if k in h:
                i = h.index(k)
                vals.setdefault(k, []).append((r[i], u[i]))
    first = {k: v[0] for k, v in vals.items()}
    rd = float(first["dram__bytes_read.sum"][0]) * SCALE.get(first["dram__bytes_read.sum"][1], 1)
    wr = float(first["dram__bytes_write.sum"][0]) * SCALE.get(first["dram__bytes_write.sum"][1], 1)
    alg = rows * (4 * vocab + 21)
    dur_us = float(first["gpu__time_duration.sum"][0])
    summary = {"kernel": "token_stats_kernel", "rows_per_launch": rows, "vocab": vocab,
               "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
               "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": (rd + wr) / alg,
               "duration_us": dur_us, "achieved_gbs_under_ncu": alg / (dur_us * 1e-6) / 1e9,
               "metrics": {k: f"{v[0]} {v[1]}" for k, v in first.items()}}
    Path(prefix + ".json").write_text(json.dumps(summary, indent=1) + "\n")
    Path("profiles/token_stats_ncu.json").write_text(json.dumps(
        {"dram_bytes_per_launch": rd + wr, "rows_per_launch": rows, "vocab": vocab,
         "source": Path(prefix).name}, indent=1) + "\n")
    md = [f"# ncu --set full: token_stats_kernel ({rows} rows x V={vocab})", "",
          "| metric | value |", "|---|---|"]
    md += [f"| {k} | {v[0]} {v[1]} |" for k, v in first.items()]
    md += ["", f"DRAM traffic {rd + wr:.4g} B vs algorithmic {alg:.4g} B "
               f"(ratio {(rd + wr) / alg:.4f})."]
    Path(prefix + ".md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
