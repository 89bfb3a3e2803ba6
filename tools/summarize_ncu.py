#!/usr/bin/env python3
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

  python tools/summarize_ncu.py launches <launches.csv> <out.md>
      per-kernel share of a `--metrics gpu__time_duration.sum` launch list
  python tools/summarize_ncu.py multi <report.ncu-rep> <out.md> [substr=alg_bytes ...]
      one row per captured kernel (duration, DRAM traffic, issue, occupancy) and,
      where an algorithmic byte count is given for a kernel-name substring, the
      achieved algorithmic GB/s and traffic/algorithmic ratio
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


def multi(rep, out_md, algs):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rs = list(csv.reader(out.splitlines()))
    h, u = rs[0], rs[1]

    def val(r, k):
        i = h.index(k)
        return float(r[i].replace(",", "")) * SCALE.get(u[i], 1.0)
    md = [f"# ncu --set full: {Path(rep).name}", "",
          "| kernel | us | DRAM B | alg B | alg GB/s | traffic/alg | DRAM % | issue % | warps % | regs |",
          "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rs[2:]:
        name = r[h.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").split("::")[-1]
        us = val(r, "gpu__time_duration.sum")
        if u[h.index("gpu__time_duration.sum")] == "nsecond":
            us /= 1e3
        dram = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        alg = next((float(b) for s_, b in algs if s_ in name), None)
        md.append("| {} | {:.1f} | {:.4g} | {} | {} | {} | {:.1f} | {:.1f} | {:.1f} | {:.0f} |".format(
            short, us, dram, f"{alg:.4g}" if alg else "-",
            f"{alg / (us * 1e-6) / 1e9:.0f}" if alg else "-",
            f"{dram / alg:.3f}" if alg else "-",
            val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            val(r, "launch__registers_per_thread")))
    Path(out_md).write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "multi":
        multi(sys.argv[2], sys.argv[3], [a.split("=") for a in sys.argv[4:]])
    else:
        full(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
