"""Aggregate ncu warp-stall samples by CUDA source line.

usage: python tools/ncu_lines.py report.ncu-rep [top_n]
Reads `ncu -i ... --page source --csv --print-source cuda,sass` and prints the
lines with the most samples and their dominant stall reasons."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    agg, cur, hdr = {}, None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        i = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            v = float(r[i])
        except ValueError:
            continue
        key = (cur, r[0])
        a = agg.setdefault(key, [0.0, r[1].strip()[:90], {}])
        a[0] += v
        for j, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    a[2][h] = a[2].get(h, 0.0) + float(r[j])
                except ValueError:
                    pass
    tot = sum(a[0] for a in agg.values()) or 1.0
    for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        why = ", ".join(f"{n[6:]} {int(c)}" for n, c in sorted(a[2].items(), key=lambda x: -x[1])[:3])
        print(f"{k[0]}:{k[1]:>5} {int(a[0]):6d} {100 * a[0] / tot:5.1f}%  {a[1]}  [{why}]")


if __name__ == "__main__":
    main()
