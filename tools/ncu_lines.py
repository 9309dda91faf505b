"""Aggregate an ncu source page (--print-source cuda,sass) per CUDA source line.

usage: ncu -i rep --page source --csv --print-source cuda,sass -k regex:K > x.csv
       python tools/ncu_lines.py x.csv [top]
"""
import csv, os, sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fpath, line, src = "?", None, ""
agg = defaultdict(lambda: [0.0, 0.0, ""])
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        line, src = r[0], r[1]
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        inst = float(d.get("Instructions Executed", "0") or 0)
        st = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    k = (fpath, line)
    agg[k][0] += inst
    agg[k][1] += st
    agg[k][2] = src.strip()[:80]
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp inst {ti:.4g}, stall samples {ts:.4g}")
col = 1 if os.environ.get("SORT") == "stall" else 0
for (f, l), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][col])[:top]:
    print(f"{100 * i / ti:6.2f}% inst {100 * s / ts:6.2f}% stall  {f}:{l}  {src}")
