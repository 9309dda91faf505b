"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) as markdown.

usage: python tools/launches_md.py launches.csv "<title line>" > profiles/<name>.md
Per kernel: launches, total us, us/launch; plus each sweep kernel's share of the
sweep (k_mark, k_pool_*, k_tile_*, k_scan*, k_sample, flush).
"""
import csv, sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
    name = r[ki].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale
title = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
print(f"# Launch list: {title}\n")
print("| kernel | launches | total us | us/launch |\n|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {n} | {t:.1f} | {t / n:.1f} |")
sweep = {k: v for k, v in agg.items()
         if any(s in k for s in ("k_mark", "k_bits", "k_append_hash", "k_pool", "k_tile", "k_sample", "k_fill_u64", "k_sweep"))}
tot = sum(t for _, t in sweep.values()) or 1
print("\nShare of the sweep kernels (serialised, cold-cache times):\n")
for k, (n, t) in sorted(sweep.items(), key=lambda kv: -kv[1][1]):
    print(f"- {k}: {100 * t / tot:.1f} %")
