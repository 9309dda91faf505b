"""Summarise an ncu report (--set full) into JSON + markdown for profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> <out-prefix>
Writes <out-prefix>.json (per-kernel metrics) and <out-prefix>.md.
"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
    "inst_executed": ("smsp__inst_executed.sum", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
}
scale_units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "msecond": 1e6, "usecond": 1e3, "nsecond": 1}
res = []
for r in rows[2:]:
    k = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
    for name, (m, _) in want.items():
        if m not in hdr:
            continue
        i = hdr.index(m)
        try:
            v = float(r[i].replace(",", ""))
        except ValueError:
            continue
        u = units[i]
        if name == "duration_ms":
            v = v * {"msecond": 1.0, "ms": 1.0, "usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "ns": 1e-6, "second": 1e3, "s": 1e3}.get(u, 1.0)
        elif "bytes" in name:
            v = v * scale_units.get(u, 1)
        k[name] = v
    if "dram_read_bytes" in k:
        k["dram_bytes"] = k["dram_read_bytes"] + k.get("dram_write_bytes", 0)
    res.append(k)
json.dump(res, open(out + ".json", "w"), indent=1)
with open(out + ".md", "w") as f:
    f.write(f"# ncu summary of `{rep.split('/')[-1]}`\n\n")
    f.write("| kernel | ms | DRAM MB (r+w) | DRAM % | L2 hit % | warps active % | issue % | regs | inst |\n|---|---|---|---|---|---|---|---|---|\n")
    for k in res:
        f.write(f"| {k['kernel']} | {k.get('duration_ms', 0):.4f} | {k.get('dram_bytes', 0) / 1e6:.1f} | "
                f"{k.get('dram_throughput_pct', 0):.1f} | {k.get('l2_hit_pct', 0):.1f} | {k.get('warps_active_pct', 0):.1f} | "
                f"{k.get('issue_active_pct', 0):.1f} | {int(k.get('registers', 0))} | {k.get('inst_executed', 0):.3g} |\n")
print(json.dumps(res, indent=1)[:2000])
