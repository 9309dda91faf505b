"""Aggregate an ncu SASS source-page CSV by CUDA source line.

usage: python tools/sass_lines.py <cubin> <kernel-mangled-substring> <ncu_source.csv> [top]
(ncu -i rep --page source --csv -k <kernel> > ncu_source.csv; cuobjdump -xelf all x.o)
"""
import collections, csv, re, subprocess, sys

cubin, kname, ncsv = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(sass) if l.startswith("//-----") and kname in l)
insts, cur = [], None
for l in sass[start + 2:]:
    if l.startswith("//-----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
    m2 = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
    if m2:
        insts.append((cur, m2.group(2)))
rows = list(csv.reader(open(ncsv)))
hdr = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")][: len(insts)]
si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
S, I = collections.Counter(), collections.Counter()
for (key, _), r in zip(insts, data):
    S[key] += f(r[si])
    I[key] += f(r[ie])
ts, ti = sum(S.values()) or 1, sum(I.values()) or 1
srcs = {}
print(f"{len(insts)} SASS instructions, {len(data)} ncu rows")
for key, v in sorted(S.items(), key=lambda kv: -kv[1])[:top]:
    if key is None:
        continue
    fn, ln = key
    if fn not in srcs:
        try:
            srcs[fn] = open(next(p for p in [f"paper_2605_00616_b200/csrc/{fn}"])).read().split("\n")
        except OSError:
            srcs[fn] = []
    txt = srcs[fn][ln - 1].strip()[:72] if ln - 1 < len(srcs[fn]) else ""
    print(f"{fn:18s}:{ln:4d} stall {100 * v / ts:5.1f}%  inst {100 * I[key] / ti:5.1f}%  {txt}")
