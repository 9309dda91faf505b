"""profiles/ncu_summary.json (read by bench.py for roofline.traffic and the
pool-build instruction counts) from one `tools/ncu_summary.py` output.

usage: python tools/update_ncu_summary.py "<what build/command>" profiles/<capture>.json[:tag] [more.json[:tag] ...]
A ":tag" suffix files that capture's kernels as "<kernel>@<tag>" (another config's
launches of a kernel the C2 sweep also runs must not be averaged into the C2 entry
bench.py reads).
Per kernel (template arguments dropped): mean over the captured launches of
DRAM bytes (read + write), executed warp instructions and the ncu duration.
"""
import json, re, sys
from collections import defaultdict

what, srcs = sys.argv[1], sys.argv[2:]
acc = defaultdict(list)
src_of = {}
for arg in srcs:
    src, _, tag = arg.partition(":")
    for k in json.load(open(src)):
        name = re.sub(r"^void ", "", k["kernel"]).split("<")[0].strip() + (f"@{tag}" if tag else "")
        acc[name].append(k)
        src_of[name] = src
out = {}
for name, ks in acc.items():
    mean = lambda f: sum(k.get(f, 0.0) for k in ks) / len(ks)  # noqa: E731
    out[name] = {"dram_bytes": mean("dram_bytes"), "inst_executed": mean("inst_executed"),
                 "duration_ms_ncu": mean("duration_ms"), "launches_captured": len(ks),
                 "source": f"{src_of[name]} ({what})"}
json.dump(out, open("profiles/ncu_summary.json", "w"), indent=1)
print(json.dumps(out, indent=1))
