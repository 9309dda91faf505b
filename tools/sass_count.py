"""Count SASS instructions per kernel in an object/cubin: python tools/sass_count.py <file.o> [substr]"""
import re, subprocess, sys, tempfile, os, glob
f = sys.argv[1]; sub = sys.argv[2] if len(sys.argv) > 2 else ""
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(f)], cwd=d, capture_output=True)
for cub in glob.glob(d + "/*.cubin"):
    txt = subprocess.run(["nvdisasm", "-c", cub], capture_output=True, text=True).stdout.split("\n")
    name, n = None, 0
    for l in txt + ["//----- end"]:
        if l.startswith("//-----"):
            if name and sub in name:
                print(f"{n:7d} {name[:110]}")
            m = re.search(r"\.text\.(\S+)", l)
            name, n = (m.group(1) if m else None), 0
        elif re.match(r"\s*/\*[0-9a-f]{4,}\*/", l):
            n += 1
