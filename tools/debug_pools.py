"""Diagnose GPU-vs-oracle pool mismatches (prints per-key differences)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import emu_oracle as O
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, build_pack_arrays
from paper_2605_00616_b200.workloads import records_llama

floor = int(sys.argv[1]) if len(sys.argv) > 1 else 256
rec = records_llama(50_000, 0)
pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
tabs = [O.Table(s.tt, s.conc, s.off, s.samples) for s in pack.soas()]
rng = np.random.default_rng(floor)
n = 400
kt = rng.integers(-5, 3000, n); kc = rng.integers(-3, 300, n); kp = rng.integers(0, 2, n)
orc = LatencyOracle(pack, OracleConfig(reliability_floor=floor))
g = orc.pools(kt, kc, kp)
w = O.pools(tabs, kt, kc, kp, floor)
bad = 0
for u in range(n):
    gb = g[1][g[0][u]:g[0][u + 1]]; wb = w[1][w[0][u]:w[0][u + 1]]
    gd = g[2][g[0][u]:g[0][u + 1]]; wd = w[2][w[0][u]:w[0][u + 1]]
    if len(gb) != len(wb) or (gb != wb).any() or (gd != wd).any():
        bad += 1
        if bad <= 6:
            t = tabs[w[5][u]]
            j = 0
            while j < min(len(gb), len(wb)) and gb[j] == wb[j]:
                j += 1
            print(f"key {u}: (tt={kt[u]}, conc={kc[u]}, ph={kp[u]}) table={w[5][u]} K gpu={len(gb)} oracle={len(wb)} first diff at {j}")
            for name, bb, dd in (("gpu", gb, gd), ("ora", wb, wd)):
                seg = [(int(t.tt[b]), int(t.conc[b]), float(d), int(t.off[b+1]-t.off[b])) for b, d in zip(bb[max(0,j-2):j+3], dd[max(0,j-2):j+3])]
                print("   ", name, seg)
            print("    cum gpu", int(sum(t.off[b+1]-t.off[b] for b in gb)), "cum ora", int(sum(t.off[b+1]-t.off[b] for b in wb)))
print("mismatching keys:", bad, "of", n)
