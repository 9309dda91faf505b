"""Small key-first canonical builds for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): mixed small / medium runs, large runs split into value
bins, and an over-full bin that falls back to the full passes."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2605_00616_b200.profile import build_pack_arrays

rng = np.random.default_rng(5)
n = 60_000
keys = rng.integers(0, 40, n)
conc = 1 + keys % 8
tt = conc + keys // 8
ph = rng.integers(0, 2, n)
cases = [(tt, conc, ph, np.exp(rng.normal(-4.0, 0.3, n)))]
k3 = rng.integers(0, 3, n)  # three keys: runs of ~10k records -> value bins
cases.append((1 + k3 + 2, 1 + k3, ph, np.exp(rng.normal(-4.0, 0.3, n))))
lat = np.exp(rng.normal(-4.0, 0.3, n))
lat[rng.random(n) < 0.5] = 0.02  # an over-full bin -> fallback
cases.append((1 + k3 + 2, 1 + k3, ph, lat))
for c in cases:
    pack = build_pack_arrays(*c, 4, canonical=True)
torch.cuda.synchronize()
print("san_kf ok")
