"""Which keys' pools differ from the oracle (floor 256, C1 pack): K, first differing index, field."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import emu_oracle as O
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, build_pack_arrays
from paper_2605_00616_b200.workloads import records_llama
rec = records_llama(50_000, 0)
pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
tabs = [O.Table(s.tt, s.conc, s.off, s.samples) for s in pack.soas()]
floor = int(os.environ.get("FLOOR", 256))
rng = np.random.default_rng(floor)
n = 400
kt = rng.integers(-5, 3000, n); kc = rng.integers(-3, 300, n); kp = rng.integers(0, 2, n)
orc = LatencyOracle(pack, OracleConfig(reliability_floor=floor))
got = orc.pools(kt, kc, kp)
want = O.pools(tabs, kt, kc, kp, floor, p=2.0)
off = want[0]
bad = 0
for u in range(n):
    a, b = off[u], off[u + 1]
    for f, name in ((3, "prob"), (4, "cdf"), (2, "dist")):
        if not np.array_equal(got[f][a:b], want[f][a:b]):
            d = np.flatnonzero(got[f][a:b] != want[f][a:b])
            print(f"key {u} ({kt[u]},{kc[u]},{kp[u]}) K={b - a} {name} differs at {d[:8]} got {got[f][a + d[0]]!r} want {want[f][a + d[0]]!r}")
            bad += 1
            break
print("bad keys", bad)
