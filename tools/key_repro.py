"""Repro helper: one key's pool alone vs inside a 20k random batch, many times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, build_pack_arrays
from paper_2605_00616_b200.workloads import records_llama
rec = records_llama(1_000_000, 3)
pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
orc = LatencyOracle(pack, OracleConfig(reliability_floor=32))
key = (2556, 114, 1)
alone = [int(np.diff(orc.pools([key[0]], [key[1]], [key[2]])[0])[0]) for _ in range(30)]
print("alone K:", sorted(set(alone)))
rng = np.random.default_rng(5)
n = 20_000
kt = rng.integers(-10, 3000, n); kc = rng.integers(-3, 300, n); kp = rng.integers(0, 2, n)
i = int(np.flatnonzero((kt == key[0]) & (kc == key[1]) & (kp == key[2]))[0])
Ks = []
allK = None
for r in range(12):
    K = np.diff(orc.pools(kt, kc, kp)[0])
    Ks.append(int(K[i]))
    if allK is None:
        allK = K
    else:
        bad = np.flatnonzero(K != allK)
        if len(bad):
            print("round", r, "differs at", [(int(kt[j]), int(kc[j]), int(kp[j]), int(allK[j]), int(K[j])) for j in bad[:6]])
print("in batch K:", Ks)
