import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, build_pack_arrays
from paper_2605_00616_b200.workloads import records_llama
rec = records_llama(1_000_000, 3)
pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
orc = LatencyOracle(pack, OracleConfig(reliability_floor=32))
rng = np.random.default_rng(int(os.environ.get("SEED", 5)))
n = int(os.environ.get("N", 2000))
kt = rng.integers(2049, 3000, n); kc = rng.integers(1, 257, n); kp = np.ones(n, np.int64)
ref = np.diff(orc.pools(kt, kc, kp)[0])
bad = 0
for r in range(int(os.environ.get("ROUNDS", 20))):
    K = np.diff(orc.pools(kt, kc, kp)[0])
    d = np.flatnonzero(K != ref)
    if len(d):
        bad += 1
        print("round", r, [(int(kt[j]), int(kc[j]), int(ref[j]), int(K[j])) for j in d[:4]])
print("N", n, "bad rounds", bad, "maxK", int(ref.max()))
