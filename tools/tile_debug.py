"""Tile-tier debug: pools of in-grid keys vs the CPU oracle (small; run under compute-sanitizer)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import emu_oracle as O
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, build_pack_arrays
from paper_2605_00616_b200.workloads import records_llama, queries_llama

n_rec = int(os.environ.get("NREC", 200_000))
rec = records_llama(n_rec, 0)
pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
tabs = O.build(*rec, canonical=True)
qt, qc, qp = queries_llama(int(os.environ.get("NQ", 20_000)), 1)
keys = np.unique(np.stack([qt, qc, qp]).T, axis=0)
kt, kc, kp = keys[:, 0].astype(np.int32), keys[:, 1].astype(np.int32), keys[:, 2].astype(np.uint8)
orc = LatencyOracle(pack, OracleConfig(reliability_floor=32))
got = orc.pools(kt, kc, kp)
want = O.pools(tabs, kt, kc, kp, 32)
K0, K1 = np.diff(want[0]), np.diff(got[0])
bad = np.flatnonzero(K0 != K1)
print("keys", len(kt), "K mismatches", len(bad), [(int(kt[i]), int(kc[i]), int(kp[i]), int(K0[i]), int(K1[i])) for i in bad[:5]])
for name, a, b in zip(("off", "bkt", "dist", "prob", "cdf"), want, got):
    print(name, "equal" if np.array_equal(a, b) else "DIFF")
