"""Repro helper: pools of 20k random keys over GPU-built packs, N rounds (IDX=host|dev)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
os.environ["EMU_INDEX_HOST"] = "1" if os.environ.get("IDX") == "host" else "0"
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, build_pack_arrays
from paper_2605_00616_b200.workloads import records_llama, records_sparse
sparse = os.environ.get('GEN') == 'sparse'
rec = (records_sparse if sparse else records_llama)(1_000_000, 3)
rng = np.random.default_rng(5)
n = 20_000
ingrid = os.environ.get("INGRID") == "1"
if ingrid:
    kt = rng.integers(1, 131_072 if sparse else 2048, n); kc = rng.integers(1, 256, n)
else:
    kt = rng.integers(-10, 140_000 if sparse else 3000, n); kc = rng.integers(-3, 300, n)
kp = rng.integers(0, 2, n)
ref = None
for r in range(int(os.environ.get("ROUNDS", 4))):
    pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
    orc = LatencyOracle(pack, OracleConfig(reliability_floor=int(os.environ.get('FLOOR', 32))))
    out = orc.pools(kt, kc, kp)
    if ref is None:
        ref = out
    elif not all(np.array_equal(a, b) for a, b in zip(ref, out)):
        K0, K1 = np.diff(ref[0]), np.diff(out[0])
        bad = np.flatnonzero(K0 != K1)
        print("round", r, "K differs for", len(bad), "keys; first:",
              [(int(kt[i]), int(kc[i]), int(kp[i]), int(K0[i]), int(K1[i])) for i in bad[:8]])
        if not len(bad):
            for name, a, b in zip(("off", "bkt", "dist", "prob", "cdf", "tid"), ref, out):
                if not np.array_equal(a, b):
                    d = np.flatnonzero(a != b)
                    key = np.searchsorted(ref[0], d[:5], side="right") - 1
                    print(name, "differs at", d[:5].tolist(), "keys", [(int(kt[k]), int(kc[k]), int(kp[k]), int(K0[k])) for k in key])
        raise SystemExit("pools differ between rounds")
print(os.environ.get("IDX"), "ok")
