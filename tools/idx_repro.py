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
kt = rng.integers(-10, 140_000 if sparse else 3000, n); kc = rng.integers(-3, 300, n); kp = rng.integers(0, 2, n)
ref = None
for r in range(int(os.environ.get("ROUNDS", 4))):
    pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
    orc = LatencyOracle(pack, OracleConfig(reliability_floor=int(os.environ.get('FLOOR', 32))))
    out = orc.pools(kt, kc, kp)
    if ref is None:
        ref = out
    else:
        assert all(np.array_equal(a, b) for a, b in zip(ref, out)), "pools differ between rounds"
print(os.environ.get("IDX"), "ok")
