"""One warm-up + N profiled cold sweeps of the bench workload (for ncu)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2605_00616_b200 import LatencyOracle, OracleConfig
from paper_2605_00616_b200.device import DeviceTables
from paper_2605_00616_b200.profile import pack_from_device
from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, records_llama

Q = int(os.environ.get("Q", 10_000_000))
sweeps = int(os.environ.get("SWEEPS", 2))
rng = os.environ.get("RNG", "explicit")
tables = DeviceTables.build(*records_llama(1_000_000, 0), canonical=True)
orc = LatencyOracle(pack_from_device(tables, 1000, keep_host=False), OracleConfig(reliability_floor=32), _validate=False)
qt, qc, qp = (torch.as_tensor(a, device="cuda") for a in queries_llama(Q, 1))
us, ui = explicit_uniforms(Q, 1000)
us = torch.as_tensor(us.view(np.int64), device="cuda"); ui = torch.as_tensor(ui.view(np.int32), device="cuda")
for _ in range(sweeps):
    orc.flush()
    lat, sidx = orc.sample_batch(qt, qc, qp, rng=rng, u_sel=us, u_idx=ui, seed=1)
for _ in range(int(os.environ.get("WARM", 0))):  # warm sweeps (no flush): one k_sweep pass each
    lat, sidx = orc.sample_batch(qt, qc, qp, rng=rng, u_sel=us, u_idx=ui, seed=1)
torch.cuda.synchronize()
print("slots used", orc.cached_slots())
