"""Warm C2 sweeps (every key cached): step time and per-kernel times (CUDA events)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, _lib
from paper_2605_00616_b200.device import DeviceTables
from paper_2605_00616_b200.profile import pack_from_device
from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, records_llama
Q = 10_000_000
tables = DeviceTables.build(*records_llama(1_000_000, 0), canonical=True)
orc = LatencyOracle(pack_from_device(tables, 1000, keep_host=False), OracleConfig(reliability_floor=32), _validate=False)
qt, qc, qp = (torch.as_tensor(a, device="cuda") for a in queries_llama(Q, 1))
us, ui = explicit_uniforms(Q, 1000)
us = torch.as_tensor(us.view(np.int64), device="cuda"); ui = torch.as_tensor(ui.view(np.int32), device="cuda")
lat = torch.empty(Q, dtype=torch.float64, device="cuda"); sidx = torch.empty(Q, dtype=torch.int32, device="cuda")
step = lambda: orc.sample_batch(qt, qc, qp, rng="explicit", u_sel=us, u_idx=ui, seed=1, out_lat=lat, out_sidx=sidx)
for _ in range(3):
    step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    step()
b.record(); torch.cuda.synchronize()
_lib.profile_enable(True)
for _ in range(5):
    step()
k = {n: round(t / 5, 4) for n, (t, c) in _lib.profile_all().items()}
_lib.profile_enable(False)
print(os.environ.get("TAG", ""), "warm step ms", round(a.elapsed_time(b) / 20, 4), k, flush=True)
