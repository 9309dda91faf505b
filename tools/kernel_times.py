"""Per-kernel library CUDA-event times over N cold sweeps of the bench workload
(C2: 1M records, 10M queries).  Knob sweeps: run under different EMU_* env values.
    SWEEPS=10 python tools/kernel_times.py"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, _lib
from paper_2605_00616_b200.device import DeviceTables
from paper_2605_00616_b200.profile import pack_from_device
from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, records_llama

Q = int(os.environ.get("Q", 10_000_000))
sweeps = int(os.environ.get("SWEEPS", 10))
rng = os.environ.get("RNG", "explicit")
tables = DeviceTables.build(*records_llama(1_000_000, 0), canonical=True)
orc = LatencyOracle(pack_from_device(tables, 1000, keep_host=False), OracleConfig(reliability_floor=32), _validate=False)
qt, qc, qp = (torch.as_tensor(a, device="cuda") for a in queries_llama(Q, 1))
us, ui = explicit_uniforms(Q, 1000)
us = torch.as_tensor(us.view(np.int64), device="cuda"); ui = torch.as_tensor(ui.view(np.int32), device="cuda")
lat = torch.empty(Q, dtype=torch.float64, device="cuda")
for _ in range(3):
    orc.flush()
    orc.sample_batch(qt, qc, qp, rng=rng, u_sel=us, u_idx=ui, seed=1, out_lat=lat)
torch.cuda.synchronize()
_lib.profile_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(sweeps):
    orc.flush()
    orc.sample_batch(qt, qc, qp, rng=rng, u_sel=us, u_idx=ui, seed=1, out_lat=lat)
e1.record()
torch.cuda.synchronize()
out = {"step_ms": e0.elapsed_time(e1) / sweeps}
for k, (ms, n) in sorted(_lib.profile_all().items()):
    out[k] = round(ms / sweeps, 4)
print(os.environ.get("TAG", ""), out, flush=True)
