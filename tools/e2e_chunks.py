import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_00616_b200 import LatencyOracle, OracleConfig
from paper_2605_00616_b200.device import DeviceTables
from paper_2605_00616_b200.profile import pack_from_device
from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, records_llama
t = DeviceTables.build(*records_llama(1_000_000, 0), canonical=True)
orc = LatencyOracle(pack_from_device(t, 1000, keep_host=False), OracleConfig(reliability_floor=32), _validate=False)
Q = 10_000_000
pin = lambda a: torch.as_tensor(a).pin_memory().numpy()
qt, qc, qp = (pin(a) for a in queries_llama(Q, 1))
us, ui = explicit_uniforms(Q, 1000)
us = pin(us.view(np.int64)).view(np.uint64); ui = pin(ui.view(np.int32)).view(np.uint32)
hl = torch.empty(Q, dtype=torch.float64).pin_memory().numpy()
def step():
    orc.flush(); orc.sample_batch(qt, qc, qp, rng="explicit", u_sel=us, u_idx=ui, seed=1, out_lat=hl, out_sidx=False)
for _ in range(2): step()
t0 = time.perf_counter()
for _ in range(8): step()
print(os.environ.get("EMU_HOST_CHUNK"), "e2e ms", (time.perf_counter() - t0) / 8 * 1e3)
