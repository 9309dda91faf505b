"""Config 5's oracle calls (scenario batches on a cache warming across scenarios): per-kernel totals."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
import bench_configs as B
from paper_2605_00616_b200 import _lib
from paper_2605_00616_b200.workloads import records_llama
_, orc = B.oracle_for(records_llama(1_000_000, 0), 32)
rates = np.geomspace(1, 64, 32); gammas = np.geomspace(0.125, 2, 16)
steps = 1_000_000
gen = torch.Generator(device="cuda"); gen.manual_seed(7)
lat = torch.empty(steps, dtype=torch.float64, device="cuda"); sidx = torch.empty(steps, dtype=torch.int32, device="cuda")
scen = [(r, g) for r in rates for g in gammas][: int(os.environ.get("SCEN", 128))]
orc.flush(); torch.cuda.synchronize()
_lib.profile_enable(True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = 0.0
for k, (r, g) in enumerate(scen):
    tt, cc, ph = B.scenario_keys(steps, r, g, gen)
    a.record(); orc.sample_batch(tt, cc, ph, rng="philox", seed=k, out_lat=lat, out_sidx=sidx); b.record(); b.synchronize()
    ms += a.elapsed_time(b)
kern = _lib.profile_all()
_lib.profile_enable(False)
print(os.environ.get("TAG", ""), "scenarios", len(scen), "ms", round(ms, 2), {k: (round(v[0], 2), v[1]) for k, v in sorted(kern.items(), key=lambda kv: -kv[1][0])})
