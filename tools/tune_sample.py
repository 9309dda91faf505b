"""Time sampler variants (EMU_SAMPLE_VARIANT=qpt,hint) on the bench workload."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, json
sys.path.insert(0, %r)
import numpy as np, torch
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, _lib
from paper_2605_00616_b200.device import DeviceTables
from paper_2605_00616_b200.profile import pack_from_device
from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, records_llama
tables = DeviceTables.build(*records_llama(1_000_000, 0), canonical=True)
orc = LatencyOracle(pack_from_device(tables, 1000, keep_host=False), OracleConfig(reliability_floor=32), _validate=False)
Q = 10_000_000
qt, qc, qp = (torch.as_tensor(a, device="cuda") for a in queries_llama(Q, 1))
us, ui = explicit_uniforms(Q, 1000)
us = torch.as_tensor(us.view(np.int64), device="cuda"); ui = torch.as_tensor(ui.view(np.int32), device="cuda")
res = {}
for rng in ("explicit", "philox"):
    for _ in range(2):
        orc.flush(); orc.sample_batch(qt, qc, qp, rng=rng, u_sel=us, u_idx=ui)
    _lib.profile_enable(True)
    for _ in range(3):
        orc.flush(); orc.sample_batch(qt, qc, qp, rng=rng, u_sel=us, u_idx=ui)
    torch.cuda.synchronize()
    for k in ("mark", "sample"):
        t, n = _lib.profile_read(k); res[rng + "_" + k] = round(t / n, 4)
    # warm cache (no flush)
    for _ in range(3):
        orc.sample_batch(qt, qc, qp, rng=rng, u_sel=us, u_idx=ui)
    torch.cuda.synchronize()
    for k in ("mark", "sample"):
        t, n = _lib.profile_read(k); res[rng + "_warm_" + k] = round(t / n, 4)
    _lib.profile_enable(False)
print(json.dumps(res))
''' % ROOT
for var in sys.argv[1:] or ["1,1", "1,0", "2,1", "4,1"]:
    env = dict(os.environ, EMU_SAMPLE_VARIANT=var)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(var, out.stdout.strip()[-400:], out.stderr.strip()[-300:])
