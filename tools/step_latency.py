"""p50/p99 of LatencyOracle.__call__ (the engine's per-step backend call) on the C2 table."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2605_00616_b200 import LatencyOracle, OracleConfig
from paper_2605_00616_b200.device import DeviceTables
from paper_2605_00616_b200.profile import pack_from_device
from paper_2605_00616_b200.workloads import queries_llama, records_llama
t = DeviceTables.build(*records_llama(1_000_000, 0), canonical=True)
orc = LatencyOracle(pack_from_device(t, 1000, keep_host=False), OracleConfig(reliability_floor=32), _validate=False)
qt, qc, qp = queries_llama(20_000, 1)
keys = list(zip(qt.tolist(), qc.tolist(), qp.tolist()))
for k in keys[:3000]:
    orc(*k)
us = []
for k in keys[3000:]:
    t0 = time.perf_counter()
    orc(*k)
    us.append((time.perf_counter() - t0) * 1e6)
us.sort()
print("p50 %.2f us  p90 %.2f  p99 %.2f  (n=%d)" % (us[len(us) // 2], us[int(0.9 * len(us))], us[int(0.99 * len(us))], len(us)))
t0 = time.perf_counter(); torch.cuda.synchronize(); print("device sync after steps: %.1f us" % ((time.perf_counter() - t0) * 1e6))
# raw C-ABI call cost (no Python argument handling)
import ctypes
from paper_2605_00616_b200 import _lib
fn = _lib.lib().emu_oracle_step
out = ctypes.c_double(); ref = ctypes.byref(out); h = orc._h
args = [(ctypes.c_int32(a), ctypes.c_int32(b), ctypes.c_int32(c)) for a, b, c in keys[3000:]]
us = []
for a, b, c in args:
    t0 = time.perf_counter()
    fn(h, a, b, c, ref)
    us.append((time.perf_counter() - t0) * 1e6)
us.sort()
print("raw ABI p50 %.2f us  p90 %.2f" % (us[len(us) // 2], us[int(0.9 * len(us))]))
t0 = time.perf_counter()
for _ in range(10000):
    pass
print("python loop overhead per iter %.3f us" % ((time.perf_counter() - t0) * 100))
