"""Per-phase cycle accounting of the pool build (needs the EMU_STATS library build)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["EMU_LIB_PATH"] = os.path.join(ROOT, "paper_2605_00616_b200/csrc/build/libemu_b200_stats.so")
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, _lib
from paper_2605_00616_b200.device import DeviceTables
from paper_2605_00616_b200.profile import pack_from_device
from paper_2605_00616_b200.workloads import queries_llama, records_llama, queries_sparse, records_sparse
floor = int(os.environ.get("FLOOR", 32))
sparse = os.environ.get('WORK') == 'sparse'
tables = DeviceTables.build(*(records_sparse if sparse else records_llama)(1_000_000, 0), canonical=True)
orc = LatencyOracle(pack_from_device(tables, 1000, keep_host=False), OracleConfig(reliability_floor=floor), _validate=False)
qt, qc, qp = (torch.as_tensor(a, device="cuda") for a in (queries_sparse if sparse else queries_llama)(int(os.environ.get('Q', 10_000_000)), 1))
lib = _lib.lib(); lib.emu_stats_read.argtypes = [ctypes.c_void_p]
buf = np.zeros(32, np.uint64)
orc.flush(); orc.sample_batch(qt, qc, qp, rng="philox"); torch.cuda.synchronize()
lib.emu_stats_read(buf.ctypes.data)
keys = int(buf[11])
names = ["radius", "refine", "window", "enumerate", "sort", "prefix", "finish"]
print("exact-resort", int(buf[12]), "wide->slow", int(buf[13]))
print("keys", keys, "avg C_sat %.1f  avg pos %.1f  avg K %.1f" % (buf[8] / keys, buf[9] / keys, buf[10] / keys))
tot = sum(int(buf[i]) for i in range(7))
for i, n in enumerate(names):
    print(f"{n:10s} {buf[i] / keys:9.0f} cycles/key  {100 * int(buf[i]) / tot:5.1f}%")
tiles, cu = int(buf[16]), int(buf[17])
if tiles:
    tk = int(buf[22]) + int(buf[19]) + int(buf[20]) + int(buf[21]) + int(buf[18])
    print("tile tier: tiles %d  avg union %.1f  keys %d  ok %d  fallback: union %d  list %d  prefix %d  window %d  avg list %.1f"
          % (tiles, cu / tiles, tk, buf[22], buf[18], buf[19], buf[20], buf[21], buf[23] / max(1, tk - int(buf[18]))))
