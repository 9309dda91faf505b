"""One cold C3 sweep (sparse long-context table, 1M records) at FLOOR (default 256), for ncu."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2605_00616_b200 import LatencyOracle, OracleConfig
from paper_2605_00616_b200.device import DeviceTables
from paper_2605_00616_b200.profile import pack_from_device
from paper_2605_00616_b200.workloads import queries_sparse, records_sparse

Q = int(os.environ.get("Q", 10_000_000))
floor = int(os.environ.get("FLOOR", 256))
tables = DeviceTables.build(*records_sparse(1_000_000, 0), canonical=True)
orc = LatencyOracle(pack_from_device(tables, 1000, keep_host=False), OracleConfig(reliability_floor=floor), _validate=False)
dq = [torch.as_tensor(a, device="cuda") for a in queries_sparse(Q, 1)]
def sweep():
    orc.flush()
    orc.sample_batch(*dq, rng="philox", seed=1)

sweep()
torch.cuda.synchronize()
n = int(os.environ.get("SWEEPS", 1))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(n):
    sweep()
b.record()
torch.cuda.synchronize()
print(os.environ.get("TAG", ""), "floor", floor, "ms/sweep", a.elapsed_time(b) / n, flush=True)
