"""Per-kernel time of one canonical table build of N records (library events)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2605_00616_b200 import _lib
from paper_2605_00616_b200.device import DeviceTables
from paper_2605_00616_b200.workloads import records_llama
n = int(os.environ.get("N", 20_000_000))
parts = [records_llama(n // 4, 100 + k) for k in range(4)]
dev = [torch.as_tensor(np.concatenate([p[i] for p in parts]), device="cuda") for i in range(4)]
for _ in range(2):
    print("free GB before build", torch.cuda.mem_get_info()[0] / 1e9, flush=True)
    t = DeviceTables.build(*dev, canonical=True); del t
torch.cuda.synchronize()
_lib.profile_enable(True)
t0 = time.perf_counter()
t = DeviceTables.build(*dev, canonical=True)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
names = ["validate", "make_keys", "digit_hist", "radix_up", "radix_scatter", "scan", "index", "conc_range"]
tot = 0
for k in names:
    ms, c = _lib.profile_read(k)
    tot += ms
    print(f"{k:14s} {ms:8.3f} ms  {c} launches")
print(f"kernels {tot:.2f} ms, wall {wall * 1e3:.2f} ms for {n} records")
