"""Where the closed-loop sweep spends its time (library CUDA events per kernel)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench_configs as B
from paper_2605_00616_b200 import _lib
class A: pass
a = A(); a.steps_sweep = int(os.environ.get("STEPS", 2000)); a.scenarios = int(os.environ.get("SCEN", 512))
_lib.profile_enable(True)
r = B.sweep(a)
torch.cuda.synchronize()
print({k: v for k, v in r.items() if k in ("steps_total", "wall_s", "steps_per_s", "rounds")})
for k in ("sched", "mark", "pool_prep", "pool_warp", "pool_grp", "pool_cta", "flush"):
    ms, n = _lib.profile_read(k)
    print(f"{k:10s} {ms:10.1f} ms {n} launches")
