"""Closed-loop sweep throughput vs horizon, with the scheduler's per-phase cycle
counters (EMU_SCHED_PROF=1 prints them to stderr when each run's scheduler is
destroyed).  STEPS="20000 100000" SCEN=512 python tools/sweep_scaling.py"""
import gc, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("EMU_SCHED_PROF", "1")
import torch
import bench_configs as B


class A:
    pass


for st in [int(x) for x in os.environ.get("STEPS", "20000 100000").split()]:
    a = A()
    a.steps_sweep = st
    a.scenarios = int(os.environ.get("SCEN", 512))
    r = B.sweep(a)
    gc.collect()
    torch.cuda.synchronize()
    print(st, {k: v for k, v in r.items() if k in ("steps_total", "wall_s", "steps_per_s", "rounds", "requests")},
          flush=True)
    sys.stderr.flush()
