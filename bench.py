#!/usr/bin/env python
"""Benchmark: batched oracle sweep on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (per GPU, weak scaling): a 1M-record Llama-3.1-8B-shaped profile
(generator G(0), built on the GPU, replicated to every rank by NCCL broadcast)
and 10M query keys from G(1 + rank).  One step = one cold sweep: flush the pool
cache, then dedupe + pool build + sample all 10M queries (LatencyOracle's lazy
cache semantics, timed together).  Inputs (10M x 21 B = 210 MB) exceed the
126 MB L2, so no explicit L2 flush is needed between steps.

value      : queries/s over all ranks (device time: CUDA events, max over ranks)
e2e        : same metric through LatencyOracle.sample_batch with pinned HOST
             query/uniform buffers; H2D + D2H inside the timed region
roofline   : dominant kernel's algorithmic bytes / its CUDA-event duration vs
             MEASURED_PEAKS.json hbm_gbs
cpu_baseline: the CPU restatement (oracle/, "port") on a bounded sample, all host cores

--impl reference runs the CPU oracle port (the reference is Python: there is
nothing to compile into oracle/_ref) on the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_QUERY = {"explicit": 41, "philox": 29}
WORKLOAD = ("C2: 10M-query batched oracle sweep over a 1M-record Llama-3.1-8B-shaped profile table "
            "(synthetic generator G, M=32, p=2, eps=1e-9), cold pool cache per step")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--queries", type=int, default=10_000_000, help="queries per GPU per step")
    ap.add_argument("--records", type=int, default=1_000_000)
    ap.add_argument("--floor", type=int, default=32)
    ap.add_argument("--rng", default="explicit", choices=["explicit", "philox"])
    ap.add_argument("--cpu-sample", type=int, default=100_000, help="queries in the CPU baseline sample")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / roofline / cpu / p50 legs")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher + collectives only, on CPU over gloo (no kernels): tests/test_dist.py")
    return ap.parse_args()


def launch_ranks(args) -> bool:
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec under
    torch.distributed.run with N ranks on this node (one process per GPU,
    rendezvous on 127.0.0.1).  Returns False when already a rank."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def run_dry(args):
    """The multi-rank plumbing of run_b200 on CPU (gloo): rank env, the packed
    table broadcast, query shards, barrier-bracketed timing with the max over
    ranks, and rank 0's JSON line.  No kernels run (and none are claimed)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import emu_oracle as O  # stand-in table builder on CPU (test only)
    from paper_2605_00616_b200.dist import all_reduce_max, broadcast_soas
    from paper_2605_00616_b200.profile import TableSoA
    from paper_2605_00616_b200.workloads import queries_llama, records_llama

    rank, size, _ = env_rank()
    if size > 1:
        dist.init_process_group("gloo")
    soas = None
    if rank == 0:
        soas = [TableSoA(t.tt, t.conc, t.off, t.samples) for t in O.build(*records_llama(args.records, 0),
                                                                          canonical=True)]
    got = broadcast_soas(soas, 0, "cpu") if size > 1 else None
    nb = [int(g[0].numel()) for g in got] if got else [len(s.tt) for s in soas]
    Q = args.queries
    qt, _, _ = queries_llama(Q, 1 + rank)
    if size > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        np.sort(qt)  # placeholder work per step
    ms = all_reduce_max((time.perf_counter() - t0) * 1e3 / max(args.steps, 1), device="cpu")
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": size, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": ms, "queries_per_rank": Q, "buckets": nb, "gpu_launches": 0}), flush=True)
    if size > 1:
        dist.barrier()
        dist.destroy_process_group()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 20 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_metric(kernel: str, key: str = "dram_bytes"):
    """Per-launch metric of `kernel` from the committed ncu summary (profiles/), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            return json.load(f).get(kernel, {}).get(key)
    except (OSError, ValueError):
        return None


def cpu_baseline(tabs, qt, qc, qp, args, us=None, ui=None):
    """The CPU restatement on a bounded sample with every host core."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import emu_oracle as O  # noqa: E402  (checker / baseline only)

    cores = len(os.sched_getaffinity(0))
    n = min(args.cpu_sample, len(qt))
    t0 = time.perf_counter()
    O.sample_batch(tabs, qt[:n], qc[:n], qp[:n], args.floor, mode=args.rng, u_sel=None if us is None else us[:n],
                   u_idx=None if ui is None else ui[:n], seed=1, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "queries/s", "cores": cores, "kind": "port",
            "sample": f"first {n} queries of the workload, cold pool cache per thread, {args.rng} uniforms, "
                      f"{cores} threads (one LatencyOracle-equivalent cache each)"}


def run_reference(args):
    """--impl reference: the CPU oracle port on the same workload (rank 0 only)."""
    rank, size, _ = env_rank()
    if rank != 0:
        return
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import emu_oracle as O
    from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, records_llama

    rec = records_llama(args.records, 0)
    tabs = O.build(*rec, canonical=True)
    cores = len(os.sched_getaffinity(0))
    n = args.cpu_sample
    qt, qc, qp = queries_llama(n, 1)
    us, ui = explicit_uniforms(n, 2)
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.sample_batch(tabs, qt, qc, qp, args.floor, mode=args.rng, u_sel=us, u_idx=ui, seed=1, threads=cores)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    v = n / t
    line = {"impl": "reference", "metric": "oracle queries/sec", "value": v, "unit": "queries/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "queries_per_step": n, "records": args.records, "floor": args.floor,
                       "rng": args.rng},
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "port",
                             "sample": f"{n} queries of the workload per step, cold cache per thread"},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_00616_b200 import LatencyOracle, OracleConfig, _lib
    from paper_2605_00616_b200.device import DeviceTables
    from paper_2605_00616_b200.dist import all_reduce_max, broadcast_tables
    from paper_2605_00616_b200.profile import pack_from_device
    from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, records_llama

    rank, size, local = env_rank()
    torch.cuda.set_device(local)
    if size > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # ---- table: GPU build on rank 0, one NCCL broadcast to the rest
    rec = records_llama(args.records, 0) if rank == 0 else None
    tables = DeviceTables.build(*rec, canonical=True) if rank == 0 else None
    tables = broadcast_tables(tables)
    pack = pack_from_device(tables, 1000, keep_host=False)
    orc = LatencyOracle(pack, OracleConfig(reliability_floor=args.floor), _validate=False)
    # ---- this rank's queries (weak scaling: Q per GPU)
    Q = args.queries
    qt_h, qc_h, qp_h = queries_llama(Q, 1 + rank)
    us_h, ui_h = explicit_uniforms(Q, 1000 + rank)
    qt, qc, qp = (torch.as_tensor(a, device="cuda") for a in (qt_h, qc_h, qp_h))
    us = torch.as_tensor(us_h.view(np.int64), device="cuda")
    ui = torch.as_tensor(ui_h.view(np.int32), device="cuda")
    lat = torch.empty(Q, dtype=torch.float64, device="cuda")
    sidx = torch.empty(Q, dtype=torch.int32, device="cuda")

    def step():
        orc.flush()
        orc.sample_batch(qt, qc, qp, rng=args.rng, u_sel=us, u_idx=ui, seed=1, out_lat=lat, out_sidx=sidx)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if size > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    if size > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = all_reduce_max(ms_local)
    value = size * Q / (ms / 1e3)
    line = {"metric": "oracle queries/sec", "value": value, "unit": "queries/s", "n_gpus": size,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "queries_per_gpu": Q, "records": args.records, "floor": args.floor,
                       "rng": args.rng, "parallelism": f"dp{size} (query shards, table replicated by NCCL broadcast)",
                       "l2": "inputs 210 MB/step > 126 MB L2; no flush needed"},
            "clocks": clk, "gpu_launches": int(launches)}
    if not args.no_extras:
        # ---- roofline: per-kernel CUDA events recorded by the library on the launch stream
        _lib.profile_enable(True)
        for _ in range(2):
            step()
        kern = {}
        for name in ("flush", "mark", "pool_prep", "tile_bin", "scan", "tile_scatter", "pool_tile", "pool_warp", "pool_grp",
                     "pool_cta", "sample"):
            t, n = _lib.profile_read(name)
            kern[name] = {"ms_per_launch": t / max(n, 1), "launches": n}
        _lib.profile_enable(False)
        peak, peak_kind = measured_peak()
        bpq = BYTES_PER_QUERY[args.rng]
        t_sample = kern["sample"]["ms_per_launch"] * 1e-3
        achieved = bpq * Q / t_sample / 1e9
        step_ms = sum(v["ms_per_launch"] * v["launches"] for v in kern.values()) / 2
        line["roofline"] = {"bound": "hbm", "kernel": "k_sample", "achieved": achieved, "peak": peak,
                            "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                            "traffic": ncu_metric("k_sample"), "bytes_per_query": bpq,
                            "share_of_step": kern["sample"]["ms_per_launch"] / max(step_ms, 1e-9),
                            "kernels_ms": {k: round(v["ms_per_launch"], 4) for k, v in kern.items()},
                            "step_roofline_frac": bpq * Q / (ms / 1e3) / 1e9 / peak}
        # the pool build is per unique key and bound by instruction issue, not HBM:
        # its roofline is warp instructions (ncu count per launch) / time vs the
        # SMs' issue rate (148 SMs x 4 schedulers x SM clock)
        inst = ncu_metric("k_pool_warp", "inst_executed")
        t_pw = kern["pool_warp"]["ms_per_launch"] * 1e-3
        sm_hz = (clk.get("sm_mhz") or 1965.0) * 1e6
        line["roofline_pool_build"] = {
            "bound": "issue", "kernel": "k_pool_warp", "unit": "warp-inst/s",
            "achieved": (inst / t_pw) if inst and t_pw > 0 else None, "peak": 148 * 4 * sm_hz,
            "frac": (inst / t_pw / (148 * 4 * sm_hz)) if inst and t_pw > 0 else None,
            "inst_per_launch": inst, "share_of_step": kern["pool_warp"]["ms_per_launch"] / max(step_ms, 1e-9),
            "note": "one pool per unique key (189k keys per 10M-query cold sweep); no dense contraction, "
                    "no streaming: issue- and L2-latency-bound (DESIGN.md section 6)"}
        # ---- e2e through the public API with pinned host buffers
        pin = lambda a: torch.as_tensor(a).pin_memory().numpy()  # noqa: E731
        hq = [pin(a) for a in (qt_h, qc_h, qp_h)]
        hu = pin(us_h.view(np.int64)).view(np.uint64), pin(ui_h.view(np.int32)).view(np.uint32)
        hl = torch.empty(Q, dtype=torch.float64).pin_memory().numpy()

        def e2e_step():
            orc.flush()
            orc.sample_batch(*hq, rng=args.rng, u_sel=hu[0], u_idx=hu[1], seed=1, out_lat=hl, out_sidx=False)

        e2e_step()
        if size > 1:
            dist.barrier()
        t0 = time.perf_counter()
        n_e2e = min(20, max(3, args.steps // 2))
        for _ in range(n_e2e):
            e2e_step()
        e2e_s = (time.perf_counter() - t0) / n_e2e
        e2e_s = all_reduce_max(e2e_s)
        h2d = Q * (4 + 4 + 1 + (12 if args.rng == "explicit" else 0))
        line["e2e"] = {"value": size * Q / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": Q * 8, "ms_per_step": e2e_s * 1e3,
                       "api": "LatencyOracle.sample_batch(numpy pinned, latencies out) -> emu_oracle_sample_host "
                              "(1M-query chunks, copy-in / build+draw / copy-out on three streams)"}
        # ---- p50 latency of one engine-step query (LatencyOracle.__call__)
        if rank == 0:
            keys = list(zip(qt_h[:3000].tolist(), qc_h[:3000].tolist(), qp_h[:3000].tolist()))
            for k in keys[:300]:
                orc(*k)
            lat_us = []
            for k in keys[300:]:
                t0 = time.perf_counter()
                orc(*k)
                lat_us.append((time.perf_counter() - t0) * 1e6)
            lat_us.sort()
            line["p50_us_per_step_query"] = lat_us[len(lat_us) // 2]
            line["p99_us_per_step_query"] = lat_us[int(len(lat_us) * 0.99)]
            # ---- CPU baseline on this host (rank 0, N = 1 only)
            if size == 1:
                sys.path.insert(0, os.path.join(ROOT, "oracle"))
                import emu_oracle as O  # checker / baseline only

                tabs_h = [O.Table(s.tt, s.conc, s.off, s.samples) for s in tables.to_host()]
                line["cpu_baseline"] = cpu_baseline(tabs_h, qt_h, qc_h, qp_h, args, us_h, ui_h)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if size > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    launch_ranks(args)
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
