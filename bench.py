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
cpu_baseline: the reference's own CPU oracle (unmodified serve_emu LatencyOracle
             from baseline/_ref, one process per host core) on a bounded
             key-stratified sample; cpu_port: the C restatement (oracle/) on it

--impl reference runs that reference CPU oracle on the same workload, rank 0
only (the reference is Python: there is nothing to compile into oracle/_ref).
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
# library profiling name -> kernel (profiles/ncu_summary.json key) of the query-stream passes
STREAM_KERNELS = {"mark": "k_mark_bits", "sample": "k_sample", "sweep": "k_sweep", "sample_list": "k_sample_list"}
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
    ap.add_argument("--cpu-den", type=int, default=200,
                    help="CPU legs sample every query of 1/den of the key space (key_sample)")
    ap.add_argument("--cadence-calls", type=int, default=400, help="engine-cadence step calls for the p50")
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


REF_DIR = os.path.join(ROOT, "baseline", "_ref")  # the unmodified reference (baseline/install_ref.sh)


def key_sample(qt, qc, qp, den: int):
    """Indices of the queries whose KEY hashes into 1/den of the key space, in
    workload order.  Every selected key keeps all of its queries, so the sample
    has the full sweep's queries-per-pool ratio (~53 at C2): a cold CPU cache
    amortises each pool build over as many draws as the GPU sweep does."""
    import numpy as np

    k = ((qp.astype(np.uint64) << np.uint64(48)) | ((qt.astype(np.int64) & 0xFFFFFF).astype(np.uint64) << np.uint64(24))
         | (qc.astype(np.int64) & 0xFFFFFF).astype(np.uint64))
    h = (k * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(40)
    return np.flatnonzero(h % np.uint64(den) == 0)


_REF = {}  # set before fork: the reference pack + modules (workers inherit them)


def _ref_worker(conn, shard, floor, seed):
    RO, PH, pack = _REF["RO"], _REF["PH"], _REF["pack"]
    keys = [(int(t), int(c), PH[int(p)]) for t, c, p in zip(*shard)]
    while conn.recv() is not None:
        orc = RO.LatencyOracle(pack, RO.OracleConfig(reliability_floor=floor, rng_seed=seed))  # cold cache
        conn.send("ready")
        conn.recv()
        t0 = time.perf_counter()
        for t, c, ph in keys:
            orc.sample(t, c, ph)
        conn.send(time.perf_counter() - t0)


class ReferenceOracleArm:
    """The UNMODIFIED reference CPU oracle (serve_emu.oracle.LatencyOracle.sample,
    oracle.py:181-228, imported from baseline/_ref) on every host core: one
    process per core, each with its own cold LatencyOracle over the same pack
    and a disjoint set of keys (so each pool is built once, as in one cache).
    `step()` returns the wall time of one pass from a common start."""

    def __init__(self, soas, qt, qc, qp, floor, cores, seed=0):
        import multiprocessing as mp

        import numpy as np

        sys.path.insert(0, REF_DIR)
        import serve_emu.oracle as RO
        import serve_emu.profile as RP

        def table(kind, s):
            bk = [RP.Bucket(int(t), int(c), s.samples[s.off[i]:s.off[i + 1]].tolist())
                  for i, (t, c) in enumerate(zip(s.tt, s.conc))]
            return RP.PhaseTable.from_buckets(kind, bk)

        kinds = (RP.TableKind.DECODE, RP.TableKind.MIXED, RP.TableKind.COMBINED)
        pack = RP.ProfilePack(1000, *(table(k, s) for k, s in zip(kinds, soas)))
        pack.validate()
        _REF.update(RO=RO, PH=(RP.StepPhase.DECODE_ONLY, RP.StepPhase.PREFILL_OR_MIXED), pack=pack)
        ctx = mp.get_context("fork")
        owner = (qt.astype(np.int64) * 1_000_003 + qc.astype(np.int64) * 7 + qp) % cores  # keys -> one worker
        self.conns, self.procs = [], []
        for w in range(cores):
            sel = owner == w
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_ref_worker, args=(b, (qt[sel], qc[sel], qp[sel]), floor, seed), daemon=True)
            pr.start()
            self.conns.append(a)
            self.procs.append(pr)
        self.cores = cores

    def step(self) -> float:
        for c in self.conns:
            c.send("new")
        for c in self.conns:
            c.recv()
        t0 = time.perf_counter()
        for c in self.conns:
            c.send("go")
        for c in self.conns:
            c.recv()
        return time.perf_counter() - t0

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(timeout=5)


def ref_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "serve_emu"))


def sample_text(n, den, Q, n_keys):
    return (f"{n} queries = every query of 1/{den} of the key space ({n_keys} keys) of the {Q}-query workload, "
            f"in workload order (same queries per pool as the full sweep), cold pool cache")


def cpu_baseline(soas, qt, qc, qp, args, us=None, ui=None):
    """The reference's CPU oracle on a bounded key-stratified sample with every
    host core (kind "reference": the unmodified Python LatencyOracle); the C
    restatement (oracle/, "port") on the same sample alongside."""
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import emu_oracle as O  # noqa: E402  (checker / baseline only)

    cores = len(os.sched_getaffinity(0))
    sel = key_sample(qt, qc, qp, args.cpu_den)
    st, sc, sp = qt[sel], qc[sel], qp[sel]
    n_keys = len(np.unique((sp.astype(np.int64) << 48) | (st.astype(np.int64) << 24) | sc))
    txt = sample_text(len(sel), args.cpu_den, len(qt), n_keys)
    tabs = [O.Table(s.tt, s.conc, s.off, s.samples) for s in soas]
    t0 = time.perf_counter()
    O.sample_batch(tabs, st, sc, sp, args.floor, mode=args.rng, u_sel=None if us is None else us[sel],
                   u_idx=None if ui is None else ui[sel], seed=1, threads=cores)
    port = {"value": len(sel) / (time.perf_counter() - t0), "unit": "queries/s", "cores": cores, "kind": "port",
            "sample": txt + f"; C restatement (oracle/emu_oracle.c), {args.rng} uniforms, one cache per thread"}
    if not ref_available():
        return port, None
    arm = ReferenceOracleArm(soas, st, sc, sp, args.floor, cores)
    try:
        dt = arm.step()
    finally:
        arm.close()
    ref = {"value": len(sel) / dt, "unit": "queries/s", "cores": cores, "kind": "reference",
           "sample": txt + "; unmodified serve_emu.oracle.LatencyOracle.sample (baseline/_ref), one process and "
                           "one cold LatencyOracle per core over disjoint keys"}
    return ref, port


def run_reference(args):
    """--impl reference: the reference's own CPU oracle on the same workload
    (rank 0 only): the unmodified Python LatencyOracle from baseline/_ref on
    every host core, each step one cold pass over a key-stratified sample of
    the bench queries; the C restatement is timed beside it.  Falls back to the
    restatement (kind "port") when baseline/_ref is missing."""
    rank, size, _ = env_rank()
    if rank != 0:
        return
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import emu_oracle as O
    from paper_2605_00616_b200.profile import TableSoA
    from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, records_llama

    tabs = O.build(*records_llama(args.records, 0), canonical=True)
    soas = [TableSoA(t.tt, t.conc, t.off, t.samples) for t in tabs]
    cores = len(os.sched_getaffinity(0))
    qt, qc, qp = queries_llama(args.queries, 1)
    sel = key_sample(qt, qc, qp, args.cpu_den)
    n_keys = len(np.unique((qp[sel].astype(np.int64) << 48) | (qt[sel].astype(np.int64) << 24) | qc[sel]))
    st, sc, sp = qt[sel], qc[sel], qp[sel]
    n = len(sel)
    txt = sample_text(n, args.cpu_den, args.queries, n_keys)
    us, ui = explicit_uniforms(args.queries, 1000)
    t0 = time.perf_counter()
    O.sample_batch(tabs, st, sc, sp, args.floor, mode=args.rng, u_sel=us[sel], u_idx=ui[sel], seed=1, threads=cores)
    port = {"value": n / (time.perf_counter() - t0), "unit": "queries/s", "cores": cores, "kind": "port",
            "sample": txt + "; C restatement (oracle/emu_oracle.c)"}
    if ref_available():
        arm = ReferenceOracleArm(soas, st, sc, sp, args.floor, cores)
        times = []
        try:
            for k in range(args.warmup + args.steps):
                dt = arm.step()
                if k >= args.warmup:
                    times.append(dt)
        finally:
            arm.close()
        t = statistics.mean(times)
        cpu = {"value": n / t, "unit": "queries/s", "cores": cores, "kind": "reference",
               "sample": txt + "; unmodified serve_emu.oracle.LatencyOracle.sample (baseline/_ref), one process "
                               "and one cold LatencyOracle per core over disjoint keys"}
    else:
        t = n / port["value"]
        cpu = port
    v = n / t
    line = {"impl": "reference", "metric": "oracle queries/sec", "value": v, "unit": "queries/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "queries_per_step": n, "records": args.records, "floor": args.floor,
                       "rng": "pcg64 (the reference's own Generator)" if cpu is not port else args.rng},
            "cpu_baseline": dict(cpu), "cpu_port": port if cpu is not port else None,
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
        names = ("flush", "mark", "pool_prep", "tile_bin", "scan", "tile_scatter", "pool_tile", "pool_warp",
                 "pool_grp", "pool_cta", "sample", "sweep", "sample_list")

        def kernel_ms(fn, reps=2):
            _lib.profile_enable(True)
            for _ in range(reps):
                fn()
            out = {name: {"ms_per_step": 0.0, "launches_per_step": 0.0} for name in names}
            for name, (t, n) in _lib.profile_all().items():
                out[name] = {"ms_per_step": t / reps, "launches_per_step": n / reps}
            _lib.profile_enable(False)
            return out

        kern = kernel_ms(step)
        peak, peak_kind = measured_peak()
        bpq = BYTES_PER_QUERY[args.rng]
        step_ms = sum(v["ms_per_step"] for v in kern.values())
        # the passes over the query stream: k_mark + k_sample on the cold head,
        # k_sweep on the rest, k_sample_list on the sweep's misses
        stream = ("mark", "sample", "sweep", "sample_list")
        t_stream = sum(kern[k]["ms_per_step"] for k in stream) * 1e-3
        achieved = bpq * Q / t_stream / 1e9
        line["roofline"] = {"bound": "hbm", "kernel": "k_mark + k_sample + k_sweep + k_sample_list (query stream)",
                            "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                            "frac": achieved / peak,
                            # ncu DRAM bytes per launch x launches per step, for the kernels this step ran
                            "traffic": sum((ncu_metric(STREAM_KERNELS[k]) or 0.0) * kern[k]["launches_per_step"]
                                           for k in stream) or None,
                            "bytes_per_query": bpq,
                            "share_of_step": t_stream * 1e3 / max(step_ms, 1e-9),
                            "kernels_ms_per_step": {k: round(v["ms_per_step"], 4) for k, v in kern.items()},
                            "step_roofline_frac": bpq * Q / (ms / 1e3) / 1e9 / peak}
        # ---- warm step: the same sweep on a cache that holds every key (a long
        # what-if sweep's steady state): one k_sweep pass, nothing to build
        def warm_step():
            orc.sample_batch(qt, qc, qp, rng=args.rng, u_sel=us, u_idx=ui, seed=1, out_lat=lat, out_sidx=sidx)

        for _ in range(3):
            warm_step()
        torch.cuda.synchronize()
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nw = max(5, args.steps)
        w0.record()
        for _ in range(nw):
            warm_step()
        w1.record()
        torch.cuda.synchronize()
        wms = all_reduce_max(w0.elapsed_time(w1) / nw)
        wk = kernel_ms(warm_step)
        t_sw = wk["sweep"]["ms_per_step"] * 1e-3
        line["warm"] = {"value": size * Q / (wms / 1e3), "unit": "queries/s", "ms_per_step": wms,
                        "roofline": {"bound": "hbm", "kernel": "k_sweep", "achieved": bpq * Q / t_sw / 1e9,
                                     "peak": peak, "unit": "GB/s", "frac": bpq * Q / t_sw / 1e9 / peak,
                                     "traffic": ncu_metric("k_sweep"),
                                     "step_frac": bpq * Q / (wms / 1e3) / 1e9 / peak},
                        "kernels_ms_per_step": {k: round(v["ms_per_step"], 4) for k, v in wk.items()
                                                if v["launches_per_step"]},
                        "what": "same 10M queries, pool cache warm (no flush): LatencyOracle steady state"}
        # the pool build is per unique key and bound by instruction issue, not HBM:
        # its roofline is warp instructions (ncu count per launch, same build) /
        # CUDA-event time, summed over the pool-build kernels, vs the SMs' issue
        # rate (148 SMs x 4 schedulers x SM clock)
        pk = {"pool_prep": "k_pool_prep", "tile_bin": "k_tile_bin", "pool_tile": "k_pool_tile",
              "pool_warp": "k_pool_warp", "pool_grp": "k_pool_grp", "pool_cta": "k_pool_cta"}
        inst = {k: ncu_metric(v, "inst_executed") for k, v in pk.items()}
        have = [k for k in pk if inst[k] and kern[k]["launches_per_step"]]
        t_pool = sum(kern[k]["ms_per_step"] for k in pk) * 1e-3
        t_have = sum(kern[k]["ms_per_step"] for k in have) * 1e-3
        sm_hz = (clk.get("sm_mhz") or 1965.0) * 1e6
        i_sum = sum(inst[k] for k in have)
        line["roofline_pool_build"] = {
            "bound": "issue", "kernels": [pk[k] for k in have], "unit": "warp-inst/s",
            "achieved": i_sum / t_have if t_have > 0 else None, "peak": 148 * 4 * sm_hz,
            "frac": i_sum / t_have / (148 * 4 * sm_hz) if t_have > 0 else None,
            "inst_per_sweep": i_sum, "share_of_step": t_pool / max(step_ms * 1e-3, 1e-12),
            "note": "one pool per unique key (~189k keys per 10M-query cold sweep); no dense contraction, "
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
        # the e2e path's ceiling: pinned host -> device copy bandwidth, measured here
        hb = torch.empty(h2d, dtype=torch.uint8).pin_memory()
        db = torch.empty(h2d, dtype=torch.uint8, device="cuda")
        db.copy_(hb, non_blocking=True)
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        for _ in range(3):
            db.copy_(hb, non_blocking=True)
        p1.record()
        torch.cuda.synchronize()
        h2d_ms = p0.elapsed_time(p1) / 3
        del hb, db
        line["e2e"] = {"value": size * Q / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": Q * 8, "ms_per_step": e2e_s * 1e3,
                       "pcie": {"h2d_GBps": h2d / h2d_ms / 1e6, "h2d_floor_ms": h2d_ms,
                                "frac": h2d_ms / (e2e_s * 1e3),
                                "note": "the step's input bytes alone over PCIe (pinned, one copy) vs the e2e step"},
                       "api": "LatencyOracle.sample_batch(numpy pinned, latencies out) -> emu_oracle_sample_host "
                              "(2M-query chunks, copy-in / build+draw / copy-out on three streams)"}
        # ---- p50 latency of one engine-step query (LatencyOracle.__call__), cached keys
        if rank == 0:
            keys = list(zip(qt_h[:3000].tolist(), qc_h[:3000].tolist(), qp_h[:3000].tolist()))
            for k in keys[:300]:
                orc(*k)
            b2b = []
            for k in keys[300:]:  # back to back (no gap between calls)
                t0 = time.perf_counter()
                orc(*k)
                b2b.append((time.perf_counter() - t0) * 1e6)
            # at the engine's cadence: it sleeps each step's sampled latency before
            # the next backend call (engine.py:555-566), here ~7-100 ms
            cad = []
            for k in keys[300:300 + args.cadence_calls]:
                t0 = time.perf_counter()
                v = orc(*k)
                cad.append((time.perf_counter() - t0) * 1e6)
                time.sleep(v)
            orc.park()
            b2b.sort()
            cad.sort()
            pct = lambda a, q: a[min(len(a) - 1, int(len(a) * q))]  # noqa: E731
            line["p50_us_per_step_query"] = pct(cad, 0.5)
            line["p99_us_per_step_query"] = pct(cad, 0.99)
            line["step_query_latency"] = {
                "cadence": {"p50_us": pct(cad, 0.5), "p99_us": pct(cad, 0.99), "calls": len(cad),
                            "gap": "sleep(sampled latency) between calls, as EmulatorEngine does"},
                "back_to_back": {"p50_us": pct(b2b, 0.5), "p99_us": pct(b2b, 0.99), "calls": len(b2b)},
                "api": "LatencyOracle.__call__(tt, conc, phase) -> emu_oracle_step (resident step server)"}
            # ---- CPU baselines on this host (rank 0, N = 1 only)
            if size == 1:
                ref, port = cpu_baseline(tables.to_host(), qt_h, qc_h, qp_h, args, us_h, ui_h)
                line["cpu_baseline"] = ref
                if port is not None:
                    line["cpu_port"] = port
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
