#!/usr/bin/env python
"""Secondary measurements for BASELINE.json configs 1, 3, 4, 5 (one JSON line each).

The driver's headline is bench.py (config 2).  This script measures the
other configs on one GPU so every SURVEY §8 row has a number:

  c1  C1 pack (50k records) + the 10k-step reference-scheduler trace
      (tests/golden/c1_trace.npz): PCG64 stream replay (bit-exact with the
      reference LatencyOracle), batched Philox draws, and the per-step
      LatencyOracle.__call__ latency.  CPU: the oracle port, same queries.
  c3  sparse long-context profile (1M records, tt <= 131072), 10M queries,
      M = 32 and M = 256, cold sweeps.
  c4  offline table build from 100M synthetic records (device-resident
      inputs), canonical order; records/s and the build's HBM bytes/s.
  codec  pack JSON load and trace JSONL ingest, native vs the reference's json path
  c5  what-if sweep: 512 scenarios (32 request rates x 16 burstiness
      values) x 1M steps, keys generated on the GPU per scenario, Philox
      draws; plus the synthetic token fill over 256M entries.

    python bench_configs.py [c1 c3 c4 c5 codec sweep] [--steps K]
    torchrun --nproc-per-node N bench_configs.py c4 sweep   (range-partitioned build, sharded sweep)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import torch  # noqa: E402

import emu_oracle as O  # noqa: E402  (CPU baseline only)
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, _lib, token_fill  # noqa: E402
from paper_2605_00616_b200.device import DeviceTables  # noqa: E402
from paper_2605_00616_b200.profile import pack_from_device  # noqa: E402
from paper_2605_00616_b200.workloads import (  # noqa: E402
    explicit_uniforms,
    queries_sparse,
    records_llama,
    records_sparse,
)

CORES = len(os.sched_getaffinity(0))


def timed(fn, steps, warmup=2):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def oracle_for(rec, floor):
    t = DeviceTables.build(*rec, canonical=True)
    return t, LatencyOracle(pack_from_device(t, 1000, keep_host=False), OracleConfig(reliability_floor=floor),
                            _validate=False)


def c1(args):
    tr = np.load(os.path.join(ROOT, "tests", "golden", "c1_trace.npz"))
    qt, qc, qp = tr["tt"], tr["conc"], tr["phase"]
    rec = records_llama(50_000, 0)
    tables, orc = oracle_for(rec, 32)
    golden = np.load(os.path.join(ROOT, "tests", "golden", "c1_golden.npz"))["lat_seq"]

    def replay():
        orc.flush()
        orc.set_rng_state(np.random.default_rng(0).bit_generator.state)
        return orc.sample_batch(qt, qc, qp, rng="pcg64")

    lat, _ = replay()
    exact = bool(np.array_equal(lat, golden))
    ms_replay = timed(replay, args.steps)
    dq = [torch.as_tensor(a, device="cuda") for a in (qt, qc, qp)]

    def batched():
        orc.flush()
        orc.sample_batch(*dq, rng="philox", seed=1)

    ms_batch = timed(batched, args.steps)
    keys = list(zip(qt.tolist(), qc.tolist(), qp.tolist()))
    for k in keys[:500]:
        orc(*k)
    us = []
    for k in keys[500:3500]:
        t0 = time.perf_counter()
        orc(*k)
        us.append((time.perf_counter() - t0) * 1e6)
    us.sort()
    tabs = O.build(*rec, canonical=True)
    t0 = time.perf_counter()
    O.sample_pcg64(tabs, qt, qc, qp, 32, state6=O.pcg64_state6(0))
    cpu_s = time.perf_counter() - t0
    return {"config": "c1", "workload": "50k-record pack, 10k reference-scheduler step keys (312 unique), M=32",
            "pcg64_replay_ms": ms_replay, "pcg64_replay_queries_per_s": len(qt) / (ms_replay / 1e3),
            "pcg64_bit_exact_vs_reference": exact, "batched_philox_ms": ms_batch,
            "batched_queries_per_s": len(qt) / (ms_batch / 1e3), "p50_us_per_step_query": us[len(us) // 2],
            "p99_us_per_step_query": us[int(0.99 * len(us))],
            "cpu_baseline": {"value": len(qt) / cpu_s, "unit": "queries/s", "cores": 1, "kind": "port",
                             "sample": "the same 10k trace, PCG64 stream, cold cache"}}


def c3(args):
    rec = records_sparse(1_000_000, 0)
    Q = args.queries
    qt, qc, qp = queries_sparse(Q, 1)
    dq = [torch.as_tensor(a, device="cuda") for a in (qt, qc, qp)]
    out = {"config": "c3", "workload": f"sparse long-context: 1M records (tt <= 131072), {Q} queries, cold sweep"}
    tables = DeviceTables.build(*rec, canonical=True)
    info = tables.info(1)
    out["mixed_buckets"] = info["n_buckets"]
    tabs = O.build(*rec, canonical=True)
    for floor in (32, 256):
        orc = LatencyOracle(pack_from_device(tables, 1000, keep_host=False), OracleConfig(reliability_floor=floor),
                            _validate=False)

        def sweep():
            orc.flush()
            orc.sample_batch(*dq, rng="philox", seed=1)

        ms = timed(sweep, max(1, args.steps // 2), warmup=1)
        _lib.profile_enable(True)
        sweep()
        kern = {k: round(_lib.profile_read(k)[0], 4) for k in ("mark", "pool_prep", "tile_bin", "scan", "tile_scatter",
                                                                "pool_tile", "pool_warp", "pool_grp", "pool_cta", "sample")}
        _lib.profile_enable(False)
        n = 2_000
        t0 = time.perf_counter()
        O.sample_batch(tabs, qt[:n], qc[:n], qp[:n], floor, mode="philox", seed=1, threads=CORES)
        cpu = n / (time.perf_counter() - t0)
        out[f"M{floor}"] = {"ms_per_sweep": ms, "queries_per_s": Q / (ms / 1e3), "kernels_ms": kern,
                            "cpu_baseline": {"value": cpu, "unit": "queries/s", "cores": CORES, "kind": "port",
                                             "sample": f"first {n} queries, cold cache per thread"}}
        del orc
    return out


def world():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def c4_dist(args):
    """Config 4 across ranks: each rank synthesises n/size records,
    tt-range partition (all-reduced histogram -> splitters), one all_to_all per
    column over NCCL, local canonical build of its tt slice, then the slices are
    re-replicated (one all_gather of the packed slice payloads) and every rank
    indexes the full tables.  Time = max over ranks, end to end."""
    import torch.distributed as dist

    from paper_2605_00616_b200.capture import records_device
    from paper_2605_00616_b200.dist import all_gather_tables, exchange_records, partition_by_tt, table_arrays

    rank, size = world()
    n = args.records_c4
    dev = list(records_device(n // size, seed=100 + rank))

    def step():
        spl = partition_by_tt(dev[0], size)
        cols = exchange_records(dev, dev[0], spl)
        t = DeviceTables.build(*cols, canonical=True)
        full = DeviceTables.from_device(all_gather_tables(table_arrays(t)))
        nb = sum(full.info(i)["n_buckets"] for i in range(3))
        del t, full
        return nb

    step()
    times = []
    for _ in range(max(1, args.steps // 3)):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        nb = step()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    tl = torch.tensor([statistics.mean(times), float(nb)], dtype=torch.float64, device="cuda")
    dist.all_reduce(tl[:1], op=dist.ReduceOp.MAX)
    dist.all_reduce(tl[1:], op=dist.ReduceOp.MAX)  # every rank holds the full tables
    ms = float(tl[0].item()) * 1e3
    return {"config": "c4", "workload": f"{n} synthetic records (generator G) over {size} ranks: tt-range partition, "
                                        "NCCL all_to_all exchange, per-rank canonical build, all_gather "
                                        "re-replication + full-table index on every rank",
            "n_gpus": size, "ms_per_build": ms, "records_per_s": n / (ms / 1e3), "buckets_total": int(tl[1].item()),
            "scaling": "strong"}


def c4(args):
    from paper_2605_00616_b200.capture import records_device

    if world()[1] > 1:
        return c4_dist(args)

    n = args.records_c4
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev = list(records_device(n, seed=100))  # generator G + ground-truth latencies on the device
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    m = 2_000_000
    cols = [d[:m].cpu().numpy() for d in dev]

    keep = []

    def build():  # the previous build's tables are freed outside the timed call (cudaFree syncs the device)
        keep.append(DeviceTables.build(*dev, canonical=True))

    build()  # warm-up (grows the stream-ordered scratch pool)
    times = []
    for _ in range(max(3, args.steps)):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        build()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        del keep[:-1]
    keep.clear()
    ms = statistics.median(times)
    _lib.profile_enable(True)
    t = DeviceTables.build(*dev, canonical=True)
    nb = sum(t.info(i)["n_buckets"] for i in range(3))
    kern = _lib.profile_all()
    _lib.profile_enable(False)
    sc_ms, passes = kern.get("onesweep", (0.0, 0))
    del t
    algo_bytes = 33 * n + 48 * nb / 3
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    t0 = time.perf_counter()
    O.build(cols[0], cols[1], cols[2], cols[3], canonical=True)
    cpu = m / (time.perf_counter() - t0)
    return {"config": "c4", "workload": f"{n} synthetic records (generator G), canonical 3-table build",
            "ms_per_build": ms, "ms_per_build_all": [round(x, 2) for x in times], "records_per_s": n / (ms / 1e3),
            "buckets_total": nb,
            "roofline": {"bound": "hbm", "achieved": algo_bytes / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": algo_bytes / (ms / 1e3) / 1e9 / peak,
                         "bytes": "33 B/record + 48 B/bucket (SURVEY 8d); multi-pass sort moves more"},
            "device_generation_s": gen_s,
            "radix_sort": {"passes": passes, "onesweep_ms": sc_ms,
                           "pass_GBps": 24 * n * passes / (sc_ms / 1e3) / 1e9 if sc_ms else None,
                           "note": "onesweep LSD: each pass reads (hi u32, lo u64) 12 B and writes 12 B per record"},
            "kernels_ms": {k: [round(v[0], 3), v[1]] for k, v in sorted(kern.items(), key=lambda kv: -kv[1][0])},
            "cpu_baseline": {"value": cpu, "unit": "records/s", "cores": 1, "kind": "port",
                             "sample": f"oracle qsort build of the first {m} records"}}


def scenario_keys(n, rate, gamma, gen):
    """Synthetic step keys of one scenario (GPU): concurrency grows with the
    request rate (Little's law with a ~3 s request lifetime) and its spread
    with burstiness 1/gamma; 70 % decode steps."""
    med = max(1.0, min(256.0, rate * 3.0))
    sigma = 0.4 + 0.4 / math.sqrt(gamma)
    conc = torch.clamp(torch.round(torch.exp(math.log(med) + sigma * torch.randn(n, device="cuda", generator=gen))),
                       1, 256).to(torch.int32)
    decode = torch.rand(n, device="cuda", generator=gen) < 0.7
    chunk = torch.clamp(torch.round(torch.exp(math.log(180.0) + torch.randn(n, device="cuda", generator=gen))), 1,
                        2048).to(torch.int32)
    tt = torch.where(decode, conc, torch.clamp(conc - 1 + chunk, max=2048))
    return tt, conc, (~decode).to(torch.uint8)


def c5(args):
    _, orc = oracle_for(records_llama(1_000_000, 0), 32)
    rates = np.geomspace(1, 64, 32)
    gammas = np.geomspace(0.125, 2, 16)
    steps_per = args.steps_c5
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    lat = torch.empty(steps_per, dtype=torch.float64, device="cuda")
    sidx = torch.empty(steps_per, dtype=torch.int32, device="cuda")
    scen = [(r, g) for r in rates for g in gammas][: args.scenarios]
    orc.flush()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = 0.0
    for k, (r, g) in enumerate(scen):  # scenario keys are synthesised on the GPU outside the timed calls
        tt, cc, ph = scenario_keys(steps_per, r, g, gen)
        a.record()
        orc.sample_batch(tt, cc, ph, rng="philox", seed=k, out_lat=lat, out_sidx=sidx)  # cache warm across scenarios
        b.record()
        b.synchronize()
        ms += a.elapsed_time(b)
    # token fill throughput (synthetic entries: 256M)
    n = 256 << 20
    g2 = torch.Generator(device="cuda")
    g2.manual_seed(3)
    pre = (torch.rand(n, device="cuda", generator=g2) < 0.1).to(torch.uint8)
    plen = torch.randint(1, 2048, (n,), device="cuda", dtype=torch.int32, generator=g2)
    prog = torch.remainder(torch.randint(0, 2048, (n,), device="cuda", dtype=torch.int32, generator=g2), plen)
    chunk = torch.clamp(plen - prog, max=512).to(torch.int32)
    gen_ = torch.randint(0, 512, (n,), device="cuda", dtype=torch.int32, generator=g2)
    tgt = torch.randint(1, 512, (n,), device="cuda", dtype=torch.int32, generator=g2)
    ids = torch.empty(n, dtype=torch.int32, device="cuda")
    fin = torch.empty(n, dtype=torch.uint8, device="cuda")
    ms_fill = timed(lambda: token_fill(pre, chunk, prog, plen, gen_, tgt, out_ids=ids, out_finished=fin), 5)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    fill_gbs = 26 * n / (ms_fill / 1e3) / 1e9
    total_q = len(scen) * steps_per
    return {"config": "c5", "workload": f"{len(scen)} scenarios x {steps_per} steps (rate x burstiness grid), "
                                        "Philox draws, pool cache warm across scenarios",
            "ms_total": ms, "queries_per_s": total_q / (ms / 1e3), "steps_total": total_q,
            "token_fill": {"entries": n, "ms": ms_fill, "entries_per_s": n / (ms_fill / 1e3),
                           "roofline": {"bound": "hbm", "achieved": fill_gbs, "peak": peak, "unit": "GB/s",
                                        "frac": fill_gbs / peak, "bytes_per_entry": 26}}}


def sweep(args):
    """What-if sweep with the reference scheduler on the GPU:
    512 scenarios (32 request rates x 16 burstiness values), each a virtual-time
    run of EmulatorEngine's scheduler with the oracle in the closed loop (per-
    scenario PCG64 stream, lazy pools).  Workloads: log-normal prompt/output
    lengths (medians 200/100, the reference's generate_workload shape) and
    Gamma(burstiness) inter-arrival gaps (generate_arrivals), numpy-generated."""
    from paper_2605_00616_b200.sched import EngineConfig, Scenario, emulate

    _, orc = oracle_for(records_llama(1_000_000, 0), 32)
    rates = np.geomspace(1, 64, 32)
    gammas = np.geomspace(0.125, 2, 16)
    steps = args.steps_sweep
    cfg = EngineConfig(num_gpu_blocks=8192, block_size=16, max_model_len=4096, max_num_batched_tokens=2048,
                       max_num_seqs=256)
    g = np.random.default_rng(17)
    scen = []
    horizon = steps * 0.05  # virtual seconds comfortably beyond `steps` steps
    for r in rates:
        for gm in gammas:
            n = int(r * horizon) + 16
            p = np.clip(np.rint(g.lognormal(np.log(200), 0.6, n)), 4, 2048).astype(np.int32)
            o = np.clip(np.rint(g.lognormal(np.log(100), 0.7, n)), 2, 512).astype(np.int32)
            gaps = g.gamma(gm, 1.0 / (r * gm), n - 1)
            scen.append(Scenario(p, o, np.concatenate([[0.0], np.cumsum(gaps)])))
    scen = scen[: args.scenarios]
    rank, size = world()
    mine = list(range(rank, len(scen), size))  # scenarios shard across ranks, no collective in the loop
    torch.cuda.synchronize()
    if size > 1:
        import torch.distributed as dist

        dist.barrier()
    t0 = time.perf_counter()
    out = emulate(cfg, [scen[k] for k in mine], steps, backend="oracle", oracle=orc, seeds=mine,
                  keep_steps=steps <= 50_000)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    total = int(out["n_steps"].sum())
    if size > 1:
        tl = torch.tensor([wall, float(total)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tl[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tl[1:], op=dist.ReduceOp.MAX)  # every rank holds the full tables
        wall, total = float(tl[0].item()), int(tl[1].item())
    return {"config": "sweep", "workload": f"{len(scen)} scenarios (rate x burstiness) x up to {steps} steps, "
                                            "reference scheduler + oracle closed loop on the GPU",
            "steps_total": total, "wall_s": wall, "steps_per_s": total / wall, "rounds": out["rounds"],
            "tokens_total": int(out["tokens"].sum()), "host_s": out["host_s"], "requests": int(sum(len(s.prompt_tokens) for s in scen)),
            "cpu_reference_note": "the reference engine + LatencyOracle runs ~4k steps/s per core in virtual time "
                                  "(tests/golden/make_sched_golden.py: 21k steps in ~5 s)"}


def codec(args):
    """pack JSON -> SoA and trace JSONL -> records -> GPU tables.
    Reference-algorithm times use this package's json path (the reference's
    json.loads + per-bucket / per-record objects, profile.py:299-404); the
    native path is csrc/codec.cpp (+ the GPU build for traces)."""
    from paper_2605_00616_b200.profile import (build_pack_arrays, load_pack, parse_trace_arrays,
                                               read_trace_file, save_pack, trace_record_to_line, StepTraceRecord,
                                               StepPhase)
    import tempfile

    n = args.records_codec
    rec = records_llama(n, 0)
    pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
    data = save_pack(pack)
    os.environ["EMU_PACK_CODEC"] = "json"
    t0 = time.perf_counter()
    ref_pack = load_pack(data)
    json_s = time.perf_counter() - t0
    del os.environ["EMU_PACK_CODEC"]
    native_s = []
    for _ in range(3):
        t0 = time.perf_counter()
        fast = load_pack(data)
        native_s.append(time.perf_counter() - t0)
    same = all(np.array_equal(a.samples.view(np.uint64), b.samples.view(np.uint64)) and np.array_equal(a.off, b.off)
               and np.array_equal(a.tt, b.tt) and np.array_equal(a.conc, b.conc)
               for a, b in zip(fast.soas(), ref_pack.soas()))
    # trace ingest: JSONL text of n records
    tt, cc, ph, lat = rec
    ph_names = (StepPhase.DECODE_ONLY, StepPhase.PREFILL_OR_MIXED)
    lines = [trace_record_to_line(StepTraceRecord(i, int(a), int(b), ph_names[int(c)], float(d)))
             for i, (a, b, c, d) in enumerate(zip(tt, cc, ph, lat))]
    text = ("\n".join(lines) + "\n").encode()
    with tempfile.NamedTemporaryFile("wb", suffix=".jsonl", delete=False) as f:
        f.write(text)
        path = f.name
    t0 = time.perf_counter()
    recs = read_trace_file(path)
    read_py_s = time.perf_counter() - t0
    parse_s = []
    for _ in range(3):
        t0 = time.perf_counter()
        cols = parse_trace_arrays(text)
        parse_s.append(time.perf_counter() - t0)
    exact = (np.array_equal(cols[4].view(np.uint64), np.array([r.latency_s for r in recs]).view(np.uint64))
             and np.array_equal(cols[1], tt) and np.array_equal(cols[2], cc))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p2 = build_pack_arrays(cols[1], cols[2], cols[3], cols[4], 1000, step=cols[0], canonical=True, keep_host=False)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    os.unlink(path)
    t0 = time.perf_counter()
    O.build(tt, cc, ph, lat, canonical=True)
    cpu_build_s = time.perf_counter() - t0
    return {"config": "codec", "workload": f"{n}-record Llama-shaped profile: pack JSON ({len(data) / 1e6:.1f} MB) "
                                           f"and trace JSONL ({len(text) / 1e6:.1f} MB)",
            "pack_load": {"json_path_s": json_s, "native_s": min(native_s), "speedup": json_s / min(native_s),
                          "bit_exact_vs_json_path": bool(same), "MB_per_s": len(data) / 1e6 / min(native_s)},
            "trace_ingest": {"read_trace_file_s": read_py_s, "native_parse_s": min(parse_s),
                             "records_per_s": n / min(parse_s), "speedup": read_py_s / min(parse_s),
                             "bit_exact_vs_parse_trace_line": bool(exact), "threads": min(32, CORES),
                             "gpu_build_s": build_s, "cpu_port_build_s": cpu_build_s,
                             "end_to_end_records_per_s": n / (min(parse_s) + build_s)}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c4", "c3", "c5", "codec", "sweep"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--queries", type=int, default=10_000_000)
    ap.add_argument("--records-c4", type=int, default=100_000_000)
    ap.add_argument("--scenarios", type=int, default=512)
    ap.add_argument("--steps-c5", type=int, default=1_000_000)
    ap.add_argument("--records-codec", type=int, default=1_000_000)
    ap.add_argument("--steps-sweep", type=int, default=20_000)
    args = ap.parse_args()
    size = int(os.environ.get("WORLD_SIZE", 1))
    if size > 1:  # torchrun: one process per GPU; configs c4 and sweep shard, the rest run on rank 0's GPU
        import torch.distributed as dist

        local = int(os.environ.get("LOCAL_RANK", 0))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = int(os.environ.get("RANK", 0))
    for c in args.configs:
        if size > 1 and c not in ("c4", "sweep"):
            continue
        res = {"c1": c1, "c3": c3, "c4": c4, "c5": c5, "codec": codec, "sweep": sweep}[c](args)
        if rank == 0:
            print(json.dumps(res), flush=True)
        import gc

        gc.collect()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
