"""Golden virtual-time runs of the UNMODIFIED reference scheduler (dev container).

    python tests/golden/make_sched_golden.py

The reference EmulatorEngine (engine.py:360-483) is driven in virtual time the
way tests/golden/make_golden.py drives it: admit every request whose arrival
offset is <= t, schedule a step, ask the backend for its latency, apply the
outcome, t += latency (an empty schedule jumps t to the next arrival).
Workloads and arrivals come from the reference's generate_workload /
generate_arrivals (bench.py:77-116).  Writes sched_golden.npz with, per
scenario: the engine config, request lengths and arrival offsets, and per
step (tt, conc, phase, latency, tokens emitted, requests finished, cumulative
preemptions).

Scenarios
  gt_*      backend = GroundTruthBackend(noise_cv=0.05): the device scheduler
            replays the recorded latencies (keys must match exactly);
  oracle    backend = LatencyOracle(C1 pack, OracleConfig(32, rng_seed=11)):
            the device scheduler draws from its own PCG64 stream in the closed
            loop (keys AND latencies must match exactly).
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from serve_emu.bench import WorkloadSpec, generate_arrivals, generate_workload  # noqa: E402
from serve_emu.engine import EmulatorEngine, EngineConfig, GroundTruthBackend, GroundTruthParams  # noqa: E402
from serve_emu.oracle import LatencyOracle, OracleConfig  # noqa: E402
from serve_emu.profile import StepPhase, StepTraceRecord, build_pack, load_pack, save_pack  # noqa: E402

from paper_2605_00616_b200.workloads import records_llama  # noqa: E402


def run(cfg, entries, arrivals, backend, n_steps):
    eng = EmulatorEngine(cfg, backend=lambda t, c, p: 0.01)
    t, i, rows = 0.0, 0, []
    while len(rows) < n_steps:
        while i < len(entries) and arrivals[i] <= t:
            eng.admit(*entries[i])
            i += 1
        prep = eng._schedule_step()
        if prep is None:
            if i >= len(entries):
                break
            t = arrivals[i]
            continue
        lat = backend(prep.total_tokens, prep.concurrency, prep.phase)
        out = eng._apply_outcome(prep)
        rows.append((prep.total_tokens, prep.concurrency, 0 if prep.phase is StepPhase.DECODE_ONLY else 1, lat,
                     len(out.emissions), len(out.finished), eng._preemptions))
        t += lat
    return rows


def main():
    scen = {
        "gt_c1": (EngineConfig(num_gpu_blocks=4096, block_size=16, max_model_len=4096, max_num_batched_tokens=512,
                               max_num_seqs=64), (4000, 200, 100, 7), (8.0, 1.0, 42)),
        "gt_tight": (EngineConfig(num_gpu_blocks=260, block_size=16, max_model_len=4096, max_num_batched_tokens=256,
                                  max_num_seqs=32), (3000, 300, 150, 8), (20.0, 1.0, 43)),
        "gt_bursty": (EngineConfig(num_gpu_blocks=1024, block_size=16, max_model_len=4096, max_num_batched_tokens=384,
                                   max_num_seqs=48), (3000, 150, 80, 9), (16.0, 0.25, 44)),
        # max_num_seqs > 128: the device decode pass spans several lane groups
        "gt_wide": (EngineConfig(num_gpu_blocks=4096, block_size=16, max_model_len=4096, max_num_batched_tokens=2048,
                                 max_num_seqs=256), (6000, 120, 160, 11), (400.0, 1.0, 46)),
        "gt_wide300": (EngineConfig(num_gpu_blocks=6000, block_size=16, max_model_len=4096, max_num_batched_tokens=4096,
                                    max_num_seqs=300), (6000, 120, 160, 12), (500.0, 0.5, 47)),
        "oracle": (EngineConfig(num_gpu_blocks=1500, block_size=16, max_model_len=4096, max_num_batched_tokens=512,
                                max_num_seqs=64), (3000, 200, 100, 10), (12.0, 1.0, 45)),
    }
    tt, conc, ph, lat = records_llama(50_000, 0)
    recs = [StepTraceRecord(k, int(a), int(b), StepPhase.DECODE_ONLY if p == 0 else StepPhase.PREFILL_OR_MIXED,
                            float(l)) for k, (a, b, p, l) in enumerate(zip(tt, conc, ph, lat))]
    c1pack = load_pack(save_pack(build_pack(recs, 1000)))
    out = {}
    for name, (cfg, (nreq, pmed, omed, wseed), (rate, burst, aseed)) in scen.items():
        entries = generate_workload(nreq, pmed, omed, seed=wseed)
        arrivals = generate_arrivals(WorkloadSpec(entries=entries, request_rate=rate, burstiness=burst, seed=aseed))
        if name == "oracle":
            backend = LatencyOracle(c1pack, OracleConfig(reliability_floor=32, rng_seed=11))
            n_steps = 3000
        else:
            backend = GroundTruthBackend(GroundTruthParams(noise_cv=0.05), seed=3)
            n_steps = 6000 if not name.startswith("gt_wide") else 2500
        rows = run(cfg, entries, arrivals, backend, n_steps)
        a = np.array(rows, dtype=np.float64)
        out[f"{name}_cfg"] = np.array([cfg.num_gpu_blocks, cfg.block_size, cfg.max_model_len,
                                       cfg.max_num_batched_tokens, cfg.max_num_seqs], dtype=np.int64)
        out[f"{name}_prompt"] = np.array([e[0] for e in entries], dtype=np.int32)
        out[f"{name}_output"] = np.array([e[1] for e in entries], dtype=np.int32)
        out[f"{name}_arrivals"] = np.array(arrivals, dtype=np.float64)
        out[f"{name}_keys"] = a[:, :3].astype(np.int32)
        out[f"{name}_lat"] = a[:, 3]
        out[f"{name}_stats"] = a[:, 4:].astype(np.int64)
        print(name, len(rows), "steps, preemptions", int(a[-1, 6]), "finished", int(a[:, 5].sum()))
    np.savez_compressed(os.path.join(HERE, "sched_golden.npz"), **out)


if __name__ == "__main__":
    main()
