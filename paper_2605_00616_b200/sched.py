"""The reference scheduler in virtual time on the GPU.

``emulate`` runs S independent what-if scenarios of the reference engine
(``EmulatorEngine.admit`` / ``_schedule_step`` / ``_apply_outcome``,
/root/reference/pkg/src/serve_emu/engine.py:323-483) in virtual time, one GPU
warp per scenario (``emu_sched_*`` in csrc/sched.cu): arrivals <= t are
admitted, a step is scheduled, its latency is taken from the backend, the
outcome applied and t advanced by the latency.  Backends:

* ``"oracle"``: a :class:`LatencyOracle` in the closed loop -- scenario s draws
  from its own numpy PCG64 stream seeded ``seeds[s]``, exactly what a reference
  engine with ``LatencyOracle(pack, OracleConfig(..., rng_seed=seeds[s]))``
  would draw; pools are built lazily (paused scenarios, batched build);
* ``"ground_truth"``: ``ground_truth_latency`` with Philox noise (capture stand-in);
* ``"replay"``: recorded per-step latencies (parity with a recorded run).

Workloads (request lengths, arrival offsets) come from the caller, e.g. the
reference's ``generate_workload`` / ``generate_arrivals`` (bench.py:77-116).
"""
from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .capture import GroundTruthParams
from .oracle import LatencyOracle, pcg64_state6


@dataclass
class EngineConfig:
    """Scheduler knobs (engine.py:77-104)."""

    num_gpu_blocks: int
    block_size: int = 16
    max_model_len: int = 4096
    max_num_batched_tokens: int = 512
    max_num_seqs: int = 64


@dataclass
class Scenario:
    prompt_tokens: np.ndarray  # int32 [n]
    output_tokens: np.ndarray  # int32 [n]
    arrival_s: np.ndarray      # f64 [n], ascending offsets


def step_key_domain(config: EngineConfig):
    """Every step key the scheduler can produce: decode steps (c, c) and mixed
    steps (t, c) with c <= t <= max_num_batched_tokens, c <= max_num_seqs."""
    c = np.arange(1, config.max_num_seqs + 1, dtype=np.int64)
    dec = (c, c, np.zeros(len(c), np.uint8))
    reps = np.maximum(0, config.max_num_batched_tokens - c + 1)
    mc = np.repeat(c, reps)
    start = np.repeat(c - np.concatenate([[0], np.cumsum(reps)[:-1]]), reps)
    mt = np.arange(len(mc), dtype=np.int64) + start
    mix = (mt, mc, np.ones(len(mc), np.uint8))
    return tuple(np.concatenate([d, m]) for d, m in zip(dec, mix))


def prefetch_domain(oracle: LatencyOracle, config: EngineConfig) -> int:
    """Build the pools of every step key of `config` up front (emu_oracle_prefetch):
    pools are pure functions of the key, so this changes no draw -- it only
    removes the closed loop's pause-and-build rounds."""
    torch = _lib.require_cuda()
    tt, cc, ph = step_key_domain(config)
    cols = [torch.as_tensor(tt.astype(np.int32), device="cuda"), torch.as_tensor(cc.astype(np.int32), device="cuda"),
            torch.as_tensor(ph, device="cuda")]
    _lib.check(_lib.lib().emu_oracle_prefetch(oracle._h, *[_lib.ptr(c) for c in cols], len(tt), _lib.stream_ptr()))
    return len(tt)


def _concat(parts, off: np.ndarray, dtype) -> np.ndarray:
    """np.concatenate into one request table, scenario slices copied by a thread
    pool (numpy copies release the GIL; large sweeps are first-touch bound)."""
    out = np.empty(int(off[-1]), dtype)
    if off[-1] < (1 << 22) or len(parts) == 1:
        for k, p in enumerate(parts):
            out[off[k]:off[k + 1]] = np.asarray(p)
        return out
    from concurrent.futures import ThreadPoolExecutor

    def put(k):
        out[off[k]:off[k + 1]] = np.asarray(parts[k])

    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(put, range(len(parts))))
    return out


def _phases(tm: dict) -> dict:
    """Seconds per phase of emulate() (wall clock, host side; `run` includes the kernel)."""
    ks = list(tm)
    return {b: round(tm[b] - tm[a], 4) for a, b in zip(ks, ks[1:])}


def emulate(config: EngineConfig, scenarios: Sequence[Scenario], max_steps: int, *, backend: str = "oracle",
            oracle: LatencyOracle | None = None, seeds: Sequence[int] | None = None,
            gt_params: GroundTruthParams | None = None, gt_seed: int = 0, latencies=None,
            prefetch: bool | None = None, keep_steps: bool = True) -> dict:
    """Per-step arrays [S, max_steps] (tt, conc, phase, latency, tokens, finished,
    preemptions) and n_steps [S]; steps past n_steps[s] are unused.  With the
    oracle backend, `prefetch` (default: when the key domain has <= 2M keys)
    builds every reachable pool first, so the closed loop runs in one launch."""
    _lib.require_cuda()
    tm = {"start": time.perf_counter()}
    S = len(scenarios)
    off = np.zeros(S + 1, np.int64)
    off[1:] = np.cumsum([len(sc.prompt_tokens) for sc in scenarios])
    prompt = _concat([sc.prompt_tokens for sc in scenarios], off, np.int32)
    target = _concat([sc.output_tokens for sc in scenarios], off, np.int32)
    arrival = _concat([sc.arrival_s for sc in scenarios], off, np.float64)
    L = _lib.lib()
    h = ctypes.c_void_p()
    tm["concat"] = time.perf_counter()
    _lib.check(L.emu_sched_create(S, _lib.ptr(off), _lib.ptr(prompt), _lib.ptr(target), _lib.ptr(arrival),
                                  int(config.num_gpu_blocks), int(config.block_size), int(config.max_model_len),
                                  int(config.max_num_batched_tokens), int(config.max_num_seqs), int(max_steps),
                                  ctypes.byref(h)))
    tm["create"] = time.perf_counter()
    try:
        _lib.check(L.emu_sched_keep_steps(h, 1 if keep_steps else 0))
        rounds = ctypes.c_int64(0)
        if backend == "oracle":
            if oracle is None:
                raise ValueError("backend='oracle' needs an oracle")
            seeds = list(seeds) if seeds is not None else [oracle.cfg.rng_seed] * S
            st = np.stack([pcg64_state6(np.random.default_rng(int(sd)).bit_generator.state) for sd in seeds])
            st = np.ascontiguousarray(st, dtype=np.uint64)
            domain = config.max_num_seqs * config.max_num_batched_tokens
            if prefetch or (prefetch is None and domain <= 2_000_000):
                prefetch_domain(oracle, config)
            tm["prefetch"] = time.perf_counter()
            _lib.check(L.emu_sched_run_oracle(h, oracle._h, _lib.ptr(st), ctypes.byref(rounds), _lib.stream_ptr()))
        elif backend == "ground_truth":
            p = gt_params or GroundTruthParams()
            p.validate()
            _lib.check(L.emu_sched_run_ground_truth(h, float(p.base_s), float(p.per_token_s), float(p.per_seq_s),
                                                    float(p.prefill_multiplier), float(p.noise_cv),
                                                    gt_seed & (2**64 - 1), _lib.stream_ptr()))
        elif backend == "replay":
            lat = np.zeros((S, max_steps), np.float64)
            for s, row in enumerate(latencies):
                row = np.asarray(row, np.float64)[:max_steps]
                lat[s, :len(row)] = row
            _lib.check(L.emu_sched_run_replay(h, _lib.ptr(lat), _lib.stream_ptr()))
        else:
            raise ValueError(f"unknown backend {backend!r}")
        tm["run"] = time.perf_counter()
        status = np.zeros(S, np.int32)
        if not keep_steps:  # totals only (long sweeps): no per-step arrays cross PCIe
            summ = np.zeros((S, 4), np.int64)
            _lib.check(L.emu_sched_summary(h, _lib.ptr(summ)))
            _lib.check(L.emu_sched_results(h, None, _lib.ptr(status), None, None, None, None, None, None, None))
            res = {"n_steps": summ[:, 0], "tokens": summ[:, 1], "finished": summ[:, 2], "preemptions": summ[:, 3]}
        else:
            res = {k: np.zeros((S, max_steps), dt) for k, dt in (("tt", np.int32), ("conc", np.int32),
                                                                ("phase", np.uint8), ("latency_s", np.float64),
                                                                ("tokens", np.int32), ("finished", np.int32),
                                                                ("preemptions", np.int64))}
            res["n_steps"] = np.zeros(S, np.int64)
            _lib.check(L.emu_sched_results(h, _lib.ptr(res["n_steps"]), _lib.ptr(status), _lib.ptr(res["tt"]),
                                           _lib.ptr(res["conc"]), _lib.ptr(res["phase"]), _lib.ptr(res["latency_s"]),
                                           _lib.ptr(res["tokens"]), _lib.ptr(res["finished"]),
                                           _lib.ptr(res["preemptions"])))
        if (status == 3).any():
            raise RuntimeError(f"scheduler invariant violated in scenarios {np.flatnonzero(status == 3).tolist()}")
        res["rounds"] = int(rounds.value)
        tm["results"] = time.perf_counter()
    finally:
        L.emu_sched_destroy(h)
    tm["destroy"] = time.perf_counter()
    res["host_s"] = _phases(tm)
    return res


__all__ = ["EngineConfig", "Scenario", "emulate", "prefetch_domain", "step_key_domain"]
