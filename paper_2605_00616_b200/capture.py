"""Batched capture stand-ins on the GPU.

``GroundTruthParams`` / ``ground_truth_latency`` mirror the reference's
synthetic step-latency model (/root/reference/pkg/src/serve_emu/engine.py:
107-147); ``ground_truth_latencies`` evaluates it for a whole batch of step
keys in one kernel (``emu_ground_truth``): the deterministic part is
bit-identical to the reference's expression, the N(0, cv) deviates come from
Philox4x32-10 keyed by (seed, record index) instead of CPython's
``random.gauss`` (the reference's stream is not reproduced).
``gen_step_keys`` / ``records_device`` synthesise the step keys of generator G
 on the device, so multi-100M-record table builds start from
device-resident records.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

from . import _lib
from .profile import StepPhase, phase_code


@dataclass
class GroundTruthParams:
    """Synthetic per-step latency model standing in for GPU execution (engine.py:107-125)."""

    base_s: float = 0.003
    per_token_s: float = 4e-5
    per_seq_s: float = 1.2e-4
    prefill_multiplier: float = 1.25
    noise_cv: float = 0.0

    def validate(self) -> None:
        if not self.base_s > 0:
            raise ValueError(f"base_s must be > 0, got {self.base_s}")
        if self.per_token_s < 0 or self.per_seq_s < 0:
            raise ValueError("per_token_s and per_seq_s must be >= 0")
        if self.prefill_multiplier < 1.0:
            raise ValueError(f"prefill_multiplier must be >= 1, got {self.prefill_multiplier}")
        if self.noise_cv < 0:
            raise ValueError(f"noise_cv must be >= 0, got {self.noise_cv}")


def ground_truth_latency(tt: int, conc: int, phase, params: GroundTruthParams, rng) -> float:
    """The reference's scalar model (engine.py:128-147), for host-side use."""
    mult = params.prefill_multiplier if phase_code(phase) == 1 else 1.0
    latency = mult * (params.base_s + params.per_token_s * tt + params.per_seq_s * conc)
    if params.noise_cv == 0:
        return latency
    while True:
        factor = 1.0 + rng.gauss(0.0, params.noise_cv)
        if factor > 0:
            return latency * factor


def ground_truth_latencies(tt, conc, phase, params: GroundTruthParams | None = None, seed: int = 0, *, out=None):
    """ground_truth_latency for every step key (CUDA tensors in, f64 CUDA tensor out)."""
    torch = _lib.require_cuda()
    params = params or GroundTruthParams()
    params.validate()
    cols = [tt.to(torch.int32).contiguous(), conc.to(torch.int32).contiguous(), phase.to(torch.uint8).contiguous()]
    n = cols[0].numel()
    if any(c.numel() != n or not c.is_cuda for c in cols):
        raise ValueError("ground_truth_latencies needs equal-length CUDA tensors")
    lat = out if out is not None else torch.empty(n, dtype=torch.float64, device=cols[0].device)
    _lib.check(_lib.lib().emu_ground_truth(*[_lib.ptr(c) for c in cols], n, float(params.base_s),
                                           float(params.per_token_s), float(params.per_seq_s),
                                           float(params.prefill_multiplier), float(params.noise_cv),
                                           seed & (2**64 - 1), _lib.ptr(lat), _lib.stream_ptr()))
    return lat


def gen_step_keys(n: int, seed: int = 0, *, conc_median: float = 24.0, conc_sigma: float = 0.8, conc_max: int = 256,
                  p_decode: float = 0.7, chunk_median: float = 180.0, chunk_sigma: float = 1.0, tt_max: int = 2048):
    """n step keys of generator G on the device: (tt int32, conc int32, phase uint8) CUDA tensors."""
    torch = _lib.require_cuda()
    tt = torch.empty(n, dtype=torch.int32, device="cuda")
    conc = torch.empty(n, dtype=torch.int32, device="cuda")
    ph = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().emu_gen_step_keys(int(n), seed & (2**64 - 1), math.log(conc_median), float(conc_sigma),
                                            int(conc_max), float(p_decode), math.log(chunk_median),
                                            float(chunk_sigma), int(tt_max), _lib.ptr(tt), _lib.ptr(conc),
                                            _lib.ptr(ph), _lib.stream_ptr()))
    return tt, conc, ph


# Llama-3-8B-like magnitudes used by the benchmark profiles (workloads.GTParams)
LLAMA_GT = GroundTruthParams(base_s=0.006, per_token_s=60e-6, per_seq_s=150e-6, prefill_multiplier=1.25,
                             noise_cv=0.05)


def records_device(n: int, seed: int = 0, params: GroundTruthParams = LLAMA_GT, **key_kw):
    """Generator G's records on the device: (tt, conc, phase, latency_s) CUDA tensors."""
    tt, conc, ph = gen_step_keys(n, seed, **key_kw)
    return tt, conc, ph, ground_truth_latencies(tt, conc, ph, params, seed)


__all__ = ["GroundTruthParams", "LLAMA_GT", "StepPhase", "gen_step_keys", "ground_truth_latencies",
           "ground_truth_latency", "records_device"]
