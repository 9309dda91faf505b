"""Synthetic workloads for the benchmark configs.

There are no Llama-shaped profiles in the reference, so records are drawn
from generator G(seed): latencies follow the reference's ground-truth model
``m * (base + per_token*tt + per_seq*conc) * (1 + N(0, cv))`` with the noise
factor redrawn while nonpositive (engine.py:128-147), with Llama-8B-like
magnitudes base 6 ms, per_token 60 us, per_seq 150 us, prefill x1.25, cv 0.05.

    conc  = clip(round(LogNormal(ln 24, 0.8)), 1, 256)
    70 %  decode : tt = conc
    30 %  mixed  : tt = min(2048, conc - 1 + clip(round(LogNormal(ln 180, 1.0)), 1, 2048))

The sparse long-context generator (config 3) uses conc ~ LogNormal(ln 8, 1.0)
<= 256, 50 % decode, mixed chunk ~ LogNormal(ln 8000, 1.3) <= 131072.
Query keys for sweeps are drawn from the same key distribution with another
seed.  All host-side numpy (workload synthesis, not the measured path).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class GTParams:
    base_s: float = 0.006
    per_token_s: float = 60e-6
    per_seq_s: float = 150e-6
    prefill_multiplier: float = 1.25
    noise_cv: float = 0.05


def _latency(g: np.random.Generator, tt, conc, mixed, p: GTParams):
    base = p.base_s + p.per_token_s * tt + p.per_seq_s * conc
    base = np.where(mixed, base * p.prefill_multiplier, base)
    f = 1.0 + g.normal(0.0, p.noise_cv, len(tt))
    bad = f <= 0
    while bad.any():
        f[bad] = 1.0 + g.normal(0.0, p.noise_cv, int(bad.sum()))
        bad = f <= 0
    return base * f


def keys_llama(n: int, seed: int):
    """(tt int32, conc int32, phase uint8) keys of generator G."""
    g = np.random.default_rng(seed)
    conc = np.clip(np.rint(g.lognormal(np.log(24.0), 0.8, n)), 1, 256).astype(np.int64)
    decode = g.random(n) < 0.7
    chunk = np.clip(np.rint(g.lognormal(np.log(180.0), 1.0, n)), 1, 2048).astype(np.int64)
    tt = np.where(decode, conc, np.minimum(2048, conc - 1 + chunk))
    return tt.astype(np.int32), conc.astype(np.int32), (~decode).astype(np.uint8), g


def records_llama(n: int, seed: int = 0, params: GTParams | None = None):
    """Generator G(seed): (tt, conc, phase, latency_s) record columns."""
    tt, conc, ph, g = keys_llama(n, seed)
    lat = _latency(g, tt.astype(np.float64), conc.astype(np.float64), ph.astype(bool), params or GTParams())
    return tt, conc, ph, lat


def queries_llama(n: int, seed: int = 1):
    tt, conc, ph, _ = keys_llama(n, seed)
    return tt, conc, ph


def keys_sparse(n: int, seed: int):
    """Sparse long-context key distribution (config 3)."""
    g = np.random.default_rng(seed)
    conc = np.clip(np.rint(g.lognormal(np.log(8.0), 1.0, n)), 1, 256).astype(np.int64)
    decode = g.random(n) < 0.5
    chunk = np.clip(np.rint(g.lognormal(np.log(8000.0), 1.3, n)), 1, 131072).astype(np.int64)
    tt = np.where(decode, conc, np.minimum(131072, conc - 1 + chunk))
    return tt.astype(np.int32), conc.astype(np.int32), (~decode).astype(np.uint8), g


def records_sparse(n: int, seed: int = 0, params: GTParams | None = None):
    tt, conc, ph, g = keys_sparse(n, seed)
    lat = _latency(g, tt.astype(np.float64), conc.astype(np.float64), ph.astype(bool), params or GTParams())
    return tt, conc, ph, lat


def queries_sparse(n: int, seed: int = 1):
    tt, conc, ph, _ = keys_sparse(n, seed)
    return tt, conc, ph


def explicit_uniforms(n: int, seed: int):
    """Caller-supplied words for rng='explicit' (u_sel u64, u_idx u32)."""
    g = np.random.default_rng(seed)
    return (g.integers(0, 2**64, n, dtype=np.uint64, endpoint=False),
            g.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32))
