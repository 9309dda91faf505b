"""Capture stand-ins on the GPU vs the reference's model.

Bit-exact bar for the deterministic part of ground_truth_latency
(engine.py:128-147, restated in capture.ground_truth_latency); the Philox
deviates are checked statistically (they are not CPython's random.gauss
stream, by design)."""
from __future__ import annotations

import random

import numpy as np
import pytest
import torch

from paper_2605_00616_b200.capture import (
    GroundTruthParams,
    gen_step_keys,
    ground_truth_latencies,
    ground_truth_latency,
    records_device,
)
from paper_2605_00616_b200.device import DeviceTables

pytestmark = pytest.mark.gpu


def test_noise_free_model_bit_exact():
    rng = np.random.default_rng(1)
    n = 200_000
    tt = rng.integers(1, 200_000, n)
    cc = rng.integers(1, 1024, n)
    ph = rng.integers(0, 2, n)
    for p in (GroundTruthParams(), GroundTruthParams(0.006, 6e-5, 1.5e-4, 1.7, 0.0)):
        got = ground_truth_latencies(torch.as_tensor(tt, device="cuda"), torch.as_tensor(cc, device="cuda"),
                                     torch.as_tensor(ph, device="cuda"), p).cpu().numpy()
        want = np.array([ground_truth_latency(int(a), int(b), int(c), p, None) for a, b, c in
                         zip(tt[:20_000], cc[:20_000], ph[:20_000])])
        assert np.array_equal(got[:20_000].view(np.uint64), want.view(np.uint64))


def test_noise_statistics_and_redraw():
    n = 4_000_000
    tt = torch.full((n,), 100, dtype=torch.int32, device="cuda")
    cc = torch.full((n,), 8, dtype=torch.int32, device="cuda")
    ph = torch.zeros(n, dtype=torch.uint8, device="cuda")
    base = ground_truth_latency(100, 8, 0, GroundTruthParams(), None)
    lat = ground_truth_latencies(tt, cc, ph, GroundTruthParams(noise_cv=0.05), seed=3)
    f = (lat / base).cpu().numpy()
    assert abs(f.mean() - 1.0) < 2e-4 and abs(f.std() - 0.05) / 0.05 < 5e-3
    again = ground_truth_latencies(tt, cc, ph, GroundTruthParams(noise_cv=0.05), seed=3)
    assert torch.equal(lat, again)
    # cv = 2: ~31 % of first draws are nonpositive and redrawn; every latency stays > 0
    wide = (ground_truth_latencies(tt, cc, ph, GroundTruthParams(noise_cv=2.0), seed=4) / base).cpu().numpy()
    assert (wide > 0).all()
    # the redraw gives the normal truncated at factor > 0: its mean is 1 + cv * pdf(a) / (1 - cdf(a)), a = -1/cv
    from math import erf, exp, pi, sqrt
    a = -0.5
    pdf, cdf = exp(-a * a / 2) / sqrt(2 * pi), 0.5 * (1 + erf(a / sqrt(2)))
    assert abs(wide.mean() - (1 + 2.0 * pdf / (1 - cdf))) < 5e-3


@pytest.mark.parametrize("bad,msg", [
    (dict(base_s=0.0), "base_s must be > 0, got 0.0"),
    (dict(per_token_s=-1.0), "per_token_s and per_seq_s must be >= 0"),
    (dict(prefill_multiplier=0.5), "prefill_multiplier must be >= 1, got 0.5"),
    (dict(noise_cv=-0.1), "noise_cv must be >= 0, got -0.1"),
])
def test_params_validation_messages(bad, msg):
    t = torch.ones(4, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError, match=msg.replace("(", r"\(")):
        ground_truth_latencies(t, t, t.to(torch.uint8), GroundTruthParams(**bad))


def test_generator_keys_and_build():
    tt, cc, ph, lat = records_device(2_000_000, seed=9)
    t, c, p = tt.cpu().numpy(), cc.cpu().numpy(), ph.cpu().numpy()
    assert abs((p == 0).mean() - 0.7) < 2e-3
    assert c.min() >= 1 and c.max() <= 256 and t.max() <= 2048
    assert (t[p == 0] == c[p == 0]).all() and (t[p == 1] >= c[p == 1] - 1).all()
    assert abs(np.median(c) - 24) <= 1
    assert (lat > 0).all().item()
    tables = DeviceTables.build(tt, cc, ph, lat, canonical=True)  # device-resident records straight into the build
    assert sum(tables.info(i)["n_samples"] for i in (0, 1)) == 2_000_000
