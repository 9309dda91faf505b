"""Device scheduler vs the unmodified reference scheduler (tests/golden/sched_golden.npz,
written by make_sched_golden.py from EmulatorEngine in virtual time)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import ROOT
from paper_2605_00616_b200 import LatencyOracle, OracleConfig
from paper_2605_00616_b200.capture import GroundTruthParams
from paper_2605_00616_b200.sched import EngineConfig, Scenario, emulate

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(ROOT, "tests", "golden", "sched_golden.npz"))


def scenario(name):
    c = G[f"{name}_cfg"]
    cfg = EngineConfig(int(c[0]), int(c[1]), int(c[2]), int(c[3]), int(c[4]))
    return cfg, Scenario(G[f"{name}_prompt"], G[f"{name}_output"], G[f"{name}_arrivals"])


@pytest.mark.parametrize("name,lists", [("gt_c1", "smem"), ("gt_tight", "smem"), ("gt_bursty", "smem"),
                                        ("gt_wide", "smem"), ("gt_wide300", "smem"), ("gt_tight", "global"),
                                        ("gt_wide", "global")])
def test_replay_matches_reference_scheduler(name, lists, monkeypatch):
    """Same latencies in -> the same step keys, emissions, finishes and preemptions.
    gt_wide / gt_wide300 run 256 / 300 requests at once (several lane groups in
    the decode pass, preemptions across group boundaries); `global` forces the
    running lists out of shared memory (the path for very large max_num_seqs)."""
    if lists == "global":
        monkeypatch.setenv("EMU_SCHED_SMEM", "0")
    cfg, sc = scenario(name)
    lat = G[f"{name}_lat"]
    n = len(lat)
    out = emulate(cfg, [sc, sc], n, backend="replay", latencies=[lat, lat])
    for s in range(2):
        assert out["n_steps"][s] == n
        keys = np.stack([out["tt"][s], out["conc"][s], out["phase"][s].astype(np.int32)], 1)
        assert np.array_equal(keys, G[f"{name}_keys"])
        st = np.stack([out["tokens"][s], out["finished"][s], out["preemptions"][s]], 1)
        assert np.array_equal(st, G[f"{name}_stats"])
        assert np.array_equal(out["latency_s"][s], lat)


def test_closed_loop_oracle_matches_reference(c1_records):
    """The closed loop with the oracle: keys AND latencies equal a reference engine
    whose backend is LatencyOracle(C1 pack, OracleConfig(32, rng_seed=11))."""
    from paper_2605_00616_b200 import build_pack_arrays

    pack = build_pack_arrays(*c1_records, num_gpu_blocks=1000, canonical=True)
    cfg, sc = scenario("oracle")
    n = len(G["oracle_lat"])
    for prefetch in (False, True):  # lazy pools (pause + build rounds) / every reachable pool first
        orc = LatencyOracle(pack, OracleConfig(reliability_floor=32, rng_seed=11))
        out = emulate(cfg, [sc, sc, sc], n, backend="oracle", oracle=orc, seeds=[11, 11, 11], prefetch=prefetch)
        for s in range(3):
            assert out["n_steps"][s] == n
            keys = np.stack([out["tt"][s], out["conc"][s], out["phase"][s].astype(np.int32)], 1)
            assert np.array_equal(keys, G["oracle_keys"])
            assert np.array_equal(out["latency_s"][s].view(np.uint64), G["oracle_lat"].view(np.uint64))
        assert (out["rounds"] == 1) if prefetch else (out["rounds"] > 1)


def test_ground_truth_backend_runs_and_is_deterministic():
    cfg, sc = scenario("gt_tight")
    p = GroundTruthParams(noise_cv=0.05)
    a = emulate(cfg, [sc] * 4, 3000, backend="ground_truth", gt_params=p, gt_seed=5)
    b = emulate(cfg, [sc] * 4, 3000, backend="ground_truth", gt_params=p, gt_seed=5)
    assert np.array_equal(a["tt"], b["tt"]) and np.array_equal(a["latency_s"], b["latency_s"])
    assert (a["latency_s"][:, :a["n_steps"].min()] > 0).all()
    assert a["preemptions"][:, -1].max() > 0  # the tight config preempts


def test_config_validation_messages():
    sc = Scenario(np.array([10], np.int32), np.array([5], np.int32), np.array([0.0]))
    with pytest.raises(ValueError, match="max_num_batched_tokens 8 must be >= block_size 16"):
        emulate(EngineConfig(100, 16, 4096, 8, 4), [sc], 10, backend="ground_truth")
    big = Scenario(np.array([4000], np.int32), np.array([200], np.int32), np.array([0.0]))
    with pytest.raises(ValueError, match="prompt_tokens \\+ max_tokens = 4200 exceeds max_model_len 4096"):
        emulate(EngineConfig(1000), [big], 10, backend="ground_truth")


def test_totals_only_run_matches_per_step_outputs():
    """keep_steps=False allocates no per-step arrays; the kernel's running totals
    equal the sums of a per-step run (replay of gt_wide: preemptions included)."""
    cfg, sc = scenario("gt_wide")
    lat = G["gt_wide_lat"]
    n = len(lat)
    full = emulate(cfg, [sc, sc], n, backend="replay", latencies=[lat, lat])
    tot = emulate(cfg, [sc, sc], n, backend="replay", latencies=[lat, lat], keep_steps=False)
    for s in range(2):
        assert tot["n_steps"][s] == full["n_steps"][s] == n
        assert tot["tokens"][s] == full["tokens"][s].sum() == G["gt_wide_stats"][:, 0].sum()
        assert tot["finished"][s] == full["finished"][s].sum()
        assert tot["preemptions"][s] == full["preemptions"][s][n - 1] == G["gt_wide_stats"][-1, 2]
    assert "tt" not in tot
