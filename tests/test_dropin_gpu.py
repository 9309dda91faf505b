"""The drop-in, inside the UNMODIFIED reference engine (B200 only).

serve_emu is imported from baseline/_ref (installed by baseline/install_ref.sh
from /root/reference/pkg; it travels to the GPU box, /root/reference does not).
The reference's EmulatorEngine is driven exactly like its own tests do
(pkg/tests/test_engine.py:400-459): requests admitted up front, the step loop
run in real time, every step recorded through on_step.  Its backend is either
the reference LatencyOracle or this package's LatencyOracle over the same pack
and seed; the step keys and sampled latencies must be identical
(engine.py:555-566 consumes one backend call per step).  An empty pack must
abort the run with the reference's message naming tt=, conc= and phase=
(engine.py:569-578, test_engine.py:439-459, test_server.py:223-247).
"""
from __future__ import annotations

import asyncio
import os
import random
import sys

import numpy as np
import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "serve_emu")),
                                 reason="reference not installed (baseline/install_ref.sh)")]


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    import serve_emu.engine as E
    import serve_emu.oracle as RO
    import serve_emu.profile as RP
    import serve_emu.server as RS

    return E, RO, RP, RS


def _ref_pack(RP, n=6000, seed=0):
    from paper_2605_00616_b200.workloads import records_llama

    tt, conc, ph, lat = records_llama(n, seed)
    recs = [RP.StepTraceRecord(i, int(a), int(b), RP.StepPhase.PREFILL_OR_MIXED if c else RP.StepPhase.DECODE_ONLY,
                               float(d) * 0.05)  # ~0.3-6 ms steps keep the real-time run short
            for i, (a, b, c, d) in enumerate(zip(tt, conc, ph, lat))]
    return RP.load_pack(RP.save_pack(RP.build_pack(recs, 4096)))  # server.py:60 loads from file


def _run_engine(E, backend, n_req=40, seed=17):
    async def scenario():
        records = []
        cfg = E.EngineConfig(num_gpu_blocks=256, block_size=16, max_model_len=2048, max_num_batched_tokens=256,
                             max_num_seqs=8)
        eng = E.EmulatorEngine(cfg, backend, on_step=lambda r: records.append(r))
        rng = random.Random(seed)
        handles = [eng.admit(rng.randint(4, 120), rng.randint(2, 40)) for _ in range(n_req)]
        await eng.start()
        for h in handles:
            await asyncio.wait_for(h.done.wait(), 60)
        stats = eng.stats()
        await eng.stop()
        return [(r.step_index, r.total_tokens, r.concurrency, r.phase, r.sampled_s) for r in records], stats

    return asyncio.run(scenario())


def test_engine_with_b200_backend_matches_reference_backend(ref):
    E, RO, RP, RS = ref
    from paper_2605_00616_b200 import LatencyOracle, OracleConfig

    pack = _ref_pack(RP)
    want, st_ref = _run_engine(E, RO.LatencyOracle(pack, RO.OracleConfig(reliability_floor=32, rng_seed=7)))
    got, st_b200 = _run_engine(E, LatencyOracle(pack, OracleConfig(reliability_floor=32, rng_seed=7)))
    assert len(want) > 100 and st_ref["aborted"] is None and st_b200["aborted"] is None
    assert got == want  # same step keys, phases and bit-identical sampled latencies
    assert st_b200["finished"] == st_ref["finished"] == 40


def test_build_backend_swap(ref, monkeypatch):
    """server.build_backend with the one-line import swap of INTEGRATION.md §1:
    the constructed backend draws the reference oracle's exact stream."""
    E, RO, RP, RS = ref
    import paper_2605_00616_b200 as B

    pack = _ref_pack(RP, 3000, 1)
    path = os.path.join(os.environ.get("TMPDIR", "/tmp"), "dropin_pack.json")
    RP.save_pack_file(pack, path)
    cfg = RS.ServerConfig(engine=E.EngineConfig(num_gpu_blocks=256), backend=RS.BACKEND_ORACLE, profile_pack=path, seed=11)
    want_backend = RS.build_backend(cfg)
    monkeypatch.setattr(RS, "LatencyOracle", lambda p, c: B.LatencyOracle(p, B.OracleConfig(
        reliability_floor=c.reliability_floor, shepard_power=c.shepard_power, epsilon_distance=c.epsilon_distance,
        rng_seed=c.rng_seed)))
    got_backend = RS.build_backend(cfg)
    assert isinstance(got_backend, B.LatencyOracle)
    rng = np.random.default_rng(3)
    for _ in range(400):
        tt, conc = int(rng.integers(1, 2100)), int(rng.integers(1, 260))
        ph = RP.StepPhase.PREFILL_OR_MIXED if rng.random() < 0.4 else RP.StepPhase.DECODE_ONLY
        assert got_backend(tt, conc, ph) == want_backend(tt, conc, ph)


def test_empty_pack_aborts_engine_naming_the_query(ref):
    E, RO, RP, RS = ref
    from paper_2605_00616_b200 import LatencyOracle, OracleConfig

    empty = RP.build_pack([], num_gpu_blocks=256)
    msgs = []
    for backend in (RO.LatencyOracle(empty, RO.OracleConfig()), LatencyOracle(empty, OracleConfig())):
        async def scenario():
            cfg = E.EngineConfig(num_gpu_blocks=256, block_size=16, max_model_len=2048, max_num_batched_tokens=256,
                                 max_num_seqs=8)
            eng = E.EmulatorEngine(cfg, backend)
            h = eng.admit(10, 5)
            await eng.start()
            await asyncio.wait_for(h.done.wait(), 10)
            kind, payload = h.events.get_nowait()
            stats = eng.stats()
            await eng.stop()
            return kind, payload, stats

        kind, payload, stats = asyncio.run(scenario())
        assert kind == "error" and stats["aborted"] is not None
        msgs.append(payload["error"])
    assert msgs[0] == msgs[1]  # same query, same exception message
    assert "tt=10" in msgs[1] and "conc=1" in msgs[1] and "phase=" in msgs[1]
    assert "profile pack has no samples in any table" in msgs[1]
