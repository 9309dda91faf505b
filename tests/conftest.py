"""Shared test setup.

Markers: ``gpu`` -- needs a CUDA device and the in-tree libemu_b200.so (run
on the B200 box with ``-m gpu``); everything else runs on CPU.
The CPU restatement in oracle/ is imported here as the parity checker only.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libemu_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def fixtures():
    with open(os.path.join(GOLDEN, "fixtures.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def c1_trace():
    return dict(np.load(os.path.join(GOLDEN, "c1_trace.npz")))


@pytest.fixture(scope="session")
def c1_golden():
    return dict(np.load(os.path.join(GOLDEN, "c1_golden.npz")))


@pytest.fixture(scope="session")
def c1_records(fixtures):
    from paper_2605_00616_b200.workloads import records_llama

    tt, conc, ph, lat = records_llama(50_000, 0)
    import hashlib

    h = hashlib.sha256()
    for a in (tt, conc, ph, lat):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == fixtures["c1"]["records_sha256"], "generator G drifted from the golden records"
    return tt, conc, ph, lat


@pytest.fixture(scope="session")
def c1_tables(c1_records):
    """Oracle-built canonical C1 tables (the checker's view of the pack)."""
    import emu_oracle as O

    return O.build(*c1_records, canonical=True)


# ------------------------------------------------- bench-config goldens (C2 / C3)
@pytest.fixture(scope="session")
def c2_golden():
    return dict(np.load(os.path.join(GOLDEN, "c2_golden.npz")))


@pytest.fixture(scope="session")
def c3_golden():
    return dict(np.load(os.path.join(GOLDEN, "c3_golden.npz")))


def records_sha(*cols) -> str:
    import hashlib

    h = hashlib.sha256()
    for a in cols:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def soa_digest(tt, conc, off, samples) -> str:
    """make_golden.py's table_digest over a SoA table."""
    import hashlib

    h = hashlib.sha256()
    for i in range(len(tt)):
        h.update(np.array([tt[i], conc[i], off[i + 1] - off[i]], dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(samples[off[i]:off[i + 1]], dtype=np.float64).tobytes())
    return h.hexdigest()


def pool_digests(off, bkt, dist, prob, tid, tables) -> np.ndarray:
    """Per key sha256(tt i32 | conc i32 | dist f64 | prob f64) of explicit pools
    (pool_off/bucket/dist/prob + table id per key; `tables` = the 3 SoA tables)."""
    import hashlib

    out = np.zeros((len(off) - 1, 32), np.uint8)
    for u in range(len(off) - 1):
        a, b = int(off[u]), int(off[u + 1])
        t = tables[int(tid[u])]
        h = hashlib.sha256()
        for arr, dt in ((t.tt[bkt[a:b]], "<i4"), (t.conc[bkt[a:b]], "<i4"), (dist[a:b], "<f8"), (prob[a:b], "<f8")):
            h.update(np.ascontiguousarray(arr, dtype=dt).tobytes())
        out[u] = np.frombuffer(h.digest(), np.uint8)
    return out


def check_full_pools(off, bkt, dist, prob, tid, tables, g, prefix):
    """The first keys' pools element by element against the golden arrays."""
    n = len(g[prefix + "off"]) - 1
    for u in range(n):
        a, b = int(off[u]), int(off[u + 1])
        ga, gb = int(g[prefix + "off"][u]), int(g[prefix + "off"][u + 1])
        t = tables[int(tid[u])]
        assert b - a == gb - ga, f"key {u}: K {b - a} vs {gb - ga}"
        assert np.array_equal(t.tt[bkt[a:b]], g[prefix + "tt"][ga:gb]), f"key {u}"
        assert np.array_equal(t.conc[bkt[a:b]], g[prefix + "conc"][ga:gb]), f"key {u}"
        assert np.array_equal(dist[a:b], g[prefix + "dist"][ga:gb]), f"key {u}"
        assert np.array_equal(prob[a:b], g[prefix + "prob"][ga:gb]), f"key {u}"
