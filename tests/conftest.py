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
