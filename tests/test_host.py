"""Host-side logic (CPU): the C-ABI library surface, pack containers and codec."""
from __future__ import annotations

import ctypes
import json
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2605_00616_b200 import _lib
from paper_2605_00616_b200.profile import (
    Bucket,
    PackFormatError,
    PackValidationError,
    PackVersionError,
    PhaseTable,
    ProfilePack,
    StepPhase,
    StepTraceRecord,
    TableKind,
    TableSoA,
    load_pack,
    parse_trace_line,
    phase_code,
    save_pack,
    trace_record_to_line,
)

DEC, MIX = StepPhase.DECODE_ONLY, StepPhase.PREFILL_OR_MIXED


def header_functions():
    text = open(os.path.join(ROOT, "include", "emu_abi.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(emu_[a-z0-9_]+)\s*\(", text,
                                 flags=re.M)))


def test_library_builds_and_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = header_functions()
    assert len(names) >= 18, names
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/emu_abi.h but not exported"
        assert n in _lib.SIGNATURES, f"{n} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(names)


def test_library_reports_version_and_errors_without_gpu():
    lib = _lib.load_library()
    assert lib.emu_version() == 1
    # argument validation fails before touching the device
    out = ctypes.c_void_p()
    rc = lib.emu_oracle_create(None, 32, 2.0, 1e-9, 0, 0, 0, 0, None, ctypes.byref(out))
    assert rc == _lib.EMU_ERR_INVALID
    assert "NULL" in _lib.last_error()


def test_status_mapping():
    from paper_2605_00616_b200.oracle import NoProfileDataError

    with pytest.raises(NoProfileDataError):
        _lib.check(_lib.EMU_ERR_NO_DATA, no_data_exc=NoProfileDataError)
    with pytest.raises(ValueError):
        _lib.check(_lib.EMU_ERR_INVALID)
    with pytest.raises(_lib.CapacityError):
        _lib.check(_lib.EMU_ERR_CAPACITY)
    with pytest.raises(_lib.EmuError):
        _lib.check(_lib.EMU_ERR_CUDA)


def test_phase_codes_accept_reference_enums():
    class RefPhase:  # duck-typed reference StepPhase
        def __init__(self, v):
            self.value = v

    assert phase_code(DEC) == 0 and phase_code(MIX) == 1
    assert phase_code(RefPhase("decode")) == 0 and phase_code(RefPhase("mixed")) == 1
    assert phase_code("mixed") == 1 and phase_code(0) == 0
    with pytest.raises(ValueError):
        phase_code("prefill")


def test_canonical_bytes_match_reference(fixtures):
    recs_pack = ProfilePack(
        7,
        PhaseTable.from_buckets(TableKind.DECODE, [Bucket(3, 3, [0.012, 0.010])]),
        PhaseTable.from_buckets(TableKind.MIXED, [Bucket(64, 1, [0.05]), Bucket(7, 2, [0.02])]),
        PhaseTable.from_buckets(TableKind.COMBINED, [Bucket(3, 3, [0.012, 0.010]), Bucket(64, 1, [0.05]),
                                                     Bucket(7, 2, [0.02])]),
        {"model": "toy", "gpu": "none"},
    )
    assert save_pack(recs_pack).decode() == fixtures["small_pack_bytes"]
    back = load_pack(save_pack(recs_pack))
    assert back == recs_pack


def test_soa_backed_table_round_trips():
    soa = TableSoA(np.array([3, 7, 64], np.int32), np.array([3, 2, 1], np.int32), np.array([0, 2, 3, 4], np.int64),
                   np.array([0.012, 0.010, 0.02, 0.05]))
    t = PhaseTable.from_soa(TableKind.COMBINED, soa)
    assert t.tt_range == (3, 64) and t.conc_range == (1, 3)
    assert [b.samples for b in t.buckets] == [[0.012, 0.010], [0.02], [0.05]]
    assert t == PhaseTable.from_buckets(TableKind.COMBINED, t.buckets)


def test_pack_errors():
    data = save_pack(ProfilePack(5, *(PhaseTable.from_buckets(k, []) for k in TableKind)))
    with pytest.raises(PackFormatError, match="malformed"):
        load_pack(b"{nope")
    obj = json.loads(data)
    obj["schema_version"] = 99
    with pytest.raises(PackVersionError):
        load_pack(json.dumps(obj))
    pack = ProfilePack(5, PhaseTable.from_buckets(TableKind.DECODE, [Bucket(3, 3, [0.01])]),
                       PhaseTable.from_buckets(TableKind.MIXED, []),
                       PhaseTable.from_buckets(TableKind.COMBINED, [Bucket(3, 3, [0.01])]))
    obj = json.loads(save_pack(pack))
    obj["tables"]["combined"]["buckets"][0]["samples"].append(0.02)
    with pytest.raises(PackValidationError, match="combined table inconsistent"):
        load_pack(json.dumps(obj))
    obj = json.loads(save_pack(pack))
    obj["tables"]["decode"]["buckets"].append({"tt": 3, "conc": 3, "samples": [0.02]})
    with pytest.raises(PackValidationError, match="duplicate"):
        load_pack(json.dumps(obj))
    obj = json.loads(save_pack(pack))
    obj["tables"]["decode"]["buckets"][0]["samples"] = []
    with pytest.raises(PackValidationError, match="no samples"):
        load_pack(json.dumps(obj))


def test_record_validation_messages():
    with pytest.raises(PackValidationError, match="decode-only"):
        StepTraceRecord(0, 2, 3, DEC, 0.01).validate()
    with pytest.raises(PackValidationError, match="latency_s must be > 0"):
        StepTraceRecord(0, 2, 2, DEC, 0.0).validate()
    StepTraceRecord(0, 2, 3, MIX, 0.01).validate()


def test_trace_lines():
    r = StepTraceRecord(4, 17, 3, MIX, 0.0123)
    assert parse_trace_line(trace_record_to_line(r)) == r
    assert json.loads(trace_record_to_line(StepTraceRecord(1, 5, 5, DEC, 0.01))) == {
        "step": 1, "tt": 5, "conc": 5, "phase": "decode", "latency_s": 0.01}
    with pytest.raises(PackFormatError):
        parse_trace_line('{"step": 1}')


def test_workload_generators_are_deterministic():
    from paper_2605_00616_b200.workloads import queries_llama, queries_sparse, records_llama

    a = records_llama(1000, 0)
    b = records_llama(1000, 0)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    tt, conc, ph = queries_llama(5000, 1)
    assert (tt[ph == 0] == conc[ph == 0]).all() and tt.max() <= 2048 and conc.max() <= 256
    tt, conc, ph = queries_sparse(5000, 1)
    assert tt.max() <= 131072


def test_scheduler_admission_checks_without_gpu():
    """emu_sched_create validates the request table on host threads before any
    device allocation (engine.py:323-336 messages, the first bad request wins)."""
    lib = _lib.load_library()
    S, n = 3, 1 << 21  # large enough for the threaded path
    off = np.array([0, n, 2 * n, 3 * n], np.int64)
    prompt = np.full(3 * n, 100, np.int32)
    target = np.full(3 * n, 50, np.int32)
    arrival = np.concatenate([np.arange(n, dtype=np.float64)] * 3)  # restarts per scenario: fine

    def create(p, t, a, blocks=1000, max_len=4096):
        h = ctypes.c_void_p()
        rc = lib.emu_sched_create(S, _lib.ptr(off), _lib.ptr(p), _lib.ptr(t), _lib.ptr(a), blocks, 16, max_len, 512,
                                  64, 10, ctypes.byref(h))
        return rc, _lib.last_error(), h

    p = prompt.copy()
    p[2 * n + 5] = 0
    p[n + 7] = 5000  # the earlier bad request reports
    rc, msg, _ = create(p, target, arrival)
    assert rc == _lib.EMU_ERR_INVALID and "exceeds max_model_len" in msg and "5050" in msg
    t = target.copy()
    t[3] = 0
    assert "max_tokens must be >= 1, got 0" in create(prompt, t, arrival)[1]
    assert "KV blocks" in create(prompt, target, arrival, blocks=5)[1]
    a = arrival.copy()
    a[n + 10] = -1.0
    assert "arrival offsets must ascend" in create(prompt, target, a)[1]
