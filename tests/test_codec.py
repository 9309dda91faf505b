"""Native codecs (csrc/codec.cpp) vs the reference's JSON paths (CPU; no GPU needed).

Golden files in tests/golden/ were written by the unmodified reference
(make_codec_golden.py): its save_pack bytes and trace lines, and what its
load_pack / read_trace_file return.  Bit-exact bar: keys, offsets, sample
and latency bit patterns; errors raise the reference's exception type and
message (documents outside the native subset take the json path)."""
from __future__ import annotations

import json
import os
import struct

import numpy as np
import pytest

from conftest import ROOT
from paper_2605_00616_b200 import profile as P
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
    load_pack,
    parse_trace_arrays,
    parse_trace_line,
    save_pack,
    trace_record_to_line,
)

GOLD = os.path.join(ROOT, "tests", "golden")


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def hex_doubles(h: str) -> np.ndarray:
    raw = bytes.fromhex(h)
    return np.array(struct.unpack("<%dd" % (len(raw) // 8), raw), dtype=np.float64)


def load_both(data, monkeypatch):
    native = load_pack(data)
    monkeypatch.setenv("EMU_PACK_CODEC", "json")
    ref = load_pack(data)
    monkeypatch.delenv("EMU_PACK_CODEC")
    return native, ref


def assert_same_pack(a: ProfilePack, b: ProfilePack):
    assert (a.num_gpu_blocks, a.schema_version, a.metadata) == (b.num_gpu_blocks, b.schema_version, b.metadata)
    for ta, tb in zip(a.soas(), b.soas()):
        assert np.array_equal(ta.tt, tb.tt) and np.array_equal(ta.conc, tb.conc)
        assert np.array_equal(ta.off, tb.off)
        assert np.array_equal(bits(ta.samples), bits(tb.samples))
    for ta, tb in ((a.decode_table, b.decode_table), (a.mixed_table, b.mixed_table),
                   (a.combined_table, b.combined_table)):
        assert (ta.tt_range, ta.conc_range) == (tb.tt_range, tb.conc_range)


def test_pack_golden_from_reference():
    data = open(os.path.join(GOLD, "codec_pack.json"), "rb").read()
    want = json.load(open(os.path.join(GOLD, "codec_expect.json")))["pack"]
    pack = load_pack(data)
    assert pack.num_gpu_blocks == want["num_gpu_blocks"] and pack.schema_version == want["schema_version"]
    assert pack.metadata == want["metadata"]
    for name, t in (("decode", pack.decode_table), ("mixed", pack.mixed_table), ("combined", pack.combined_table)):
        w = want["tables"][name]
        s = t.soa()
        assert t._buckets is None  # the native path built SoA tables, no bucket objects
        assert s.tt.tolist() == w["tt"] and s.conc.tolist() == w["conc"] and s.off.tolist() == w["off"]
        assert np.array_equal(bits(s.samples), bits(hex_doubles(w["samples_hex"])))
        assert list(t.tt_range) == w["tt_range"] and list(t.conc_range) == w["conc_range"]
    # the canonical bytes round-trip
    assert save_pack(pack) == data


def random_pack(rng, n_buckets=300, floats="wide"):
    def samples(k):
        if floats == "wide":
            e = rng.uniform(-320, 300, k)
            return [float(x) for x in (rng.uniform(1, 10, k) * 10.0 ** e)]
        return [float(x) for x in rng.uniform(1e-4, 1.0, k)]

    def table(kind, keys):
        return PhaseTable.from_buckets(kind, [Bucket(int(t), int(c), samples(int(rng.integers(1, 6))))
                                              for t, c in keys])

    keys = set()
    while len(keys) < n_buckets:
        keys.add((int(rng.integers(1, 5000)), int(rng.integers(1, 300))))
    keys = sorted(keys)
    dec = [(t, c) for t, c in keys if t >= c][: n_buckets // 2]
    mix = [k for k in keys if k not in set(dec)]
    d, m = table(TableKind.DECODE, dec), table(TableKind.MIXED, mix)
    comb = {}
    for b in d.buckets + m.buckets:
        comb.setdefault((b.tt, b.conc), []).extend(b.samples)
    c = PhaseTable.from_buckets(TableKind.COMBINED, [Bucket(t, cc, s) for (t, cc), s in comb.items()])
    return ProfilePack(int(rng.integers(1, 10**6)), d, m, c, {"k": "v", "z": "a\"b\\c\né\U0001f600"})


@pytest.mark.parametrize("seed", range(4))
def test_pack_random_matches_json_path(seed, monkeypatch):
    rng = np.random.default_rng(seed)
    pack = random_pack(rng, floats="wide" if seed % 2 else "unit")
    data = save_pack(pack)
    native, ref = load_both(data, monkeypatch)
    assert_same_pack(native, ref)
    assert native == pack


def test_pack_layout_variants(monkeypatch):
    """Pretty-printed, reordered keys, unknown keys, integer samples, empty tables."""
    rng = np.random.default_rng(7)
    pack = random_pack(rng, 40)
    doc = json.loads(save_pack(pack))
    doc["extra"] = {"nested": [1, 2.5, None, True, "x\\u0041"]}
    b0 = doc["tables"]["mixed"]["buckets"][0]
    b0["samples"] = list(range(1, len(b0["samples"]) + 1))  # JSON ints -> floats
    doc["tables"]["mixed"]["buckets"][0]["note"] = "ignored"
    doc["tables"]["decode"]["buckets"] = list(reversed(doc["tables"]["decode"]["buckets"]))
    for text in (json.dumps(doc, indent=2), json.dumps(doc, sort_keys=False), json.dumps(doc, separators=(",", ":"))):
        native, ref = load_both(text.encode(), monkeypatch)
        assert_same_pack(native, ref)
    empty = ProfilePack(3, PhaseTable(TableKind.DECODE, []), PhaseTable(TableKind.MIXED, []),
                        PhaseTable(TableKind.COMBINED, []))
    native, ref = load_both(save_pack(empty), monkeypatch)
    assert_same_pack(native, ref)


@pytest.mark.parametrize("doc,exc", [
    (b"{not json", PackFormatError),
    (b"[]", PackFormatError),
    (b'{"schema_version": 2, "tables": {}}', PackVersionError),
    (b'{"schema_version": 1}', PackFormatError),
    (b'{"schema_version": 1, "num_gpu_blocks": 1.5, "tables": {"decode": {"buckets": []}, '
     b'"mixed": {"buckets": []}, "combined": {"buckets": []}}}', PackFormatError),
    (b'{"schema_version": 1, "num_gpu_blocks": 0, "tables": {"decode": {"buckets": []}, '
     b'"mixed": {"buckets": []}, "combined": {"buckets": []}}}', PackValidationError),
    (b'{"schema_version": 1, "num_gpu_blocks": 4, "tables": {"decode": {"buckets": [{"tt": 3, "conc": 2, '
     b'"samples": [0.1, -2.0]}]}, "mixed": {"buckets": []}, "combined": {"buckets": [{"tt": 3, "conc": 2, '
     b'"samples": [0.1, 2.0]}]}}}', PackValidationError),
    (b'{"schema_version": 1, "num_gpu_blocks": 4, "tables": {"decode": {"buckets": [{"tt": 3, "conc": 2, '
     b'"samples": [0.1]}, {"tt": 3, "conc": 2, "samples": [0.2]}]}, "mixed": {"buckets": []}, '
     b'"combined": {"buckets": [{"tt": 3, "conc": 2, "samples": [0.1, 0.2]}]}}}', PackValidationError),
    (b'{"schema_version": 1, "num_gpu_blocks": 4, "tables": {"decode": {"buckets": [{"tt": 0, "conc": 2, '
     b'"samples": [0.1]}]}, "mixed": {"buckets": []}, "combined": {"buckets": []}}}', PackValidationError),
    (b'{"schema_version": 1, "num_gpu_blocks": 4, "tables": {"decode": {"buckets": [{"tt": 3, "conc": 2, '
     b'"samples": []}]}, "mixed": {"buckets": []}, "combined": {"buckets": []}}}', PackValidationError),
    (b'{"schema_version": 1, "num_gpu_blocks": 4, "tables": {"decode": {"buckets": [{"tt": 3, "conc": 2, '
     b'"samples": [NaN]}]}, "mixed": {"buckets": []}, "combined": {"buckets": [{"tt": 3, "conc": 2, '
     b'"samples": [1.0]}]}}}', PackValidationError),
    (b'{"schema_version": 1, "num_gpu_blocks": 4, "tables": {"decode": {"buckets": []}, "mixed": {"buckets": []},'
     b' "combined": {"buckets": [{"tt": 3, "conc": 2, "samples": [0.5]}]}}}', PackValidationError),
])
def test_pack_errors_match_json_path(doc, exc, monkeypatch):
    with pytest.raises(exc) as native:
        load_pack(doc)
    monkeypatch.setenv("EMU_PACK_CODEC", "json")
    with pytest.raises(exc) as ref:
        load_pack(doc)
    assert str(native.value) == str(ref.value)


# ------------------------------------------------------------------ traces
def test_trace_golden_from_reference():
    text = open(os.path.join(GOLD, "codec_trace.jsonl"), "rb").read()
    want = json.load(open(os.path.join(GOLD, "codec_expect.json")))["trace"]
    for threads in (1, 7):
        step, tt, conc, ph, lat = parse_trace_arrays(text, threads)
        assert step.tolist() == want["step"] and tt.tolist() == want["tt"] and conc.tolist() == want["conc"]
        assert [("decode", "mixed")[p] for p in ph.tolist()] == want["phase"]
        assert np.array_equal(bits(lat), bits(hex_doubles(want["latency_hex"])))


def test_trace_random_matches_parse_trace_line():
    rng = np.random.default_rng(3)
    recs = [StepTraceRecord(int(i), int(rng.integers(1, 10**6)), int(rng.integers(1, 512)),
                            StepPhase.DECODE_ONLY if rng.random() < 0.5 else StepPhase.PREFILL_OR_MIXED,
                            float(rng.uniform(1, 10) * 10.0 ** rng.uniform(-300, 300))) for i in range(5000)]
    lines = [trace_record_to_line(r) for r in recs]
    lines[10] = "   " + lines[10] + "  \r"
    lines.insert(20, "")
    lines.insert(30, "   \t")
    lines[40] = json.dumps({**json.loads(lines[40]), "extra": [1, {"a": "b"}]}, indent=1).replace("\n", " ")
    text = "\r\n".join(lines)
    ref = [parse_trace_line(s) for s in (ln.strip() for ln in text.splitlines()) if s]
    for threads in (1, 3, 16):
        step, tt, conc, ph, lat = parse_trace_arrays(text, threads)
        assert len(step) == len(ref)
        assert step.tolist() == [r.step_index for r in ref]
        assert tt.tolist() == [r.total_tokens for r in ref] and conc.tolist() == [r.concurrency for r in ref]
        assert ph.tolist() == [0 if r.phase == StepPhase.DECODE_ONLY else 1 for r in ref]
        assert np.array_equal(bits(lat), bits([r.latency_s for r in ref]))


def test_trace_outside_subset_uses_reference_semantics():
    # coercions the reference accepts (int("3") via float / numeric strings) and its errors
    ok = '{"step": 1.0, "tt": 5, "conc": 2, "phase": "mixed", "latency_s": "0.25"}\n'
    step, tt, conc, ph, lat = parse_trace_arrays(ok)
    r = parse_trace_line(ok.strip())
    assert (step[0], tt[0], conc[0], lat[0]) == (r.step_index, r.total_tokens, r.concurrency, r.latency_s)
    bad = '{"step": 1, "tt": 5, "conc": 2, "phase": "prefill", "latency_s": 0.25}\n'
    with pytest.raises(PackFormatError) as native:
        parse_trace_arrays(bad)
    with pytest.raises(PackFormatError) as ref:
        parse_trace_line(bad.strip())
    assert str(native.value) == str(ref.value)
