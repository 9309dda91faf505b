"""Profile packs for the B200 oracle: the reference's profile API, GPU-built.

Drop-in mirror of ``serve_emu.profile`` (/root/reference/pkg/src/serve_emu/
profile.py).  Names, argument meaning, invariants and error types/messages
match the reference; what changes is where the work happens:

* ``build_pack`` / ``build_pack_arrays`` run the table build on the GPU
  (``emu_tables_build``: validate -> key pack -> stable LSD radix sort ->
  segment -> phase partition), replacing the per-record dict appends of
  profile.py:230-267.  The resulting tables stay resident in HBM and are
  handed to ``LatencyOracle`` without another upload; Python ``Bucket``
  objects are materialised lazily, only if someone asks for them.
* JSON (de)serialisation keeps the reference's canonical byte format
  (profile.py:275-347) so packs interchange with the reference unchanged.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from enum import Enum
from pathlib import Path
from typing import Iterable, Iterator, Sequence

import numpy as np

SCHEMA_VERSION = 1


class StepPhase(Enum):
    """Step classification (profile.py:20-25); values are the wire strings."""

    DECODE_ONLY = "decode"
    PREFILL_OR_MIXED = "mixed"


class TableKind(Enum):
    DECODE = "decode"
    MIXED = "mixed"
    COMBINED = "combined"


class PackFormatError(ValueError):
    """Pack or trace bytes cannot be parsed at all."""


class PackVersionError(ValueError):
    """Pack schema_version is missing or unsupported."""


class PackValidationError(ValueError):
    """Parsed data violates a pack invariant."""


def phase_code(phase) -> int:
    """0 for decode-only, 1 for prefill-or-mixed.  Accepts this module's
    StepPhase, the reference's StepPhase (by .value), the wire strings and 0/1."""
    v = getattr(phase, "value", phase)
    if v == "decode" or v == 0:
        return 0
    if v == "mixed" or v == 1:
        return 1
    raise ValueError(f"unknown step phase {phase!r}")


# ---------------------------------------------------------------------------
# Records
# ---------------------------------------------------------------------------

_CHECK_MESSAGES = {
    1: lambda s, t, c, p, l: f"step_index must be >= 0, got {s}",
    2: lambda s, t, c, p, l: f"total_tokens must be >= 1, got {t}",
    3: lambda s, t, c, p, l: f"concurrency must be >= 1, got {c}",
    4: lambda s, t, c, p, l: f"decode-only step has total_tokens={t} < concurrency={c}",
    5: lambda s, t, c, p, l: f"latency_s must be > 0, got {l}",
}


def _first_failed_check(step, tt, conc, phase, lat) -> int:
    """Index (1..5) of the first StepTraceRecord.validate check that fails
    (profile.py:61-79), 0 if the record is valid."""
    if step is not None and step < 0:
        return 1
    if tt < 1:
        return 2
    if conc < 1:
        return 3
    if phase == 0 and tt < conc:
        return 4
    if not lat > 0:
        return 5
    return 0


@dataclass(frozen=True)
class StepTraceRecord:
    """One per-step observation: tt total tokens, conc running requests."""

    step_index: int
    total_tokens: int
    concurrency: int
    phase: StepPhase
    latency_s: float

    def validate(self) -> None:
        code = _first_failed_check(self.step_index, self.total_tokens, self.concurrency,
                                   phase_code(self.phase), self.latency_s)
        if code:
            raise PackValidationError(_CHECK_MESSAGES[code](
                self.step_index, self.total_tokens, self.concurrency, phase_code(self.phase), self.latency_s))


# ---------------------------------------------------------------------------
# Buckets and tables
# ---------------------------------------------------------------------------


@dataclass(eq=False)
class Bucket:
    """Raw latency samples observed at one exact (tt, conc) point."""

    tt: int
    conc: int
    samples: list[float]

    def validate(self) -> None:
        if self.tt < 1 or self.conc < 1:
            raise PackValidationError(f"bucket key ({self.tt}, {self.conc}) must be positive")
        if not self.samples:
            raise PackValidationError(f"bucket ({self.tt}, {self.conc}) has no samples")
        bad = [s for s in self.samples if not s > 0]
        if bad:
            raise PackValidationError(f"bucket ({self.tt}, {self.conc}) has nonpositive sample {bad[0]}")

    def __eq__(self, other: object) -> bool:
        # capture order is kept, comparison is as a multiset (canonical form)
        if not isinstance(other, Bucket) and not hasattr(other, "samples"):
            return NotImplemented
        return (self.tt, self.conc) == (other.tt, other.conc) and sorted(self.samples) == sorted(other.samples)


@dataclass
class TableSoA:
    """Host copy of one table in the device layout (include/emu_abi.h)."""

    tt: np.ndarray  # int32[B], sorted by (tt, conc)
    conc: np.ndarray  # int32[B]
    off: np.ndarray  # int64[B+1]
    samples: np.ndarray  # float64[N]

    @staticmethod
    def empty() -> "TableSoA":
        return TableSoA(np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(1, np.int64),
                        np.zeros(0, np.float64))

    @staticmethod
    def from_buckets(buckets: Sequence) -> "TableSoA":
        n = len(buckets)
        tt = np.fromiter((b.tt for b in buckets), dtype=np.int64, count=n)
        conc = np.fromiter((b.conc for b in buckets), dtype=np.int64, count=n)
        counts = np.fromiter((len(b.samples) for b in buckets), dtype=np.int64, count=n)
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=off[1:])
        samples = np.fromiter((s for b in buckets for s in b.samples), dtype=np.float64, count=int(off[-1]))
        if n and (tt.max() > 0x7FFFFFFF or conc.max() > 0x7FFFFFFF):
            raise PackValidationError("bucket keys must fit in int32")
        return TableSoA(tt.astype(np.int32), conc.astype(np.int32), off, samples)

    def ranges(self):
        if len(self.tt) == 0:
            return None, None
        return (int(self.tt[0]), int(self.tt[-1])), (int(self.conc.min()), int(self.conc.max()))


class PhaseTable:
    """All buckets of one table plus the key ranges used for distance scaling.

    Either holds a Python bucket list (as the reference does) or wraps a
    TableSoA produced by the GPU build, materialising ``buckets`` on demand.
    """

    def __init__(self, kind: TableKind, buckets: list[Bucket] | None = None,
                 tt_range: tuple[int, int] | None = None, conc_range: tuple[int, int] | None = None,
                 *, soa: TableSoA | None = None):
        self.kind = kind
        self._buckets = buckets
        self._soa = soa
        self.tt_range = tt_range
        self.conc_range = conc_range

    # -- construction ---------------------------------------------------------
    @classmethod
    def from_buckets(cls, kind: TableKind, buckets: Iterable) -> "PhaseTable":
        ordered = sorted(buckets, key=lambda b: (b.tt, b.conc))
        if not ordered:
            return cls(kind, [], None, None)
        tt_range = (ordered[0].tt, ordered[-1].tt)
        concs = [b.conc for b in ordered]
        return cls(kind, ordered, tt_range, (min(concs), max(concs)))

    @classmethod
    def from_soa(cls, kind: TableKind, soa: TableSoA) -> "PhaseTable":
        tt_range, conc_range = soa.ranges()
        return cls(kind, None, tt_range, conc_range, soa=soa)

    # -- views ------------------------------------------------------------------
    @property
    def buckets(self) -> list[Bucket]:
        if self._buckets is None:
            s = self._soa
            tt, conc, off = s.tt.tolist(), s.conc.tolist(), s.off.tolist()
            smp = s.samples
            self._buckets = [Bucket(tt[i], conc[i], smp[off[i]:off[i + 1]].tolist()) for i in range(len(tt))]
        return self._buckets

    @buckets.setter
    def buckets(self, value: list[Bucket]) -> None:
        self._buckets = value
        self._soa = None

    def soa(self) -> TableSoA:
        """SoA view in (tt, conc) order, sample order preserved per bucket."""
        if self._soa is None or self._buckets is not None and len(self._buckets) != len(self._soa.tt):
            bl = self._buckets or []
            keys = [(b.tt, b.conc) for b in bl]
            if keys != sorted(keys):
                bl = sorted(bl, key=lambda b: (b.tt, b.conc))
            self._soa = TableSoA.from_buckets(bl) if bl else TableSoA.empty()
        return self._soa

    @property
    def total_samples(self) -> int:
        if self._buckets is None:
            return int(self._soa.off[-1])
        return sum(len(b.samples) for b in self._buckets)

    @property
    def is_empty(self) -> bool:
        if self._buckets is None:
            return len(self._soa.tt) == 0
        return not self._buckets

    def validate(self) -> None:
        seen: set[tuple[int, int]] = set()
        for b in self.buckets:
            b.validate()
            key = (b.tt, b.conc)
            if key in seen:
                raise PackValidationError(f"{self.kind.value} table has duplicate bucket {key}")
            seen.add(key)
        derived = PhaseTable.from_buckets(self.kind, self.buckets)
        if (derived.tt_range, derived.conc_range) != (self.tt_range, self.conc_range):
            raise PackValidationError(
                f"{self.kind.value} table ranges {self.tt_range}/{self.conc_range} do not "
                f"match bucket extrema {derived.tt_range}/{derived.conc_range}"
            )

    def _canon(self) -> dict:
        return {(b.tt, b.conc): sorted(b.samples) for b in self.buckets}

    def __eq__(self, other: object) -> bool:
        if not hasattr(other, "buckets") or not hasattr(other, "kind"):
            return NotImplemented
        return (
            getattr(self.kind, "value", self.kind) == getattr(other.kind, "value", other.kind)
            and (self.tt_range, self.conc_range) == (other.tt_range, other.conc_range)
            and self._canon() == {(b.tt, b.conc): sorted(b.samples) for b in other.buckets}
        )

    def __repr__(self) -> str:
        n = len(self._soa.tt) if self._buckets is None else len(self._buckets)
        return f"PhaseTable({self.kind.value}, {n} buckets, tt={self.tt_range}, conc={self.conc_range})"


@dataclass(eq=False)
class ProfilePack:
    """The profiling artifact the latency oracle samples from."""

    num_gpu_blocks: int
    decode_table: PhaseTable
    mixed_table: PhaseTable
    combined_table: PhaseTable
    metadata: dict[str, str] = field(default_factory=dict)
    schema_version: int = SCHEMA_VERSION
    # device tables from the GPU build (reused by LatencyOracle, not compared)
    _device: object = field(default=None, repr=False)
    _trusted: bool = field(default=False, repr=False)

    def validate(self) -> None:
        if self.num_gpu_blocks < 1:
            raise PackValidationError(f"num_gpu_blocks must be >= 1, got {self.num_gpu_blocks}")
        if self._trusted:
            return  # built by the GPU build from validated records
        for table, kind in ((self.decode_table, TableKind.DECODE), (self.mixed_table, TableKind.MIXED),
                            (self.combined_table, TableKind.COMBINED)):
            if getattr(table.kind, "value", table.kind) != kind.value:
                raise PackValidationError(f"table kind mismatch: {table.kind} != {kind}")
            table.validate()
        phase_total = self.decode_table.total_samples + self.mixed_table.total_samples
        if self.combined_table.total_samples != phase_total:
            raise PackValidationError(
                "combined table inconsistent: "
                f"{self.combined_table.total_samples} samples != decode+mixed {phase_total}"
            )

    def table_for(self, phase) -> PhaseTable:
        return self.decode_table if phase_code(phase) == 0 else self.mixed_table

    def stats(self) -> dict:
        per = {}
        for t in (self.decode_table, self.mixed_table, self.combined_table):
            nb = len(t._soa.tt) if t._buckets is None else len(t._buckets)
            per[t.kind.value] = {"buckets": nb, "samples": t.total_samples}
        return {
            "per_table": per,
            "total_buckets": sum(v["buckets"] for v in per.values()),
            "total_samples": sum(v["samples"] for v in per.values()),
            "num_gpu_blocks": self.num_gpu_blocks,
        }

    def soas(self) -> list[TableSoA]:
        return [self.decode_table.soa(), self.mixed_table.soa(), self.combined_table.soa()]

    def __eq__(self, other: object) -> bool:
        if not hasattr(other, "combined_table"):
            return NotImplemented
        return (
            self.schema_version == other.schema_version
            and self.metadata == other.metadata
            and self.num_gpu_blocks == other.num_gpu_blocks
            and self.decode_table == other.decode_table
            and self.mixed_table == other.mixed_table
            and self.combined_table == other.combined_table
        )


# ---------------------------------------------------------------------------
# GPU build
# ---------------------------------------------------------------------------


def records_to_arrays(traces: Iterable[StepTraceRecord]):
    """Columnar copy of record objects (host ingest)."""
    step, tt, conc, ph, lat = [], [], [], [], []
    for r in traces:
        step.append(r.step_index)
        tt.append(r.total_tokens)
        conc.append(r.concurrency)
        ph.append(phase_code(r.phase))
        lat.append(r.latency_s)
    return (np.asarray(tt, dtype=np.int64), np.asarray(conc, dtype=np.int64), np.asarray(ph, dtype=np.uint8),
            np.asarray(lat, dtype=np.float64), np.asarray(step, dtype=np.int64))


def build_pack(traces: Iterable[StepTraceRecord], num_gpu_blocks: int,
               metadata: dict[str, str] | None = None, *, canonical: bool = False) -> ProfilePack:
    """Bucket step records into a pack on the GPU (profile.py:230-267).

    Every record lands in its phase table and in the combined table.  With
    ``canonical=False`` (default) samples keep capture order inside a bucket,
    exactly like the reference's in-memory pack; ``canonical=True`` sorts them
    ascending (the order ``load_pack(save_pack(p))`` yields).
    """
    if num_gpu_blocks < 1:
        raise PackValidationError(f"num_gpu_blocks must be >= 1, got {num_gpu_blocks}")
    tt, conc, ph, lat, step = records_to_arrays(traces)
    return build_pack_arrays(tt, conc, ph, lat, num_gpu_blocks, metadata, step=step, canonical=canonical)


def build_pack_arrays(tt, conc, phase, latency_s, num_gpu_blocks: int, metadata: dict[str, str] | None = None,
                      *, step=None, canonical: bool = False, keep_host: bool = True) -> ProfilePack:
    """GPU build from columnar records (numpy arrays or CUDA tensors)."""
    from .device import DeviceTables

    if num_gpu_blocks < 1:
        raise PackValidationError(f"num_gpu_blocks must be >= 1, got {num_gpu_blocks}")
    dev = DeviceTables.build(tt, conc, phase, latency_s, step=step, canonical=canonical)
    return pack_from_device(dev, num_gpu_blocks, metadata, keep_host=keep_host)


def pack_from_device(dev, num_gpu_blocks: int, metadata: dict[str, str] | None = None,
                     keep_host: bool = True) -> ProfilePack:
    soas = dev.to_host() if keep_host else [TableSoA.empty()] * 3
    kinds = (TableKind.DECODE, TableKind.MIXED, TableKind.COMBINED)
    tables = [PhaseTable.from_soa(k, s) for k, s in zip(kinds, soas)]
    if not keep_host:
        for t, i in zip(tables, range(3)):
            info = dev.info(i)
            t.tt_range, t.conc_range = info["tt_range"], info["conc_range"]
    return ProfilePack(num_gpu_blocks, tables[0], tables[1], tables[2], dict(metadata or {}), SCHEMA_VERSION,
                       _device=dev, _trusted=True)


# ---------------------------------------------------------------------------
# Canonical JSON (byte-compatible with the reference, profile.py:275-347)
# ---------------------------------------------------------------------------


def _table_json(table: PhaseTable) -> dict:
    if table._buckets is None:
        s = table._soa
        off = s.off.tolist()
        rows = [
            {"tt": int(s.tt[i]), "conc": int(s.conc[i]), "samples": sorted(s.samples[off[i]:off[i + 1]].tolist())}
            for i in range(len(s.tt))
        ]
    else:
        rows = [{"tt": b.tt, "conc": b.conc, "samples": sorted(b.samples)}
                for b in sorted(table.buckets, key=lambda b: (b.tt, b.conc))]
    return {"buckets": rows}


def save_pack(pack: ProfilePack) -> bytes:
    """Canonical JSON: buckets by key, samples ascending, sorted object keys."""
    doc = {
        "schema_version": pack.schema_version,
        "metadata": dict(sorted(pack.metadata.items())),
        "num_gpu_blocks": pack.num_gpu_blocks,
        "tables": {k: _table_json(t) for k, t in (("decode", pack.decode_table), ("mixed", pack.mixed_table),
                                                    ("combined", pack.combined_table))},
    }
    return json.dumps(doc, sort_keys=True, separators=(",", ":")).encode("utf-8")


def _parse_table(tables_obj: dict, kind: TableKind) -> PhaseTable:
    raw = tables_obj.get(kind.value)
    if not isinstance(raw, dict) or not isinstance(raw.get("buckets"), list):
        raise PackFormatError(f"table {kind.value!r} is missing or malformed")
    out = []
    for entry in raw["buckets"]:
        try:
            out.append(Bucket(int(entry["tt"]), int(entry["conc"]), [float(x) for x in entry["samples"]]))
        except (KeyError, TypeError, ValueError) as exc:
            raise PackFormatError(f"malformed bucket in {kind.value} table: {exc}") from None
    return PhaseTable.from_buckets(kind, out)


def _load_pack_json(text: str) -> ProfilePack:
    """The reference's json.loads path (profile.py:299-347): the fallback of
    load_pack and the source of its exact error messages."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise PackFormatError(f"malformed pack JSON: {exc}") from None
    if not isinstance(doc, dict):
        raise PackFormatError("pack JSON top level must be an object")
    version = doc.get("schema_version")
    if version != SCHEMA_VERSION:
        raise PackVersionError(f"unsupported schema_version {version!r}, expected {SCHEMA_VERSION}")
    tables_obj = doc.get("tables")
    if not isinstance(tables_obj, dict):
        raise PackFormatError("pack JSON is missing the tables object")
    decode, mixed, combined = (_parse_table(tables_obj, k) for k in
                               (TableKind.DECODE, TableKind.MIXED, TableKind.COMBINED))
    metadata = doc.get("metadata", {})
    if not isinstance(metadata, dict):
        raise PackFormatError("metadata must be an object")
    blocks = doc.get("num_gpu_blocks")
    if not isinstance(blocks, int) or isinstance(blocks, bool):
        raise PackFormatError("num_gpu_blocks must be an integer")
    pack = ProfilePack(blocks, decode, mixed, combined, {str(k): str(v) for k, v in metadata.items()}, version)
    pack.validate()
    return pack


def _load_pack_native(raw: bytes):
    """emu_pack_parse_json (csrc/codec.cpp): the pack as three TableSoA, or None
    when the document is outside the native subset (-> the json path)."""
    import ctypes

    from . import _lib

    L = _lib.lib()
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(raw, len(raw))
    rc = L.emu_pack_parse_json(buf, len(raw), ctypes.byref(h))
    if rc == _lib.EMU_ERR_UNSUPPORTED:
        return None
    _lib.check(rc, invalid_exc=PackFormatError)
    try:
        ver, blocks, mlen = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        sizes = np.zeros(6, dtype=np.int64)
        _lib.check(L.emu_pack_parsed_info(h, ctypes.byref(ver), ctypes.byref(blocks), _lib.ptr(sizes),
                                          ctypes.byref(mlen)))
        soas = []
        for t in range(3):
            B, N = int(sizes[2 * t]), int(sizes[2 * t + 1])
            s = TableSoA(np.empty(B, np.int32), np.empty(B, np.int32), np.empty(B + 1, np.int64),
                         np.empty(N, np.float64))
            _lib.check(L.emu_pack_parsed_copy(h, t, _lib.ptr(s.tt), _lib.ptr(s.conc), _lib.ptr(s.off),
                                              _lib.ptr(s.samples)))
            soas.append(s)
        mbuf = ctypes.create_string_buffer(max(1, mlen.value))
        _lib.check(L.emu_pack_parsed_metadata(h, mbuf, mlen.value))
        metadata = json.loads(mbuf.raw[:mlen.value].decode("utf-8"))
    finally:
        L.emu_pack_parsed_free(h)
    return int(ver.value), int(blocks.value), metadata, soas


def _validate_soa_table(kind: TableKind, s: TableSoA) -> None:
    """PhaseTable.validate for a SoA table without materialising buckets: the
    first bucket (in (tt, conc) order) that fails Bucket.validate or repeats a
    key raises exactly the message the bucket walk would raise."""
    B = len(s.tt)
    if B == 0:
        return
    counts = np.diff(s.off)
    bad = (s.tt < 1) | (s.conc < 1) | (counts == 0)
    nonpos = ~(s.samples > 0)
    if nonpos.any():
        seg = np.searchsorted(s.off, np.flatnonzero(nonpos), side="right") - 1
        bad[seg] = True
    dup = np.zeros(B, dtype=bool)
    dup[1:] = (s.tt[1:] == s.tt[:-1]) & (s.conc[1:] == s.conc[:-1])
    hit = np.flatnonzero(bad | dup)
    if len(hit) == 0:
        return
    i = int(hit[0])
    Bucket(int(s.tt[i]), int(s.conc[i]), s.samples[s.off[i]:s.off[i + 1]].tolist()).validate()
    raise PackValidationError(f"{kind.value} table has duplicate bucket {(int(s.tt[i]), int(s.conc[i]))}")


def load_pack(data: bytes | str) -> ProfilePack:
    """Parse and validate pack bytes; ranges are derived from the buckets.

    Well-formed documents go through the native codec (csrc/codec.cpp) into
    SoA tables -- bit-identical to the reference's parse -- and are validated
    vectorised; anything else takes the reference's json.loads path, which
    raises its exact errors."""
    raw = data.encode("utf-8") if isinstance(data, str) else bytes(data)
    parsed = None
    if os.environ.get("EMU_PACK_CODEC", "native") != "json":
        parsed = _load_pack_native(raw)
    if parsed is None:
        return _load_pack_json(raw.decode("utf-8"))
    version, blocks, metadata, soas = parsed
    kinds = (TableKind.DECODE, TableKind.MIXED, TableKind.COMBINED)
    tables = [PhaseTable.from_soa(k, s) for k, s in zip(kinds, soas)]
    pack = ProfilePack(blocks, *tables, {str(k): str(v) for k, v in metadata.items()}, version)
    if pack.num_gpu_blocks < 1:
        raise PackValidationError(f"num_gpu_blocks must be >= 1, got {pack.num_gpu_blocks}")
    for k, s in zip(kinds, soas):
        _validate_soa_table(k, s)
    phase_total = int(soas[0].off[-1]) + int(soas[1].off[-1])
    if int(soas[2].off[-1]) != phase_total:
        raise PackValidationError(
            f"combined table inconsistent: {int(soas[2].off[-1])} samples != decode+mixed {phase_total}")
    return pack


def save_pack_file(pack: ProfilePack, path: str | Path) -> None:
    Path(path).write_bytes(save_pack(pack))


def load_pack_file(path: str | Path) -> ProfilePack:
    return load_pack(Path(path).read_bytes())


# ---------------------------------------------------------------------------
# Trace files (JSON lines, one StepTraceRecord per line)
# ---------------------------------------------------------------------------


def trace_record_to_line(rec: StepTraceRecord) -> str:
    return json.dumps({"step": rec.step_index, "tt": rec.total_tokens, "conc": rec.concurrency,
                       "phase": rec.phase.value, "latency_s": rec.latency_s}, separators=(",", ":"))


def parse_trace_line(line: str) -> StepTraceRecord:
    try:
        o = json.loads(line)
        return StepTraceRecord(int(o["step"]), int(o["tt"]), int(o["conc"]), StepPhase(o["phase"]),
                               float(o["latency_s"]))
    except (json.JSONDecodeError, KeyError, TypeError, ValueError) as exc:
        raise PackFormatError(f"malformed trace line: {exc}") from None


def read_trace_file(path: str | Path) -> list[StepTraceRecord]:
    with open(path, "r", encoding="utf-8") as f:
        return [parse_trace_line(s) for s in (ln.strip() for ln in f) if s]


def iter_trace_dir(path: str | Path) -> Iterator[StepTraceRecord]:
    for file in sorted(Path(path).glob("*.jsonl")):
        yield from read_trace_file(file)


def parse_trace_arrays(text: bytes | str, threads: int = 0):
    """JSONL trace text -> record columns (step i64, tt i32, conc i32, phase u8,
    latency_s f64) in file order, via emu_trace_parse_jsonl (csrc/codec.cpp,
    multithreaded).  Same records as [parse_trace_line(l) for l in lines]; a
    line outside the native subset re-reads the text line by line with
    parse_trace_line (the reference's errors and coercions)."""
    import ctypes

    from . import _lib

    raw = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    L = _lib.lib()
    buf = ctypes.create_string_buffer(raw, len(raw))
    n = int(L.emu_trace_count_lines(buf, len(raw)))
    cols = (np.empty(n, np.int64), np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.uint8),
            np.empty(n, np.float64))
    n_out, bad = ctypes.c_int64(), ctypes.c_int64()
    threads = threads or min(32, len(os.sched_getaffinity(0)))
    rc = L.emu_trace_parse_jsonl(buf, len(raw), int(threads), n, *(_lib.ptr(c) for c in cols),
                                 ctypes.byref(n_out), ctypes.byref(bad))
    if rc == _lib.EMU_ERR_UNSUPPORTED:
        recs = [parse_trace_line(s) for s in (ln.strip() for ln in raw.decode("utf-8").splitlines()) if s]
        return records_to_arrays_with_step(recs)
    _lib.check(rc, invalid_exc=PackFormatError)
    return cols


def records_to_arrays_with_step(recs: Sequence[StepTraceRecord]):
    n = len(recs)
    return (np.fromiter((r.step_index for r in recs), np.int64, n),
            np.fromiter((r.total_tokens for r in recs), np.int64, n).astype(np.int32),
            np.fromiter((r.concurrency for r in recs), np.int64, n).astype(np.int32),
            np.fromiter((phase_code(r.phase) for r in recs), np.uint8, n),
            np.fromiter((r.latency_s for r in recs), np.float64, n))


def read_trace_arrays(path: str | Path, threads: int = 0):
    """read_trace_file's records as columns (native parse of the whole file)."""
    return parse_trace_arrays(Path(path).read_bytes(), threads)


def build_pack_from_traces(paths, num_gpu_blocks: int, metadata: dict[str, str] | None = None, *,
                           canonical: bool = True) -> ProfilePack:
    """Trace JSONL files -> GPU-built pack: the native ingest feeding
    emu_tables_build (cli.py:202-208 reads the files with read_trace_file and
    calls build_pack).  Records are concatenated in the given path order."""
    parts = [read_trace_arrays(p) for p in paths]
    step, tt, conc, ph, lat = (np.concatenate([c[i] for c in parts]) if parts else np.zeros(0)
                               for i in range(5))
    return build_pack_arrays(tt, conc, ph, lat, num_gpu_blocks, metadata, step=step, canonical=canonical)
