"""Latency oracle on the B200: density-aware neighbour pooling + Shepard draws.

Drop-in mirror of ``serve_emu.oracle`` (/root/reference/pkg/src/serve_emu/
oracle.py).  ``LatencyOracle(pack, cfg)`` is the engine backend
(``Callable[[int, int, StepPhase], float]``, engine.py:283-290, :555-557) and
returns bit-identical latencies to the reference for the same pack and seed:
the device replays numpy's PCG64 stream, ``Generator.choice``'s inverse CDF
and ``Generator.integers``' Lemire draw exactly.

All computation -- neighbour search, Shepard weights, CDFs, draws -- runs in
``libemu_b200.so`` on the GPU; this module only validates arguments, moves
buffers and maps status codes to the reference's exceptions.  Beyond the
reference surface it adds ``sample_batch`` (millions of independent draws per
call for trace replay / what-if sweeps) and ``pools`` (explicit pool CSR).
"""
from __future__ import annotations

import collections
import ctypes
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import DeviceTables
from .profile import Bucket, PhaseTable, ProfilePack, StepPhase, TableSoA, phase_code

_I32_MIN, _I32_MAX = -(1 << 31), (1 << 31) - 1


class NoProfileDataError(RuntimeError):
    """Raised when the queried table (and any fallback) holds no samples."""


@dataclass(frozen=True)
class OracleQuery:
    total_tokens: int
    concurrency: int
    phase: StepPhase

    def validate(self) -> None:
        if self.total_tokens < 1 or self.concurrency < 1:
            raise ValueError(f"query ({self.total_tokens}, {self.concurrency}) must be positive")


@dataclass
class OracleConfig:
    """Sampling knobs (oracle.py:38-59): floor M, Shepard power p, distance clamp eps."""

    reliability_floor: int = 32
    shepard_power: float = 2.0
    epsilon_distance: float = 1e-9
    rng_seed: int = 0

    def validate(self) -> None:
        if self.reliability_floor < 1:
            raise ValueError(f"reliability_floor must be >= 1, got {self.reliability_floor}")
        if not self.shepard_power > 0:
            raise ValueError(f"shepard_power must be > 0, got {self.shepard_power}")
        if not self.epsilon_distance > 0:
            raise ValueError(f"epsilon_distance must be > 0, got {self.epsilon_distance}")


def _check(rc: int) -> None:
    _lib.check(rc, no_data_exc=NoProfileDataError)


_PHASE_MEMO: dict = {}  # phase object -> code, for the per-step call


def _i32(v: int, what: str) -> int:
    v = int(v)
    if not _I32_MIN < v <= _I32_MAX:
        raise ValueError(f"{what}={v} is outside the int32 range the B200 oracle supports")
    return v


def pcg64_state6(bitgen_state: dict) -> np.ndarray:
    """numpy PCG64 state dict -> 6 x u64 {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger}."""
    if bitgen_state.get("bit_generator") != "PCG64":
        raise TypeError(f"the B200 oracle replays PCG64 streams, got {bitgen_state.get('bit_generator')}")
    s, inc = bitgen_state["state"]["state"], bitgen_state["state"]["inc"]
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m, bitgen_state["has_uint32"], bitgen_state["uinteger"]],
                    dtype=np.uint64)


def state6_to_dict(st: np.ndarray) -> dict:
    v = [int(x) for x in st]
    return {"bit_generator": "PCG64", "state": {"state": (v[0] << 64) | v[1], "inc": (v[2] << 64) | v[3]},
            "has_uint32": v[4], "uinteger": v[5]}


# ---------------------------------------------------------------------------
# Scalar helpers (reference surface)
# ---------------------------------------------------------------------------


def normalized_distance(query: tuple[int, int], bucket: tuple[int, int], tt_range: tuple[int, int],
                        conc_range: tuple[int, int]) -> float:
    """Range-normalised Euclidean distance (oracle.py:62-77), computed by the
    same device routine the neighbour search uses (emu_distance)."""
    torch = _lib.require_cuda()
    a = torch.tensor([_i32(query[0], "tt"), _i32(query[1], "conc"), _i32(bucket[0], "tt"),
                      _i32(bucket[1], "conc")], dtype=torch.int32, device="cuda")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _check(_lib.lib().emu_distance(_lib.ptr(a[0:1]), _lib.ptr(a[1:2]), _lib.ptr(a[2:3]), _lib.ptr(a[3:4]), 1,
                                   _i32(tt_range[0], "tt"), _i32(tt_range[1], "tt"), _i32(conc_range[0], "conc"),
                                   _i32(conc_range[1], "conc"), _lib.ptr(out), _lib.stream_ptr()))
    return float(out.item())


# Device tables + oracle handles for packs/tables used through the functional
# API, keyed by object identity (the reference's pack/table classes define
# __eq__ and are unhashable) and invalidated if the content size changes.
# Bounded (least recently used first out): an entry made by sample_latency
# holds its pack, so the weakref alone would never release it.
_tables_cache: "collections.OrderedDict[int, tuple]" = collections.OrderedDict()
_TABLES_CACHE_MAX = 16


def _nbuckets(t) -> int:
    b = getattr(t, "_buckets", None)
    if b is None and getattr(t, "_soa", None) is not None:
        return len(t._soa.tt)
    return len(t.buckets)


def _fingerprint(tables) -> tuple:
    return tuple((_nbuckets(t), t.total_samples) for t in tables)


def _single_table_pack(table) -> ProfilePack:
    """A pack whose decode (and combined) table is `table`: lets the oracle
    kernels run pool_neighbors on an arbitrary PhaseTable."""
    soa = table.soa() if hasattr(table, "soa") else (
        TableSoA.from_buckets(sorted(table.buckets, key=lambda b: (b.tt, b.conc))) if table.buckets
        else TableSoA.empty())
    from .profile import TableKind

    return ProfilePack(1, PhaseTable.from_soa(TableKind.DECODE, soa), PhaseTable.from_soa(TableKind.MIXED,
                                                                                           TableSoA.empty()),
                       PhaseTable.from_soa(TableKind.COMBINED, soa))


def _cached_oracle(obj, tables, make_pack, floor: int, p: float, eps: float) -> "LatencyOracle":
    fp = _fingerprint(tables)
    key = id(obj)
    entry = _tables_cache.get(key)
    if entry is None or entry[0]() is not obj or entry[1] != fp:
        ref = weakref.ref(obj, lambda _r, k=key: _tables_cache.pop(k, None))
        entry = (ref, fp, make_pack(), {})
        _tables_cache[key] = entry
        while len(_tables_cache) > _TABLES_CACHE_MAX:
            _tables_cache.popitem(last=False)
    _tables_cache.move_to_end(key)
    oracles = entry[3]
    okey = (floor, p, eps)
    if okey not in oracles:
        oracles[okey] = LatencyOracle(entry[2], OracleConfig(floor, p, eps, 0), _validate=False)
    return oracles[okey]


def pool_neighbors(table: PhaseTable, query: tuple[int, int], floor: int) -> list[tuple[Bucket, float]]:
    """Shortest distance-sorted bucket prefix whose cumulative sample count
    reaches `floor` (oracle.py:108-121), ties by ascending (tt, conc)."""
    if table.is_empty:
        raise NoProfileDataError(f"{table.kind.value} table has no data")
    if floor < 1:
        raise ValueError(f"floor must be >= 1, got {floor}")
    orc = _cached_oracle(table, [table], lambda: _single_table_pack(table), int(floor), 2.0, 1e-9)
    off, bkt, dist, _prob, _cdf, _tid = orc.pools([query[0]], [query[1]], [0])
    ordered = table.buckets
    if [(b.tt, b.conc) for b in ordered] != sorted((b.tt, b.conc) for b in ordered):
        ordered = sorted(ordered, key=lambda b: (b.tt, b.conc))
    return [(ordered[int(b)], float(d)) for b, d in zip(bkt, dist)]


def sample_latency(pack: ProfilePack, query: OracleQuery, cfg: OracleConfig, rng: np.random.Generator) -> float:
    """One draw for `query` (oracle.py:147-165), consuming `rng` exactly like
    the reference: the Generator's PCG64 state is replayed on the device and
    written back."""
    query.validate()
    cfg.validate()
    table = pack.decode_table if phase_code(query.phase) == 0 else pack.mixed_table
    if table.is_empty:
        table = pack.combined_table
    if table.is_empty:
        raise NoProfileDataError("profile pack has no samples in any table")
    tables = (pack.decode_table, pack.mixed_table, pack.combined_table)
    orc = _cached_oracle(pack, tables, lambda: pack, int(cfg.reliability_floor), float(cfg.shepard_power),
                         float(cfg.epsilon_distance))
    orc.set_rng_state(rng.bit_generator.state)
    value = orc.sample(query.total_tokens, query.concurrency, query.phase)
    rng.bit_generator.state = orc.rng_state()
    return value


# ---------------------------------------------------------------------------
# The engine-facing oracle
# ---------------------------------------------------------------------------

def _words(t, dtypes, name):
    """Uniform words are passed by bit pattern: accept signed or unsigned CUDA tensors."""
    if t is None:
        return None
    if not (hasattr(t, "is_cuda") and t.is_cuda and t.dtype in dtypes):
        raise TypeError(f"{name} must be a CUDA tensor of dtype {dtypes}")
    return t.contiguous()


_RNG_MODES = {"explicit": _lib.EMU_RNG_EXPLICIT, "philox": _lib.EMU_RNG_PHILOX}


class LatencyOracle:
    """Engine-facing sampler over a pack, with a device-side pool cache.

    Stateless apart from its rng (numpy PCG64 seeded with cfg.rng_seed, held
    on the device); share one instance per sampling stream (oracle.py:181-185).
    """

    def __init__(self, pack: ProfilePack, cfg: OracleConfig | None = None, *, arena_slots: int = 0,
                 hash_slots: int = 0, dom_tt: int = 0, dom_conc: int = 0, _validate: bool = True):
        self.cfg = cfg or OracleConfig()
        self.cfg.validate()
        if _validate:
            pack.validate()
        self._pack = pack
        self.tables = DeviceTables.from_pack(pack)
        host = self.tables._host
        self._plane_table = [0 if not self._table_empty(0) else 2, 1 if not self._table_empty(1) else 2]
        h = ctypes.c_void_p()
        _check(_lib.lib().emu_oracle_create(self.tables.handle, int(self.cfg.reliability_floor),
                                            float(self.cfg.shepard_power), float(self.cfg.epsilon_distance),
                                            int(dom_tt), int(dom_conc), int(arena_slots), int(hash_slots),
                                            _lib.stream_ptr(), ctypes.byref(h)))
        self._h = h
        self._host = host
        self._step = _lib.lib().emu_oracle_step  # per-step hot path: no per-call lookups
        self._step_out = ctypes.c_double()
        self._step_out_ref = ctypes.byref(self._step_out)
        self.set_rng_state(np.random.default_rng(self.cfg.rng_seed).bit_generator.state)

    def _table_empty(self, i: int) -> bool:
        return self.tables.info(i)["n_buckets"] == 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.emu_oracle_destroy(h)
            self._h = None

    # -- rng ----------------------------------------------------------------------
    def rng_state(self) -> dict:
        """numpy PCG64 state dict of the device-held stream."""
        st = np.zeros(6, dtype=np.uint64)
        _check(_lib.lib().emu_oracle_get_pcg64(self._h, _lib.ptr(st)))
        return state6_to_dict(st)

    def set_rng_state(self, state: dict) -> None:
        st = pcg64_state6(state)
        _check(_lib.lib().emu_oracle_seed_pcg64(self._h, _lib.ptr(st)))

    @property
    def _rng(self) -> np.random.Generator:
        """A numpy Generator positioned where the device stream is (a copy)."""
        g = np.random.Generator(np.random.PCG64())
        g.bit_generator.state = self.rng_state()
        return g

    # -- reference surface ------------------------------------------------------------
    def sample(self, tt: int, conc: int, phase) -> float:
        """One draw on this oracle's stream (oracle.py:224-226)."""
        ph = _PHASE_MEMO.get(phase) if phase.__hash__ is not None else None
        if ph is None:
            ph = phase_code(phase)
            if phase.__hash__ is not None and len(_PHASE_MEMO) < 64:
                _PHASE_MEMO[phase] = ph
        if not (type(tt) is int and type(conc) is int and _I32_MIN < tt <= _I32_MAX and _I32_MIN < conc <= _I32_MAX):
            tt, conc = _i32(tt, "tt"), _i32(conc, "conc")
        rc = self._step(self._h, tt, conc, ph, self._step_out_ref)
        if rc:
            _check(rc)
        return self._step_out.value

    __call__ = sample

    def _pooled(self, phase, tt: int, conc: int) -> tuple[np.ndarray, list[np.ndarray]]:
        """(probs, [sample arrays]) of the pool for (phase, tt, conc) (oracle.py:200-222)."""
        ph = phase_code(phase)
        off, bkt, _dist, prob, _cdf, tid = self.pools([tt], [conc], [ph])
        soa = self._host_table(int(tid[0]))
        return prob.copy(), [soa.samples[soa.off[b]:soa.off[b + 1]] for b in bkt]

    def _host_table(self, i: int) -> TableSoA:
        return self.tables.to_host()[i]

    # -- batched surface -------------------------------------------------------------------
    def pools(self, tt, conc, phase):
        """Explicit pools of U keys: (pool_off[U+1], bucket, dist, prob, cdf, table_id[U]) numpy arrays.
        Bucket indices refer to table `table_id` in (tt, conc) order."""
        torch = _lib.require_cuda()
        kt = torch.as_tensor(np.asarray(tt, dtype=np.int64).astype(np.int32), device="cuda")
        kc = torch.as_tensor(np.asarray(conc, dtype=np.int64).astype(np.int32), device="cuda")
        kp = torch.as_tensor(np.asarray([phase_code(p) for p in np.atleast_1d(np.asarray(phase, dtype=object))],
                                        dtype=np.uint8), device="cuda")
        U = kt.numel()
        off = torch.zeros(U + 1, dtype=torch.int64, device="cuda")
        tid = torch.zeros(max(U, 1), dtype=torch.int32, device="cuda")
        cap = max(1, U * min(int(self.cfg.reliability_floor), 64))
        for _ in range(2):
            bkt = torch.empty(cap, dtype=torch.int32, device="cuda")
            dist = torch.empty(cap, dtype=torch.float64, device="cuda")
            prob = torch.empty(cap, dtype=torch.float64, device="cuda")
            cdf = torch.empty(cap, dtype=torch.float64, device="cuda")
            rc = _lib.lib().emu_oracle_pool(self._h, _lib.ptr(kt), _lib.ptr(kc), _lib.ptr(kp), U, _lib.ptr(off),
                                            _lib.ptr(bkt), _lib.ptr(dist), _lib.ptr(prob), _lib.ptr(cdf), cap,
                                            _lib.ptr(tid), _lib.stream_ptr())
            if rc == _lib.EMU_ERR_CAPACITY:
                cap = int(off[-1].item())
                continue
            _check(rc)
            break
        n = int(off[-1].item())
        return (off.cpu().numpy(), bkt[:n].cpu().numpy(), dist[:n].cpu().numpy(), prob[:n].cpu().numpy(),
                cdf[:n].cpu().numpy(), tid[:U].cpu().numpy())

    def sample_batch(self, tt, conc, phase, *, rng: str = "philox", u_sel=None, u_idx=None, seed: int | None = None,
                     ctr_base: int = 0, out_lat=None, out_sidx=None):
        """Q independent draws.

        rng="philox"  : on-device Philox4x32-10 keyed by (seed, ctr_base + i);
        rng="explicit": caller-supplied words u_sel (u64) and u_idx (u32) per query
                        (u = (u_sel >> 11) * 2^-53; Lemire on u_idx, continuation
                        words hash32(prev));
        rng="pcg64"   : continues this oracle's numpy PCG64 stream -- identical to
                        calling sample() Q times in order.
        Inputs may be CUDA tensors (results stay on the device: (lat f64, sidx i32)
        tensors) or host arrays (results come back as numpy arrays; copies are
        pipelined with the device work; out_sidx=False skips the index copy-out and
        returns sidx=None).  sidx indexes the samples of the table each query resolved to.
        """
        torch = _lib.require_cuda()
        on_dev = hasattr(tt, "is_cuda") and tt.is_cuda
        seed = self.cfg.rng_seed if seed is None else int(seed)
        if rng == "pcg64":
            return self._sample_pcg64_batch(tt, conc, phase, on_dev)
        if rng not in _RNG_MODES:
            raise ValueError(f"unknown rng mode {rng!r}")
        mode = _RNG_MODES[rng]
        if mode == _lib.EMU_RNG_EXPLICIT and (u_sel is None or u_idx is None):
            raise ValueError("rng='explicit' needs u_sel and u_idx")
        if on_dev:
            qt = tt.to(torch.int32).contiguous()
            qc = conc.to(torch.int32).contiguous()
            qp = phase.to(torch.uint8).contiguous()
            Q = qt.numel()
            us = _words(u_sel, (torch.int64, torch.uint64), "u_sel")
            ui = _words(u_idx, (torch.int32, torch.uint32), "u_idx")
            lat = out_lat if out_lat is not None else torch.empty(Q, dtype=torch.float64, device=qt.device)
            sidx = out_sidx if out_sidx is not None else torch.empty(Q, dtype=torch.int32, device=qt.device)
            _check(_lib.lib().emu_oracle_sample(self._h, _lib.ptr(qt), _lib.ptr(qc), _lib.ptr(qp), Q, mode,
                                                _lib.ptr(us), _lib.ptr(ui), seed & (2**64 - 1), int(ctr_base),
                                                _lib.ptr(lat), _lib.ptr(sidx), _lib.stream_ptr()))
            return lat, sidx
        qt = np.ascontiguousarray(tt, dtype=np.int32)
        qc = np.ascontiguousarray(conc, dtype=np.int32)
        qp = np.ascontiguousarray(phase, dtype=np.uint8)
        Q = len(qt)
        us = np.ascontiguousarray(u_sel, dtype=np.uint64) if u_sel is not None else None
        ui = np.ascontiguousarray(u_idx, dtype=np.uint32) if u_idx is not None else None
        lat = np.empty(Q, dtype=np.float64) if out_lat is None else out_lat
        if out_sidx is False:  # latencies only: no index copy-out
            sidx = None
        else:
            sidx = np.empty(Q, dtype=np.int32) if out_sidx is None else out_sidx
        _check(_lib.lib().emu_oracle_sample_host(self._h, _lib.ptr(qt), _lib.ptr(qc), _lib.ptr(qp), Q, mode,
                                                 _lib.ptr(us), _lib.ptr(ui), seed & (2**64 - 1), int(ctr_base),
                                                 _lib.ptr(lat), _lib.ptr(sidx), _lib.stream_ptr()))
        return lat, sidx

    def _sample_pcg64_batch(self, tt, conc, phase, on_dev: bool):
        torch = _lib.require_cuda()
        if on_dev:
            qt, qc, qp = tt.to(torch.int32).contiguous(), conc.to(torch.int32).contiguous(), \
                phase.to(torch.uint8).contiguous()
        else:
            qt = torch.as_tensor(np.ascontiguousarray(tt, dtype=np.int32), device="cuda")
            qc = torch.as_tensor(np.ascontiguousarray(conc, dtype=np.int32), device="cuda")
            qp = torch.as_tensor(np.ascontiguousarray(phase, dtype=np.uint8), device="cuda")
        Q = qt.numel()
        st_host = pcg64_state6(self.rng_state())
        st = torch.as_tensor(st_host.view(np.int64), device="cuda")
        lat = torch.empty(Q, dtype=torch.float64, device="cuda")
        sidx = torch.empty(Q, dtype=torch.int32, device="cuda")
        _check(_lib.lib().emu_oracle_sample_pcg64(self._h, _lib.ptr(qt), _lib.ptr(qc), _lib.ptr(qp), Q,
                                                  _lib.ptr(st), _lib.ptr(lat), _lib.ptr(sidx), _lib.stream_ptr()))
        self.set_rng_state(state6_to_dict(st.cpu().numpy().view(np.uint64)))
        if on_dev:
            return lat, sidx
        return lat.cpu().numpy(), sidx.cpu().numpy()

    def flush(self) -> None:
        """Drop every cached pool."""
        _check(_lib.lib().emu_oracle_flush(self._h, _lib.stream_ptr()))

    def park(self) -> None:
        """Stop the resident step server now (it otherwise stays up for
        EMU_STEP_SERVER_IDLE_US after the last step, so a device-wide
        synchronize would wait that long); the next step relaunches it."""
        _check(_lib.lib().emu_oracle_park(self._h))

    def cached_slots(self) -> int:
        n_pools, n_slots = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.lib().emu_oracle_stats(self._h, ctypes.byref(n_pools), ctypes.byref(n_slots)))
        return n_slots.value
