"""Device-resident profile tables (owner of an ``emu_tables_t`` handle)."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .profile import PackValidationError, TableSoA, _CHECK_MESSAGES

_DT = {"i4": np.int32, "i8": np.int64, "f8": np.float64}


class _CudaArray:
    """Minimal __cuda_array_interface__ exporter so torch can alias library
    memory without a copy; keeps the owning handle alive."""

    def __init__(self, owner, ptr: int, n: int, typestr: str):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def _as_host_or_tensor(a, dtype):
    """numpy array (contiguous, dtype) or CUDA tensor (contiguous, dtype)."""
    if hasattr(a, "is_cuda"):
        import torch

        tdt = {np.int32: torch.int32, np.int64: torch.int64, np.uint8: torch.uint8, np.float64: torch.float64}[dtype]
        return a.to(dtype=tdt).contiguous()
    return np.ascontiguousarray(a, dtype=dtype)


class DeviceTables:
    """Three canonical tables (decode, mixed, combined) resident in HBM."""

    def __init__(self, handle: ctypes.c_void_p, host: list[TableSoA] | None = None):
        self._h = handle
        self._host = host

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.emu_tables_destroy(h)
            self._h = None

    # -- construction -----------------------------------------------------------
    @classmethod
    def from_soas(cls, soas: list[TableSoA]) -> "DeviceTables":
        _lib.require_cuda()
        views = []
        keep = []
        for s in soas:
            arrs = [np.ascontiguousarray(s.tt, np.int32), np.ascontiguousarray(s.conc, np.int32),
                    np.ascontiguousarray(s.off, np.int64), np.ascontiguousarray(s.samples, np.float64)]
            keep.append(arrs)
            views.append(_lib.TableView(len(arrs[0]), len(arrs[3]), *[a.ctypes.data for a in arrs]))
        h = ctypes.c_void_p()
        rc = _lib.lib().emu_tables_create(ctypes.byref(views[0]), ctypes.byref(views[1]), ctypes.byref(views[2]),
                                          _lib.stream_ptr(), ctypes.byref(h))
        _lib.check(rc, invalid_exc=PackValidationError)
        return cls(h, list(soas))

    @classmethod
    def from_device(cls, flat: list) -> "DeviceTables":
        """Tables from 12 device tensors [tt, conc, off, samples] x (decode, mixed, combined)."""
        _lib.require_cuda()
        views = []
        for i in range(3):
            tt, conc, off, smp = flat[4 * i:4 * i + 4]
            views.append(_lib.TableView(tt.numel(), smp.numel(), tt.data_ptr(), conc.data_ptr(), off.data_ptr(),
                                        smp.data_ptr()))
        h = ctypes.c_void_p()
        rc = _lib.lib().emu_tables_create(ctypes.byref(views[0]), ctypes.byref(views[1]), ctypes.byref(views[2]),
                                          _lib.stream_ptr(), ctypes.byref(h))
        _lib.check(rc, invalid_exc=PackValidationError)
        return cls(h, None)

    @classmethod
    def from_pack(cls, pack) -> "DeviceTables":
        """Tables of any pack (this package's or the reference's, by duck type)."""
        dev = getattr(pack, "_device", None)
        if isinstance(dev, DeviceTables):
            return dev
        soas = []
        for t in (pack.decode_table, pack.mixed_table, pack.combined_table):
            if hasattr(t, "soa"):
                soas.append(t.soa())
            else:
                soas.append(TableSoA.from_buckets(sorted(t.buckets, key=lambda b: (b.tt, b.conc)))
                            if t.buckets else TableSoA.empty())
        return cls.from_soas(soas)

    @classmethod
    def build(cls, tt, conc, phase, latency_s, *, step=None, canonical: bool = False) -> "DeviceTables":
        """emu_tables_build over columnar records (host arrays or CUDA tensors)."""
        _lib.require_cuda()
        tt_a = np.asarray(tt) if not hasattr(tt, "is_cuda") else tt
        if not hasattr(tt, "is_cuda"):
            t64 = np.asarray(tt, dtype=np.int64)
            c64 = np.asarray(conc, dtype=np.int64)
            if len(t64) and (t64.max() > 0x7FFFFFFF or c64.max() > 0x7FFFFFFF or t64.min() < -0x80000000
                             or c64.min() < -0x80000000):
                raise PackValidationError("total_tokens/concurrency must fit in int32")
        arrs = [_as_host_or_tensor(tt, np.int32), _as_host_or_tensor(conc, np.int32),
                _as_host_or_tensor(phase, np.uint8), _as_host_or_tensor(latency_s, np.float64)]
        st = _as_host_or_tensor(step, np.int64) if step is not None else None
        n = len(arrs[0])
        if any(len(a) != n for a in arrs[1:]) or (st is not None and len(st) != n):
            raise ValueError("record columns must have equal length")
        h = ctypes.c_void_p()
        bad_i = ctypes.c_int64(-1)
        bad_c = ctypes.c_int32(0)
        rc = _lib.lib().emu_tables_build(*[_lib.ptr(a) for a in arrs], _lib.ptr(st), n, 1 if canonical else 0,
                                         _lib.stream_ptr(), ctypes.byref(h), ctypes.byref(bad_i),
                                         ctypes.byref(bad_c))
        if rc == _lib.EMU_ERR_INVALID and bad_i.value >= 0:
            i = bad_i.value

            def at(a):
                return None if a is None else (a[i].item() if hasattr(a[i], "item") else a[i])

            msg = _CHECK_MESSAGES[bad_c.value](at(st), int(at(arrs[0])), int(at(arrs[1])), int(at(arrs[2])),
                                              float(at(arrs[3])))
            raise PackValidationError(f"trace record {i}: {msg}")
        _lib.check(rc, invalid_exc=PackValidationError)
        del tt_a
        return cls(h, None)

    # -- views ------------------------------------------------------------------
    def info(self, table_id: int) -> dict:
        inf = _lib.TableInfo()
        _lib.check(_lib.lib().emu_tables_info(self._h, table_id, ctypes.byref(inf)))
        empty = inf.n_buckets == 0
        return {"n_buckets": inf.n_buckets, "n_samples": inf.n_samples,
                "tt_range": None if empty else (inf.tt_lo, inf.tt_hi),
                "conc_range": None if empty else (inf.conc_lo, inf.conc_hi)}

    def device_arrays(self, table_id: int) -> dict:
        """Zero-copy torch views of the handle-owned device arrays."""
        import torch

        d = _lib.TableDev()
        _lib.check(_lib.lib().emu_tables_device(self._h, table_id, ctypes.byref(d)))
        spec = {"bkt_tt": (d.bkt_tt, d.n_buckets, "<i4"), "bkt_conc": (d.bkt_conc, d.n_buckets, "<i4"),
                "bkt_off": (d.bkt_off, d.n_buckets + 1, "<i8"), "samples": (d.samples, d.n_samples, "<f8"),
                "row_tt": (d.row_tt, d.n_rows, "<i4"), "row_start": (d.row_start, d.n_rows + 1, "<i8")}
        out = {}
        for k, (p, n, ts) in spec.items():
            if n == 0:
                out[k] = torch.zeros(0, dtype={"<i4": torch.int32, "<i8": torch.int64, "<f8": torch.float64}[ts],
                                     device="cuda")
            else:
                out[k] = torch.as_tensor(_CudaArray(self, p, n, ts), device="cuda")
        return out

    def to_host(self) -> list[TableSoA]:
        if self._host is None:
            import torch

            torch.cuda.current_stream().synchronize()
            host = []
            for i in range(3):
                a = self.device_arrays(i)
                host.append(TableSoA(a["bkt_tt"].cpu().numpy().copy(), a["bkt_conc"].cpu().numpy().copy(),
                                     a["bkt_off"].cpu().numpy().copy(), a["samples"].cpu().numpy().copy()))
            self._host = host
        return self._host
