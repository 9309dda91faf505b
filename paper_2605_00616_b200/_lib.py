"""ctypes binding of libemu_b200.so (the C ABI declared in include/emu_abi.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises.  Status codes map to the reference's
exception types (include/emu_abi.h header comment).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EMU_LIB_PATH") or os.path.join(_PKG, "libemu_b200.so")
CSRC = os.path.join(_PKG, "csrc")

EMU_OK, EMU_ERR_NO_DATA, EMU_ERR_INVALID, EMU_ERR_CUDA, EMU_ERR_CAPACITY, EMU_ERR_UNSUPPORTED = 0, 1, 2, 3, 4, 5
EMU_RNG_EXPLICIT, EMU_RNG_PHILOX = 0, 1

c_int, c_i32, c_i64, c_u64, c_dbl, c_vp = (ctypes.c_int, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                           ctypes.c_double, ctypes.c_void_p)


class TableView(ctypes.Structure):
    _fields_ = [("n_buckets", c_i64), ("n_samples", c_i64), ("bkt_tt", c_vp), ("bkt_conc", c_vp),
                ("bkt_off", c_vp), ("samples", c_vp)]


class TableInfo(ctypes.Structure):
    _fields_ = [("n_buckets", c_i64), ("n_samples", c_i64), ("tt_lo", c_i32), ("tt_hi", c_i32),
                ("conc_lo", c_i32), ("conc_hi", c_i32)]


class TableDev(ctypes.Structure):
    _fields_ = [("n_buckets", c_i64), ("n_samples", c_i64), ("n_rows", c_i64), ("bkt_tt", c_vp),
                ("bkt_conc", c_vp), ("bkt_off", c_vp), ("samples", c_vp), ("row_tt", c_vp),
                ("row_start", c_vp)]


# name -> (restype, argtypes); every symbol of include/emu_abi.h
SIGNATURES = {
    "emu_tables_create": (c_int, [ctypes.POINTER(TableView)] * 3 + [c_vp, ctypes.POINTER(c_vp)]),
    "emu_tables_build": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_vp, ctypes.POINTER(c_vp),
                                 ctypes.POINTER(c_i64), ctypes.POINTER(c_i32)]),
    "emu_tables_info": (c_int, [c_vp, c_int, ctypes.POINTER(TableInfo)]),
    "emu_tables_device": (c_int, [c_vp, c_int, ctypes.POINTER(TableDev)]),
    "emu_tables_destroy": (None, [c_vp]),
    "emu_oracle_create": (c_int, [c_vp, c_i32, c_dbl, c_dbl, c_i32, c_i32, c_i64, c_i64, c_vp,
                                  ctypes.POINTER(c_vp)]),
    "emu_oracle_destroy": (None, [c_vp]),
    "emu_oracle_flush": (c_int, [c_vp, c_vp]),
    "emu_oracle_pool": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp,
                                c_vp]),
    "emu_oracle_sample": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_vp, c_u64, c_u64, c_vp,
                                  c_vp, c_vp]),
    "emu_oracle_sample_pcg64": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "emu_oracle_sample_host": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_vp, c_u64, c_u64,
                                       c_vp, c_vp, c_vp]),
    "emu_oracle_seed_pcg64": (c_int, [c_vp, c_vp]),
    "emu_oracle_get_pcg64": (c_int, [c_vp, c_vp]),
    "emu_oracle_step": (c_int, [c_vp, c_i32, c_i32, c_i32, ctypes.POINTER(c_dbl)]),
    "emu_oracle_park": (c_int, [c_vp]),
    "emu_oracle_stats": (c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "emu_distance": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "emu_token_fill": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "emu_ground_truth": (c_int, [c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_u64, c_vp, c_vp]),
    "emu_gen_step_keys": (c_int, [c_i64, c_u64, c_dbl, c_dbl, c_i32, c_dbl, c_dbl, c_dbl, c_i32, c_vp, c_vp, c_vp,
                                  c_vp]),
    "emu_oracle_prefetch": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "emu_sched_create": (c_int, [c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i64,
                                 ctypes.POINTER(c_vp)]),
    "emu_sched_run_replay": (c_int, [c_vp, c_vp, c_vp]),
    "emu_sched_run_ground_truth": (c_int, [c_vp, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_u64, c_vp]),
    "emu_sched_run_oracle": (c_int, [c_vp, c_vp, c_vp, ctypes.POINTER(c_i64), c_vp]),
    "emu_sched_results": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "emu_sched_summary": (c_int, [c_vp, c_vp]),
    "emu_sched_keep_steps": (c_int, [c_vp, c_i32]),
    "emu_sched_destroy": (None, [c_vp]),
    "emu_pack_parse_json": (c_int, [c_vp, c_i64, ctypes.POINTER(c_vp)]),
    "emu_pack_parsed_info": (c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64), c_vp,
                                     ctypes.POINTER(c_i64)]),
    "emu_pack_parsed_copy": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp, c_vp]),
    "emu_pack_parsed_metadata": (c_int, [c_vp, c_vp, c_i64]),
    "emu_pack_parsed_free": (None, [c_vp]),
    "emu_trace_count_lines": (c_i64, [c_vp, c_i64]),
    "emu_trace_parse_jsonl": (c_int, [c_vp, c_i64, c_int, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                      ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "emu_launch_count": (c_i64, []),
    "emu_profile_enable": (c_int, [c_int]),
    "emu_profile_read": (c_int, [ctypes.c_char_p, ctypes.POINTER(c_dbl), ctypes.POINTER(c_i64)]),
    "emu_profile_names": (c_int, [ctypes.c_char_p, c_i64]),
    "emu_build_scratch_release": (c_int, []),
    "emu_last_error": (ctypes.c_char_p, []),
    "emu_version": (c_int, []),
}

_lib = None


class EmuError(RuntimeError):
    """CUDA-side failure of the B200 oracle library."""


class CapacityError(EmuError):
    pass


def build(force: bool = False) -> str:
    """Compile libemu_b200.so for sm_100a (make in csrc/)."""
    args = ["make", "-s", "-C", CSRC]
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(args, check=True)
    return LIB_PATH


def load_library() -> ctypes.CDLL:
    """Load (not build) the in-tree library and declare every signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EmuError(
            f"{LIB_PATH} is missing: build it with `make -C {CSRC}` or __graft_entry__.build(); "
            "there is no CPU fallback"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    return load_library()


def last_error() -> str:
    msg = lib().emu_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, no_data_exc=None, invalid_exc=ValueError) -> None:
    """Raise the reference-shaped exception for a nonzero status."""
    if rc == EMU_OK:
        return
    msg = last_error()
    if rc == EMU_ERR_NO_DATA:
        if no_data_exc is None:
            from .oracle import NoProfileDataError as no_data_exc  # noqa: N813
        raise no_data_exc(msg)
    if rc == EMU_ERR_INVALID:
        raise invalid_exc(msg)
    if rc == EMU_ERR_CAPACITY:
        raise CapacityError(msg)
    raise EmuError(msg or f"libemu_b200 status {rc}")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise EmuError("the B200 oracle needs a CUDA device (no CPU fallback)")
    load_library()
    return torch


def stream_ptr(torch_mod=None):
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    """Raw pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return ctypes.c_void_p(0)
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(t.ctypes.data)


def launch_count() -> int:
    """Kernels launched by libemu_b200 in this process."""
    return int(lib().emu_launch_count())


def profile_enable(on: bool = True) -> None:
    check(lib().emu_profile_enable(1 if on else 0))


def profile_read(kernel: str) -> tuple[float, int]:
    """(total ms, launches) of `kernel` since the last read (CUDA events on the launch stream)."""
    ms, n = ctypes.c_double(), ctypes.c_int64()
    check(lib().emu_profile_read(kernel.encode(), ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


def profile_all() -> dict:
    """{kernel name: (total ms, launches)} for every kernel recorded since the last read."""
    buf = ctypes.create_string_buffer(1 << 16)
    check(lib().emu_profile_names(buf, len(buf)))
    return {k: profile_read(k) for k in buf.value.decode().split("\n") if k}
