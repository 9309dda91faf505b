"""B200-native density-aware profile oracle (the hot path of LLM-Emu, arXiv 2605.00616).

Drop-in for the oracle/profile surface of the reference ``serve_emu`` package
(/root/reference/pkg/src/serve_emu/__init__.py:24-34): same names, argument
meaning and exceptions, with every neighbour search, Shepard CDF, draw, token
fill and table build executed by hand-written sm_100a CUDA in
``libemu_b200.so`` (C ABI: include/emu_abi.h).  No CPU fallback.
"""
from .oracle import (
    LatencyOracle,
    NoProfileDataError,
    OracleConfig,
    OracleQuery,
    normalized_distance,
    pool_neighbors,
    sample_latency,
)
from .profile import (
    Bucket,
    PackFormatError,
    PackValidationError,
    PackVersionError,
    PhaseTable,
    ProfilePack,
    StepPhase,
    StepTraceRecord,
    TableKind,
    build_pack,
    build_pack_arrays,
    build_pack_from_traces,
    iter_trace_dir,
    load_pack,
    load_pack_file,
    parse_trace_arrays,
    parse_trace_line,
    read_trace_arrays,
    read_trace_file,
    save_pack,
    save_pack_file,
    trace_record_to_line,
)
from .tokens import token_fill

__all__ = [
    "Bucket",
    "LatencyOracle",
    "NoProfileDataError",
    "OracleConfig",
    "OracleQuery",
    "PackFormatError",
    "PackValidationError",
    "PackVersionError",
    "PhaseTable",
    "ProfilePack",
    "StepPhase",
    "StepTraceRecord",
    "TableKind",
    "build_pack",
    "build_pack_arrays",
    "build_pack_from_traces",
    "iter_trace_dir",
    "load_pack",
    "load_pack_file",
    "normalized_distance",
    "parse_trace_arrays",
    "parse_trace_line",
    "pool_neighbors",
    "read_trace_arrays",
    "read_trace_file",
    "sample_latency",
    "save_pack",
    "save_pack_file",
    "token_fill",
    "trace_record_to_line",
]
