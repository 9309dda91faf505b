"""Golden inputs for the native codecs, written by the UNMODIFIED reference.

    python tests/golden/make_codec_golden.py      (dev container: imports /root/reference/pkg/src)

Writes
  codec_pack.json    save_pack(build_pack(records)) bytes of the reference
                     (profile.py:230-296), 3,000 synthetic records of generator G
                     plus a few hand-made edge buckets (tiny / huge / subnormal
                     latencies, repeated values, int32 extremes of the keys);
  codec_trace.jsonl  trace_record_to_line of 2,000 records (profile.py:350-362);
  codec_expect.json  what the reference's load_pack / read_trace_file return for
                     them: per-table bucket keys, offsets and the samples' exact
                     bit patterns (hex), trace columns (latency bits as hex).
Tests load only these files (no /root/reference on the GPU box).
"""
from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from serve_emu import profile as P  # noqa: E402  (reference)

from paper_2605_00616_b200.workloads import records_llama  # noqa: E402  (synthetic record columns)


def hexd(x: float) -> str:
    return struct.pack("<d", x).hex()


def main():
    tt, conc, ph, lat = records_llama(3_000, 11)
    recs = [P.StepTraceRecord(i, int(t), int(c), P.StepPhase.DECODE_ONLY if p == 0 else P.StepPhase.PREFILL_OR_MIXED,
                              float(l)) for i, (t, c, p, l) in enumerate(zip(tt, conc, ph, lat))]
    edge = [(5, 5, 0, 5e-324), (5, 5, 0, 1e-300), (5, 5, 0, 1e300), (7, 3, 1, 0.1), (7, 3, 1, 0.1),
            (2147483647, 1, 1, 3.0), (2147483647, 2147483647, 0, 2.5), (1, 1, 0, 1.0000000000000002)]
    for i, (t, c, p, l) in enumerate(edge):
        recs.append(P.StepTraceRecord(len(recs), t, c, P.StepPhase.DECODE_ONLY if p == 0 else
                                      P.StepPhase.PREFILL_OR_MIXED, l))
    pack = P.build_pack(recs, 1234, {"model": "llama-3-8b-synthetic", "gpu": "B200", "note": "é utf-8"})
    data = P.save_pack(pack)
    with open(os.path.join(HERE, "codec_pack.json"), "wb") as f:
        f.write(data)
    back = P.load_pack(data)
    tables = {}
    for name, t in (("decode", back.decode_table), ("mixed", back.mixed_table), ("combined", back.combined_table)):
        bl = t.buckets
        off = np.zeros(len(bl) + 1, np.int64)
        off[1:] = np.cumsum([len(b.samples) for b in bl])
        tables[name] = {"tt": [b.tt for b in bl], "conc": [b.conc for b in bl], "off": off.tolist(),
                        "samples_hex": "".join(hexd(s) for b in bl for s in b.samples),
                        "tt_range": list(t.tt_range) if t.tt_range else None,
                        "conc_range": list(t.conc_range) if t.conc_range else None}
    trace = recs[:2000]
    lines = [P.trace_record_to_line(r) for r in trace]
    with open(os.path.join(HERE, "codec_trace.jsonl"), "w") as f:
        f.write("\n".join(lines) + "\n")
    rt = P.read_trace_file(os.path.join(HERE, "codec_trace.jsonl"))
    expect = {
        "pack": {"num_gpu_blocks": back.num_gpu_blocks, "schema_version": back.schema_version,
                 "metadata": back.metadata, "tables": tables},
        "trace": {"step": [r.step_index for r in rt], "tt": [r.total_tokens for r in rt],
                  "conc": [r.concurrency for r in rt], "phase": [r.phase.value for r in rt],
                  "latency_hex": "".join(hexd(r.latency_s) for r in rt)},
    }
    with open(os.path.join(HERE, "codec_expect.json"), "w") as f:
        json.dump(expect, f)
    print("pack bytes", len(data), "trace lines", len(lines))


if __name__ == "__main__":
    main()
