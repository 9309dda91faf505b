"""Generate golden vectors from the UNMODIFIED reference (run in the dev container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports serve_emu from /root/reference/pkg/src (read-only) and writes small
fixtures next to this file.  /root/reference does not exist on the GPU box:
tests load only the .npz/.json files written here.

Fixtures
  c1_trace.npz     10k step keys (tt, conc, phase) from the reference scheduler
                   (EmulatorEngine._schedule_step/_apply_outcome, engine.py:360-483)
                   driven in virtual time by generate_workload(.., seed=7) and
                   generate_arrivals(rate=8, burstiness=1, seed=42) (bench.py:77-116)
                   with a ground-truth backend for step times; plus the token ids
                   _apply_outcome emitted for the entries of the first steps.
  c1_golden.npz    on the C1 pack (generator G(0), 50k records, canonicalised with
                   load_pack(save_pack(.))): LatencyOracle(pack, OracleConfig(32,
                   rng_seed=0)).sample over the trace (latencies + final PCG64 state),
                   pools/probs of the first 600 unique keys, pack hashes.
  fixtures.json    reference test fixtures re-run: tie-break order, anchored Shepard
                   distances, acceptance-C1 random tables (pools + distances),
                   test_oracle brute-force tables, acceptance-C2/C3 draw summaries.
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import random
import sys
from collections import Counter

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from serve_emu.bench import WorkloadSpec, generate_arrivals, generate_workload  # noqa: E402
from serve_emu.engine import EmulatorEngine, EngineConfig, GroundTruthBackend, GroundTruthParams  # noqa: E402
from serve_emu.oracle import (  # noqa: E402
    LatencyOracle,
    OracleConfig,
    OracleQuery,
    pool_neighbors,
    sample_latency,
)
from serve_emu.profile import (  # noqa: E402
    Bucket,
    PhaseTable,
    ProfilePack,
    StepPhase,
    StepTraceRecord,
    TableKind,
    build_pack,
    load_pack,
    save_pack,
)

from paper_2605_00616_b200.workloads import records_llama  # noqa: E402  (numpy-only module)

DEC, MIX = StepPhase.DECODE_ONLY, StepPhase.PREFILL_OR_MIXED


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def records_hash(tt, conc, ph, lat) -> str:
    h = hashlib.sha256()
    for a in (tt, conc, ph, lat):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def c1_trace(n_steps=10_000, token_steps=400):
    """Virtual-time run of the reference scheduler; returns step keys and the
    token-fill inputs/outputs of the first `token_steps` steps."""
    cfg = EngineConfig(num_gpu_blocks=4096, block_size=16, max_model_len=4096, max_num_batched_tokens=512,
                       max_num_seqs=64)
    eng = EmulatorEngine(cfg, backend=lambda t, c, p: 0.01)
    gt = GroundTruthBackend(GroundTruthParams(noise_cv=0.05), seed=3)
    entries = generate_workload(4000, 200, 100, seed=7)
    arrivals = generate_arrivals(WorkloadSpec(entries=entries, request_rate=8.0, burstiness=1.0, seed=42))
    t, i, keys = 0.0, 0, []
    tok = {k: [] for k in ("is_prefill", "chunk", "progress", "prompt_len", "generated", "target", "ids", "fin")}
    while len(keys) < n_steps:
        while i < len(entries) and arrivals[i] <= t:
            p, o = entries[i]
            eng.admit(p, o)
            i += 1
        prep = eng._schedule_step()
        if prep is None:
            if i >= len(entries):
                break
            t = arrivals[i]
            continue
        lat = gt(prep.total_tokens, prep.concurrency, prep.phase)
        if len(keys) < token_steps:
            before = [(e.is_prefill, e.chunk, e.req.prefill_progress, e.req.prompt_len, e.req.generated,
                       e.req.target_output_len, e.req) for e in prep.entries]
        outcome = eng._apply_outcome(prep)
        if len(keys) < token_steps:
            emitted = {id(r): k for r, k in outcome.emissions}
            finished = {id(r) for r in outcome.finished}
            for pre, ch, pg, pl, gen, tg, req in before:
                tok["is_prefill"].append(int(pre))
                tok["chunk"].append(ch)
                tok["progress"].append(pg)
                tok["prompt_len"].append(pl)
                tok["generated"].append(gen)
                tok["target"].append(tg)
                tok["ids"].append(emitted.get(id(req), -1))
                tok["fin"].append(int(id(req) in finished))
        keys.append((prep.total_tokens, prep.concurrency, 0 if prep.phase is DEC else 1))
        t += lat
    k = np.array(keys, dtype=np.int64)
    return k, {name: np.array(v, dtype=np.int32) for name, v in tok.items()}


def c1_pack():
    tt, conc, ph, lat = records_llama(50_000, 0)
    recs = [StepTraceRecord(i, int(tt[i]), int(conc[i]), MIX if ph[i] else DEC, float(lat[i])) for i in range(len(tt))]
    raw = build_pack(recs, 1000)
    canon = load_pack(save_pack(raw))
    return (tt, conc, ph, lat), raw, canon


def table_digest(table) -> str:
    h = hashlib.sha256()
    for b in table.buckets:
        h.update(np.array([b.tt, b.conc, len(b.samples)], dtype=np.int64).tobytes())
        h.update(np.asarray(b.samples, dtype=np.float64).tobytes())
    return h.hexdigest()


def main():
    out = {}
    # ---------------------------------------------------------------- C1 trace
    keys, tok = c1_trace()
    np.savez_compressed(os.path.join(HERE, "c1_trace.npz"), tt=keys[:, 0].astype(np.int32),
                        conc=keys[:, 1].astype(np.int32), phase=keys[:, 2].astype(np.uint8),
                        **{"tok_" + k: v for k, v in tok.items()})
    print("trace steps", len(keys), "token entries", len(tok["ids"]))
    # ---------------------------------------------------------------- C1 pack
    (tt, conc, ph, lat), raw, canon = c1_pack()
    cfg = OracleConfig(reliability_floor=32, rng_seed=0)
    orc = LatencyOracle(canon, cfg)
    lat_seq = np.array([orc.sample(int(a), int(b), MIX if c else DEC) for a, b, c in keys], dtype=np.float64)
    st = orc._rng.bit_generator.state
    # pools of the first unique keys (in trace order)
    seen, uk = set(), []
    for a, b, c in keys:
        if (a, b, c) not in seen:
            seen.add((a, b, c))
            uk.append((a, b, c))
    n_unique = len(uk)
    uk = uk[:600]
    p_off, p_tt, p_conc, p_dist, p_prob = [0], [], [], [], []
    for a, b, c in uk:
        table = canon.mixed_table if c else canon.decode_table
        pooled = pool_neighbors(table, (int(a), int(b)), 32)
        probs, _ = orc._pooled(MIX if c else DEC, int(a), int(b))
        for (bk, d), pr in zip(pooled, probs):
            p_tt.append(bk.tt)
            p_conc.append(bk.conc)
            p_dist.append(d)
            p_prob.append(pr)
        p_off.append(len(p_tt))
    # second stream: a different seed / floor / power on mixed-only queries
    orc2 = LatencyOracle(canon, OracleConfig(reliability_floor=8, shepard_power=1.5, rng_seed=12345))
    lat2 = np.array([orc2.sample(int(a), int(b), MIX if c else DEC) for a, b, c in keys[:3000]], dtype=np.float64)
    np.savez_compressed(
        os.path.join(HERE, "c1_golden.npz"),
        lat_seq=lat_seq, lat_seq_m8_p15=lat2,
        final_state=np.array([st["state"]["state"] >> 64, st["state"]["state"] & (2**64 - 1),
                              st["state"]["inc"] >> 64, st["state"]["inc"] & (2**64 - 1), st["has_uint32"],
                              st["uinteger"]], dtype=np.uint64),
        uk=np.array(uk, dtype=np.int64), p_off=np.array(p_off, np.int64), p_tt=np.array(p_tt, np.int32),
        p_conc=np.array(p_conc, np.int32), p_dist=np.array(p_dist, np.float64), p_prob=np.array(p_prob, np.float64))
    out["c1"] = {
        "records_sha256": records_hash(tt, conc, ph, lat),
        "n_records": int(len(tt)),
        "n_unique_keys": n_unique,
        "canonical_pack_sha256": sha(save_pack(canon)),
        "buckets": [len(canon.decode_table.buckets), len(canon.mixed_table.buckets),
                    len(canon.combined_table.buckets)],
        "raw_table_digest": [table_digest(t) for t in (raw.decode_table, raw.mixed_table, raw.combined_table)],
        "canon_table_digest": [table_digest(t) for t in (canon.decode_table, canon.mixed_table,
                                                         canon.combined_table)],
    }
    # ------------------------------------------------------- test fixtures
    tie = PhaseTable.from_buckets(TableKind.DECODE, [Bucket(4, 5, [0.01]), Bucket(6, 5, [0.01]),
                                                     Bucket(5, 4, [0.01]), Bucket(5, 6, [0.01])])
    out["tie_break"] = [[b.tt, b.conc] for b, _ in pool_neighbors(tie, (5, 5), 100)]
    anchors = [Bucket(1, 1, [9.001] * 10), Bucket(1001, 101, [9.002] * 10)]
    near = [Bucket(600, 50, [0.010] * 10), Bucket(700, 50, [0.020] * 10), Bucket(900, 50, [0.040] * 10)]
    t3 = PhaseTable.from_buckets(TableKind.DECODE, anchors + near)
    out["shepard3_dists"] = [d for _, d in pool_neighbors(t3, (500, 50), 30)]
    pack3 = ProfilePack(16, t3, PhaseTable.from_buckets(TableKind.MIXED, []),
                        PhaseTable.from_buckets(TableKind.COMBINED,
                                                [Bucket(b.tt, b.conc, list(b.samples)) for b in anchors + near]))
    rng = np.random.default_rng(20240810)
    draws = [sample_latency(pack3, OracleQuery(500, 50, DEC), OracleConfig(reliability_floor=30), rng)
             for _ in range(100_000)]
    c = Counter(draws)
    out["shepard3_counts"] = [c[0.010], c[0.020], c[0.040]]
    out["shepard3_seq_sha256"] = sha(np.array(draws, dtype=np.float64).tobytes())
    # acceptance criterion 3 (variance)
    r3 = random.Random(99)
    samples = [r3.lognormvariate(math.log(0.005), 0.35) for _ in range(1000)]
    t_var = PhaseTable.from_buckets(TableKind.DECODE, [Bucket(12, 12, samples)])
    pack_var = ProfilePack(16, t_var, PhaseTable.from_buckets(TableKind.MIXED, []),
                           PhaseTable.from_buckets(TableKind.COMBINED, [Bucket(12, 12, list(samples))]))
    gen = np.random.default_rng(31337)
    dv = [sample_latency(pack_var, OracleQuery(12, 12, DEC), OracleConfig(reliability_floor=500), gen)
          for _ in range(10_000)]
    out["variance_seq_sha256"] = sha(np.array(dv, dtype=np.float64).tobytes())
    # acceptance criterion 1 tables (random.Random(2024)), pools + distances
    rng1 = random.Random(2024)
    tables = []
    for _ in range(100):
        nb = rng1.randint(1, 500)
        ks = set()
        while len(ks) < nb:
            ks.add((rng1.randint(1, 2000), rng1.randint(1, 128)))
        buckets = [Bucket(tt_, cc_, [0.001] * rng1.randint(1, 40)) for tt_, cc_ in ks]
        table = PhaseTable.from_buckets(TableKind.COMBINED, buckets)
        q = (rng1.randint(1, 2200), rng1.randint(1, 140))
        fl = rng1.choice([1, 8, 32, 256, 10**9])
        pooled = pool_neighbors(table, q, fl)
        tables.append({"query": list(q), "floor": fl,
                       "pool": [[b.tt, b.conc] for b, _ in pooled], "dist": [d for _, d in pooled]})
    out["acceptance_c1"] = tables
    # canonical bytes of a small mixed pack (profile round trip)
    recs = [StepTraceRecord(0, 3, 3, DEC, 0.012), StepTraceRecord(1, 3, 3, DEC, 0.010),
            StepTraceRecord(2, 64, 1, MIX, 0.05), StepTraceRecord(3, 7, 2, MIX, 0.02)]
    out["small_pack_bytes"] = save_pack(build_pack(recs, 7, {"model": "toy", "gpu": "none"})).decode()
    with open(os.path.join(HERE, "fixtures.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote fixtures; unique keys in trace:", n_unique)


if __name__ == "__main__":
    main()
