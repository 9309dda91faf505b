"""Golden vectors at the bench configs, from the UNMODIFIED reference (dev container only).

    python tests/golden/make_golden_big.py

Imports serve_emu from /root/reference/pkg/src (read-only).  Writes
tests/golden/c2_golden.npz and c3_golden.npz; tests load only those files.

C2 (BASELINE configs[1]): pack = build_pack over records_llama(1_000_000, 0)
   canonicalised with load_pack(save_pack(.)) (server.py:60 loads from file);
   keys = the first 2,000 unique keys of the bench workload queries_llama(10M, 1)
   (bench.py rank 0) + 500 keys outside the table's range; per key the
   reference pool (_pool_order, oracle.py:80-105) and probabilities
   (LatencyOracle._pooled -> _selection_probs, oracle.py:124-127, :200-222);
   LatencyOracle.sample over the first 10,000 bench queries (rng_seed 0) with
   its final PCG64 state; canonical table digests.
C3 (configs[2]): pack over records_sparse(1_000_000, 0); keys = the first 800
   unique keys of queries_sparse(10M, 1) + 200 outside the range; pools at
   floor 32 and 256.

Per key the fixture holds sha256(tt i32[K] | conc i32[K] | dist f64[K] | prob f64[K])
(little endian) and, for the first 200 keys, the arrays themselves.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from serve_emu.oracle import LatencyOracle, OracleConfig, _pool_order  # noqa: E402
from serve_emu.profile import StepPhase, StepTraceRecord, build_pack, load_pack, save_pack  # noqa: E402

from paper_2605_00616_b200.workloads import (  # noqa: E402  (numpy-only module)
    queries_llama,
    queries_sparse,
    records_llama,
    records_sparse,
)

DEC, MIX = StepPhase.DECODE_ONLY, StepPhase.PREFILL_OR_MIXED
N_FULL = 200


def records_hash(*cols) -> str:
    h = hashlib.sha256()
    for a in cols:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def table_digest(table) -> str:  # same definition as make_golden.py
    h = hashlib.sha256()
    for b in table.buckets:
        h.update(np.array([b.tt, b.conc, len(b.samples)], dtype=np.int64).tobytes())
        h.update(np.asarray(b.samples, dtype=np.float64).tobytes())
    return h.hexdigest()


def pool_digest(tt, conc, dist, prob) -> bytes:
    h = hashlib.sha256()
    for a, dt in ((tt, "<i4"), (conc, "<i4"), (dist, "<f8"), (prob, "<f8")):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.digest()


def canonical_pack(tt, conc, ph, lat):
    recs = [StepTraceRecord(i, int(a), int(b), MIX if c else DEC, float(d))
            for i, (a, b, c, d) in enumerate(zip(tt.tolist(), conc.tolist(), ph.tolist(), lat.tolist()))]
    return load_pack(save_pack(build_pack(recs, 1000)))


def first_unique(qt, qc, qp, n):
    seen, out = set(), []
    for k in zip(qt.tolist(), qc.tolist(), qp.tolist()):
        if k not in seen:
            seen.add(k)
            out.append(k)
            if len(out) == n:
                break
    return out


def outside_keys(n, tt_hi, seed):
    g = np.random.default_rng(seed)
    tt = np.where(g.random(n) < 0.5, g.integers(-20, 1, n), g.integers(tt_hi + 1, tt_hi + tt_hi // 2, n))
    conc = g.integers(-5, 320, n)
    return list(zip(tt.tolist(), conc.tolist(), g.integers(0, 2, n).tolist()))


def pools_of(canon, keys, floor):
    orc = LatencyOracle(canon, OracleConfig(reliability_floor=floor))
    dig, off, ptt, pc, pd, pp = [], [0], [], [], [], []
    for i, (t, c, p) in enumerate(keys):
        ph = MIX if p else DEC
        idx = orc._indices[ph] if not orc._indices[ph].empty else orc._combined
        table = canon.mixed_table if p else canon.decode_table
        if table.is_empty:
            table = canon.combined_table
        chosen, dists = _pool_order(idx.tts, idx.concs, idx.counts, idx.tt_range, idx.conc_range, (t, c), floor)
        probs, _ = orc._pooled(ph, t, c)
        btt = np.array([table.buckets[j].tt for j in chosen], np.int32)
        bc = np.array([table.buckets[j].conc for j in chosen], np.int32)
        dig.append(np.frombuffer(pool_digest(btt, bc, dists, probs), np.uint8))
        if i < N_FULL:
            ptt += btt.tolist()
            pc += bc.tolist()
            pd += list(dists)
            pp += list(probs)
            off.append(len(ptt))
    return dict(digest=np.stack(dig), off=np.array(off, np.int64), tt=np.array(ptt, np.int32),
                conc=np.array(pc, np.int32), dist=np.array(pd, np.float64), prob=np.array(pp, np.float64))


def keys_array(keys):
    k = np.array(keys, dtype=np.int64)
    return k[:, 0].astype(np.int32), k[:, 1].astype(np.int32), k[:, 2].astype(np.uint8)


def main():
    t0 = time.time()
    # ------------------------------------------------------------------ C2
    rec = records_llama(1_000_000, 0)
    canon = canonical_pack(*rec)
    print("C2 pack", time.time() - t0, flush=True)
    qt, qc, qp = queries_llama(10_000_000, 1)
    keys = first_unique(qt[:200_000], qc[:200_000], qp[:200_000], 2000) + outside_keys(500, 2048, 77)
    kt, kc, kp = keys_array(keys)
    pools = pools_of(canon, keys, 32)
    print("C2 pools", time.time() - t0, flush=True)
    orc = LatencyOracle(canon, OracleConfig(reliability_floor=32, rng_seed=0))
    n_seq = 10_000
    lat_seq = np.array([orc.sample(int(a), int(b), MIX if c else DEC)
                        for a, b, c in zip(qt[:n_seq], qc[:n_seq], qp[:n_seq])], dtype=np.float64)
    st = orc._rng.bit_generator.state
    final = np.array([st["state"]["state"] >> 64, st["state"]["state"] & (2**64 - 1), st["state"]["inc"] >> 64,
                      st["state"]["inc"] & (2**64 - 1), st["has_uint32"], st["uinteger"]], dtype=np.uint64)
    print("C2 stream", time.time() - t0, flush=True)
    np.savez_compressed(
        os.path.join(HERE, "c2_golden.npz"), key_tt=kt, key_conc=kc, key_phase=kp,
        **{"pool_" + k: v for k, v in pools.items()},
        seq_tt=qt[:n_seq], seq_conc=qc[:n_seq], seq_phase=qp[:n_seq], lat_seq=lat_seq, final_state=final,
        records_sha256=np.array(records_hash(*rec)), queries_sha256=np.array(records_hash(qt, qc, qp)),
        canon_digest=np.array([table_digest(t) for t in (canon.decode_table, canon.mixed_table,
                                                         canon.combined_table)]))
    # ------------------------------------------------------------------ C3
    rec = records_sparse(1_000_000, 0)
    canon = canonical_pack(*rec)
    print("C3 pack", time.time() - t0, flush=True)
    qt, qc, qp = queries_sparse(10_000_000, 1)
    keys = first_unique(qt[:100_000], qc[:100_000], qp[:100_000], 800) + outside_keys(200, 131072, 78)
    kt, kc, kp = keys_array(keys)
    out = dict(key_tt=kt, key_conc=kc, key_phase=kp, records_sha256=np.array(records_hash(*rec)),
               queries_sha256=np.array(records_hash(qt, qc, qp)),
               canon_digest=np.array([table_digest(t) for t in (canon.decode_table, canon.mixed_table,
                                                                canon.combined_table)]))
    for floor in (32, 256):
        pools = pools_of(canon, keys, floor)
        out.update({f"m{floor}_" + k: v for k, v in pools.items()})
        print("C3 pools M", floor, time.time() - t0, flush=True)
    np.savez_compressed(os.path.join(HERE, "c3_golden.npz"), **out)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
