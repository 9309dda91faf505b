"""The reference's own oracle/profile tests, restated against this package.

Each test cites the reference test it restates (pkg/tests/...).  They drive
the public API exactly as serve_emu's tests drive serve_emu, so passing them
shows the drop-in keeps the reference's observable behaviour; every
computation underneath runs in libemu_b200.so on the GPU.
"""
from __future__ import annotations

import math
import random
from collections import Counter

import numpy as np
import pytest

from paper_2605_00616_b200 import (
    Bucket,
    LatencyOracle,
    NoProfileDataError,
    OracleConfig,
    OracleQuery,
    PackValidationError,
    PhaseTable,
    ProfilePack,
    StepPhase,
    StepTraceRecord,
    TableKind,
    build_pack,
    load_pack,
    normalized_distance,
    pool_neighbors,
    sample_latency,
    save_pack,
)

pytestmark = pytest.mark.gpu
DEC, MIX = StepPhase.DECODE_ONLY, StepPhase.PREFILL_OR_MIXED


def make_pack(decode, mixed, blocks=16):
    """Pack whose combined table merges both phases (cf. test_oracle.py:39-50)."""
    merged: dict[tuple[int, int], list[float]] = {}
    for b in list(decode) + list(mixed):
        merged.setdefault((b.tt, b.conc), []).extend(b.samples)
    return ProfilePack(
        blocks,
        PhaseTable.from_buckets(TableKind.DECODE, [Bucket(b.tt, b.conc, list(b.samples)) for b in decode]),
        PhaseTable.from_buckets(TableKind.MIXED, [Bucket(b.tt, b.conc, list(b.samples)) for b in mixed]),
        PhaseTable.from_buckets(TableKind.COMBINED, [Bucket(k[0], k[1], v) for k, v in merged.items()]),
    )


def sorted_prefix(table, query, floor):
    """Independent brute force: full (d, tt, conc) sort, shortest prefix >= floor
    (test_oracle.py:53-67, test_acceptance.py:82-99)."""
    ranked = sorted(((normalized_distance(query, (b.tt, b.conc), table.tt_range, table.conc_range), b.tt, b.conc, b)
                     for b in table.buckets), key=lambda r: r[:3])
    out, total = [], 0
    for d, _, _, b in ranked:
        out.append((b, d))
        total += len(b.samples)
        if total >= floor:
            break
    return out


def keys_of(pooled):
    return [(b.tt, b.conc) for b, _ in pooled]


def anchored(near, n_anchor=10):
    """Range anchors pin spans to tt 1000 / conc 100 (test_oracle.py:165-174)."""
    return [Bucket(1, 1, [9.001] * n_anchor), Bucket(1001, 101, [9.002] * n_anchor), *near]


# ------------------------------------------------------ normalized_distance
@pytest.mark.parametrize("q,b,tr,cr,want,tol", [
    ((3, 3), (3, 3), (1, 10), (1, 10), 0.0, 0.0),                       # test_oracle.py:71-72
    ((51, 6), (101, 11), (1, 101), (1, 11), math.sqrt(0.5), 1e-9),      # :74-77
    ((10, 9), (20, 4), (0, 100), (4, 4), 0.1, 1e-12),                   # :79-81 degenerate axis
])
def test_distance_examples(q, b, tr, cr, want, tol):
    assert abs(normalized_distance(q, b, tr, cr) - want) <= tol


# ------------------------------------------------------ pool_neighbors
def test_exact_hit_meets_floor():  # test_oracle.py:85-92
    t = PhaseTable.from_buckets(TableKind.DECODE, [Bucket(3, 3, [0.01] * 5), Bucket(9, 9, [0.02] * 5)])
    got = pool_neighbors(t, (3, 3), 1)
    assert keys_of(got) == [(3, 3)] and got[0][1] == 0.0


def test_expands_until_floor():  # :94-106
    t = PhaseTable.from_buckets(TableKind.DECODE, [Bucket(10, 5, [0.01] * 4), Bucket(12, 5, [0.02] * 7),
                                                   Bucket(40, 5, [0.03] * 50)])
    got = pool_neighbors(t, (10, 5), 10)
    assert keys_of(got) == [(10, 5), (12, 5)] and sum(len(b.samples) for b, _ in got) == 11
    assert got == sorted_prefix(t, (10, 5), 10)


def test_exhaustion_and_empty():  # :108-117
    t = PhaseTable.from_buckets(TableKind.DECODE, [Bucket(i, 1, [0.01] * 10) for i in range(1, 11)])
    assert len(pool_neighbors(t, (5, 1), 10**6)) == 10
    with pytest.raises(NoProfileDataError):
        pool_neighbors(PhaseTable.from_buckets(TableKind.DECODE, []), (1, 1), 1)
    with pytest.raises(ValueError):
        pool_neighbors(t, (5, 1), 0)


def test_equidistant_ties_ascend_by_key():  # :119-126
    t = PhaseTable.from_buckets(TableKind.DECODE, [Bucket(4, 5, [0.01]), Bucket(6, 5, [0.01]), Bucket(5, 4, [0.01]),
                                                   Bucket(5, 6, [0.01])])
    assert keys_of(pool_neighbors(t, (5, 5), 100)) == [(4, 5), (5, 4), (5, 6), (6, 5)]


def test_brute_force_random_small_tables():  # :128-146
    rng = random.Random(7)
    for _ in range(20):
        seen, buckets = set(), []
        for _ in range(rng.randint(1, 120)):
            k = (rng.randint(1, 60), rng.randint(1, 12))
            if k not in seen:
                seen.add(k)
                buckets.append(Bucket(*k, [0.01] * rng.randint(1, 9)))
        t = PhaseTable.from_buckets(TableKind.COMBINED, buckets)
        q = (rng.randint(1, 70), rng.randint(1, 14))
        fl = rng.choice([1, 4, 32, 10**9])
        got, want = pool_neighbors(t, q, fl), sorted_prefix(t, q, fl)
        assert keys_of(got) == keys_of(want)
        assert [d for _, d in got] == [d for _, d in want]  # bit-equal distances


def test_prefix_is_minimal():  # :148-162
    rng = random.Random(3)
    for _ in range(20):
        buckets = [Bucket(tt, c, [0.01] * rng.randint(1, 6)) for tt in range(1, 12) for c in range(1, 4)]
        t = PhaseTable.from_buckets(TableKind.COMBINED, buckets)
        fl = rng.randint(1, 40)
        got = pool_neighbors(t, (rng.randint(1, 12), rng.randint(1, 4)), fl)
        total = sum(len(b.samples) for b, _ in got)
        if len(got) < len(buckets):
            assert total >= fl and total - len(got[-1][0].samples) < fl


def test_acceptance_1_brute_force_100_tables():  # test_acceptance.py:102-123
    rng = random.Random(2024)
    for _ in range(100):
        n = rng.randint(1, 500)
        keys = set()
        while len(keys) < n:
            keys.add((rng.randint(1, 2000), rng.randint(1, 128)))
        t = PhaseTable.from_buckets(TableKind.COMBINED, [Bucket(a, b, [0.001] * rng.randint(1, 40)) for a, b in keys])
        q = (rng.randint(1, 2200), rng.randint(1, 140))
        fl = rng.choice([1, 8, 32, 256, 10**9])
        got, want = pool_neighbors(t, q, fl), sorted_prefix(t, q, fl)
        assert keys_of(got) == keys_of(want) and [d for _, d in got] == [d for _, d in want]


# ------------------------------------------------------ sample_latency
def test_single_bucket_single_value():  # test_oracle.py:178-182
    pack = make_pack([Bucket(3, 3, [0.020])], [])
    g = np.random.default_rng(0)
    assert all(sample_latency(pack, OracleQuery(3, 3, DEC), OracleConfig(reliability_floor=1), g) == 0.020
               for _ in range(20))


def test_exact_hit_dominates():  # :184-193
    pack = make_pack(anchored([Bucket(500, 50, [0.010] * 10), Bucket(900, 50, [0.099] * 10)]), [])
    g = np.random.default_rng(42)
    draws = {sample_latency(pack, OracleQuery(500, 50, DEC), OracleConfig(reliability_floor=20), g)
             for _ in range(20_000)}
    assert draws == {0.010}


def test_two_bucket_mixture():  # :195-207
    pack = make_pack(anchored([Bucket(600, 50, [0.010] * 10), Bucket(800, 50, [0.030] * 10)]), [])
    assert [round(d, 12) for _, d in pool_neighbors(pack.decode_table, (500, 50), 20)] == [0.1, 0.3]
    g = np.random.default_rng(123)
    n = 100_000
    c = Counter(sample_latency(pack, OracleQuery(500, 50, DEC), OracleConfig(reliability_floor=20), g)
                for _ in range(n))
    assert abs(c[0.010] / n - 0.9) <= 0.01 and abs(c[0.030] / n - 0.1) <= 0.01


def test_membership_and_determinism():  # :209-226
    rng = random.Random(11)
    recs = [StepTraceRecord(i, rng.randint(1, 50) + 5, rng.randint(1, 6), MIX, rng.uniform(0.001, 0.1))
            for i in range(100)]
    pack = build_pack(recs, 8)
    values = {s for b in pack.mixed_table.buckets for s in b.samples}
    cfg = OracleConfig(reliability_floor=9, rng_seed=5)
    g1, g2 = np.random.default_rng(5), np.random.default_rng(5)
    a = [sample_latency(pack, OracleQuery(20, 3, MIX), cfg, g1) for _ in range(200)]
    b = [sample_latency(pack, OracleQuery(20, 3, MIX), cfg, g2) for _ in range(200)]
    assert a == b and set(a) <= values


def test_fallback_and_empty():  # :228-239
    pack = make_pack([], [Bucket(64, 1, [0.05] * 3)])
    g = np.random.default_rng(0)
    assert sample_latency(pack, OracleQuery(3, 3, DEC), OracleConfig(reliability_floor=1), g) == 0.05
    with pytest.raises(NoProfileDataError):
        sample_latency(make_pack([], []), OracleQuery(3, 3, DEC), OracleConfig(), g)
    with pytest.raises(ValueError):
        sample_latency(pack, OracleQuery(0, 3, DEC), OracleConfig(), g)
    with pytest.raises(ValueError):
        sample_latency(pack, OracleQuery(3, 3, DEC), OracleConfig(reliability_floor=0), g)


def test_variance_preserved():  # :241-248 and acceptance criterion 3 (test_acceptance.py:168-186)
    r = random.Random(99)
    samples = [r.lognormvariate(math.log(0.005), 0.35) for _ in range(1000)]
    pack = make_pack([Bucket(12, 12, samples)], [])
    g = np.random.default_rng(31337)
    draws = [sample_latency(pack, OracleQuery(12, 12, DEC), OracleConfig(reliability_floor=500), g)
             for _ in range(10_000)]
    assert abs(np.var(draws) - np.var(samples)) / np.var(samples) <= 0.10


def test_acceptance_2_three_bucket_shepard(fixtures):  # test_acceptance.py:129-162
    near = [Bucket(600, 50, [0.010] * 10), Bucket(700, 50, [0.020] * 10), Bucket(900, 50, [0.040] * 10)]
    pack = make_pack(anchored(near), [])
    cfg = OracleConfig(reliability_floor=30, shepard_power=2.0)
    d = [dd for _, dd in pool_neighbors(pack.decode_table, (500, 50), 30)]
    assert [round(x, 12) for x in d] == [0.1, 0.2, 0.4]
    w = [1 / x**2 for x in d]
    g = np.random.default_rng(20240810)
    n = 100_000
    seq = [sample_latency(pack, OracleQuery(500, 50, DEC), cfg, g) for _ in range(n)]
    c = Counter(seq)
    for v, wi in zip((0.010, 0.020, 0.040), w):
        assert abs(c[v] / n - wi / sum(w)) <= 0.01
    # and the exact sequence the reference drew with this seed
    import hashlib

    assert hashlib.sha256(np.array(seq).tobytes()).hexdigest() == fixtures["shepard3_seq_sha256"]


# ------------------------------------------------------ LatencyOracle
def test_oracle_pooled_matches_functional():  # test_oracle.py:252-271
    rng = random.Random(4)
    recs = []
    for i in range(200):
        tt, c = rng.randint(2, 40), rng.randint(1, 5)
        recs.append(StepTraceRecord(i, max(tt, c), c, DEC, rng.uniform(0.001, 0.02)))
    pack = build_pack(recs, 8)
    cfg = OracleConfig(reliability_floor=17, rng_seed=1)
    orc = LatencyOracle(pack, cfg)
    for q in [(5, 2), (33, 4), (100, 1)]:
        pooled = pool_neighbors(pack.decode_table, q, cfg.reliability_floor)
        probs, samples = orc._pooled(DEC, *q)
        assert [len(s) for s in samples] == [len(b.samples) for b, _ in pooled]
        assert probs.sum() == pytest.approx(1.0)


def test_oracle_draws_are_pack_values():  # :273-278
    orc = LatencyOracle(make_pack([Bucket(4, 4, [0.011, 0.012, 0.013])], [Bucket(64, 1, [0.05])]),
                        OracleConfig(reliability_floor=2, rng_seed=0))
    assert all(orc.sample(4, 4, DEC) in {0.011, 0.012, 0.013} for _ in range(50))
    assert orc.sample(64, 1, MIX) == 0.05


def test_oracle_determinism_across_instances():  # :280-293
    rng = random.Random(6)
    recs = [StepTraceRecord(i, rng.randint(1, 30) + 3, rng.randint(1, 4), MIX, rng.uniform(0.001, 0.05))
            for i in range(150)]
    pack = build_pack(recs, 8)
    cfg = OracleConfig(reliability_floor=8, rng_seed=77)
    a, b = LatencyOracle(pack, cfg), LatencyOracle(pack, cfg)
    qs = [(rng.randint(1, 40), rng.randint(1, 5)) for _ in range(100)]
    assert [a.sample(t, c, MIX) for t, c in qs] == [b.sample(t, c, MIX) for t, c in qs]


def test_membership_property_random_packs():  # :296-316 (hypothesis -> seeded loop)
    rng = random.Random(17)
    for _ in range(40):
        keys = {(rng.randint(1, 40), rng.randint(1, 8)) for _ in range(rng.randint(1, 30))}
        buckets = [Bucket(tt, c, [rng.uniform(1e-4, 1.0) for _ in range(rng.randint(1, 5))]) for tt, c in keys]
        pack = make_pack([], buckets)
        q = OracleQuery(rng.randint(1, 50), rng.randint(1, 10), MIX)
        fl = rng.randint(1, 200)
        v = sample_latency(pack, q, OracleConfig(reliability_floor=fl), np.random.default_rng(0))
        assert any(v in b.samples for b, _ in pool_neighbors(pack.mixed_table, (q.total_tokens, q.concurrency), fl))


# ------------------------------------------------------ profile (GPU build)
def test_build_basic_shapes():  # test_profile.py:36-60
    pack = build_pack([], num_gpu_blocks=100, metadata={})
    assert all(t.buckets == [] and t.tt_range is None for t in (pack.decode_table, pack.mixed_table,
                                                                pack.combined_table))
    pack.validate()
    pack = build_pack([StepTraceRecord(i, 3, 3, DEC, v) for i, v in enumerate([0.010, 0.011, 0.012])], 10)
    assert len(pack.decode_table.buckets) == 1 and sorted(pack.decode_table.buckets[0].samples) == [0.010, 0.011,
                                                                                                     0.012]
    assert pack.mixed_table.buckets == [] and len(pack.combined_table.buckets[0].samples) == 3
    pack = build_pack([StepTraceRecord(0, 3, 3, DEC, 0.01), StepTraceRecord(1, 64, 1, MIX, 0.05)], 10)
    assert (len(pack.decode_table.buckets), len(pack.mixed_table.buckets), len(pack.combined_table.buckets)) == (1, 1, 2)


@pytest.mark.parametrize("bad", [StepTraceRecord(0, 3, 3, DEC, 0.0), StepTraceRecord(0, 3, 3, DEC, -1.0),
                                 StepTraceRecord(0, 0, 1, MIX, 0.1), StepTraceRecord(0, 3, 0, MIX, 0.1)])
def test_build_names_bad_record(bad):  # test_profile.py:62-73
    with pytest.raises(PackValidationError, match="trace record 1"):
        build_pack([StepTraceRecord(0, 2, 2, DEC, 0.01), bad], num_gpu_blocks=10)


def test_build_rejects_decode_below_concurrency():  # :75-77
    with pytest.raises(PackValidationError, match="decode-only"):
        build_pack([StepTraceRecord(0, 2, 3, DEC, 0.01)], num_gpu_blocks=10)


def test_canonical_bytes_ignore_insertion_order():  # :102-114
    recs = [StepTraceRecord(0, 3, 3, DEC, 0.012), StepTraceRecord(1, 5, 2, MIX, 0.02),
            StepTraceRecord(2, 3, 3, DEC, 0.010), StepTraceRecord(3, 9, 4, DEC, 0.03)]
    shuffled = recs[:]
    random.Random(1).shuffle(shuffled)
    shuffled = [StepTraceRecord(i, r.total_tokens, r.concurrency, r.phase, r.latency_s) for i, r in enumerate(shuffled)]
    assert save_pack(build_pack(recs, 7)) == save_pack(build_pack(shuffled, 7))


def test_acceptance_9_round_trip_and_conservation():  # test_acceptance.py:460-479
    rng = random.Random(31)
    for _ in range(50):
        recs = []
        for i in range(rng.randint(0, 400)):
            c = rng.randint(1, 32)
            ph = rng.choice([DEC, MIX])
            recs.append(StepTraceRecord(i, c if ph is DEC else rng.randint(1, 600), c, ph, rng.uniform(1e-4, 0.5)))
        pack = build_pack(recs, num_gpu_blocks=rng.randint(1, 10_000))
        assert load_pack(save_pack(pack)) == pack
        assert pack.combined_table.total_samples == len(recs)
        assert pack.decode_table.total_samples + pack.mixed_table.total_samples == len(recs)
