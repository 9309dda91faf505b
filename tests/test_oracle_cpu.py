"""Pin the CPU restatement (oracle/) against golden vectors from the reference.

These run on CPU only.  They prove the checker itself is right before it is
used to judge the CUDA path (tests/test_gpu_*.py).
"""
from __future__ import annotations

import hashlib
import math
import random

import numpy as np
import pytest

import emu_oracle as O


def digest(t: O.Table) -> str:
    h = hashlib.sha256()
    for i in range(t.nb):
        h.update(np.array([t.tt[i], t.conc[i], t.off[i + 1] - t.off[i]], dtype=np.int64).tobytes())
        h.update(t.samples[t.off[i]:t.off[i + 1]].tobytes())
    return h.hexdigest()


def one_table(buckets):
    """[table, empty, table] so phase 0 resolves to `buckets`."""
    t = O.table_from_buckets(buckets)
    e = O.Table(np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(1, np.int64), np.zeros(0))
    return [t, e, t]


class B:  # minimal bucket
    def __init__(self, tt, conc, samples):
        self.tt, self.conc, self.samples = tt, conc, samples


def test_build_matches_reference_digests(c1_records, fixtures):
    canon = O.build(*c1_records, canonical=True)
    raw = O.build(*c1_records, canonical=False)
    assert [t.nb for t in canon] == fixtures["c1"]["buckets"]
    assert [digest(t) for t in canon] == fixtures["c1"]["canon_table_digest"]
    assert [digest(t) for t in raw] == fixtures["c1"]["raw_table_digest"]


def test_pcg64_stream_matches_reference(c1_tables, c1_trace, c1_golden):
    st = O.pcg64_state6(0)
    lat, _ = O.sample_pcg64(c1_tables, c1_trace["tt"], c1_trace["conc"], c1_trace["phase"], 32, state6=st)
    assert np.array_equal(lat, c1_golden["lat_seq"])
    assert st.tolist() == c1_golden["final_state"].tolist()


def test_pcg64_stream_other_knobs(c1_tables, c1_trace, c1_golden):
    st = O.pcg64_state6(12345)
    n = len(c1_golden["lat_seq_m8_p15"])
    lat, _ = O.sample_pcg64(c1_tables, c1_trace["tt"][:n], c1_trace["conc"][:n], c1_trace["phase"][:n], 8,
                            p=1.5, state6=st)
    # p = 1.5 goes through pow(): numpy's SIMD pow may differ by 1 ulp, which can
    # only move a draw whose uniform lies within ~1e-16 of a CDF step.
    assert np.mean(lat == c1_golden["lat_seq_m8_p15"]) == 1.0


def test_pools_match_reference(c1_tables, c1_golden):
    uk = c1_golden["uk"]
    off, bkt, dist, prob, cdf, tid = O.pools(c1_tables, uk[:, 0], uk[:, 1], uk[:, 2], 32)
    g_off = c1_golden["p_off"]
    assert np.array_equal(off, g_off)
    tt = np.concatenate([c1_tables[t].tt[bkt[off[u]:off[u + 1]]] for u, t in enumerate(tid)])
    cc = np.concatenate([c1_tables[t].conc[bkt[off[u]:off[u + 1]]] for u, t in enumerate(tid)])
    assert np.array_equal(tt, c1_golden["p_tt"])
    assert np.array_equal(cc, c1_golden["p_conc"])
    assert np.array_equal(dist, c1_golden["p_dist"])  # bit-exact
    assert np.array_equal(prob, c1_golden["p_prob"])  # bit-exact (p = 2)


def test_tie_break_and_shepard_fixture(fixtures):
    tabs = one_table([B(4, 5, [0.01]), B(6, 5, [0.01]), B(5, 4, [0.01]), B(5, 6, [0.01])])
    off, bkt, *_ = O.pools(tabs, [5], [5], [0], 100)
    assert [[int(tabs[0].tt[b]), int(tabs[0].conc[b])] for b in bkt] == fixtures["tie_break"]
    near = [B(1, 1, [9.001] * 10), B(1001, 101, [9.002] * 10), B(600, 50, [0.01] * 10), B(700, 50, [0.02] * 10),
            B(900, 50, [0.04] * 10)]
    tabs = one_table(near)
    off, bkt, dist, prob, cdf, _ = O.pools(tabs, [500], [50], [0], 30)
    assert dist.tolist() == fixtures["shepard3_dists"]


def test_acceptance_c1_tables(fixtures):
    rng = random.Random(2024)
    for want in fixtures["acceptance_c1"]:
        nb = rng.randint(1, 500)
        ks = set()
        while len(ks) < nb:
            ks.add((rng.randint(1, 2000), rng.randint(1, 128)))
        buckets = [B(t, c, [0.001] * rng.randint(1, 40)) for t, c in ks]
        q = (rng.randint(1, 2200), rng.randint(1, 140))
        fl = rng.choice([1, 8, 32, 256, 10**9])
        assert [list(q), fl] == [want["query"], want["floor"]]
        tabs = one_table(buckets)
        off, bkt, dist, *_ = O.pools(tabs, [q[0]], [q[1]], [0], fl)
        assert [[int(tabs[0].tt[b]), int(tabs[0].conc[b])] for b in bkt] == want["pool"]
        assert dist.tolist() == want["dist"]


def test_shepard_sequence_matches_reference(fixtures):
    near = [B(1, 1, [9.001] * 10), B(1001, 101, [9.002] * 10), B(600, 50, [0.01] * 10), B(700, 50, [0.02] * 10),
            B(900, 50, [0.04] * 10)]
    tabs = one_table(near)
    st = O.pcg64_state6(20240810)
    n = 100_000
    lat, _ = O.sample_pcg64(tabs, np.full(n, 500), np.full(n, 50), np.zeros(n), 30, state6=st)
    assert hashlib.sha256(lat.tobytes()).hexdigest() == fixtures["shepard3_seq_sha256"]
    assert [int((lat == v).sum()) for v in (0.01, 0.02, 0.04)] == fixtures["shepard3_counts"]


def test_variance_sequence_matches_reference(fixtures):
    r3 = random.Random(99)
    samples = [r3.lognormvariate(math.log(0.005), 0.35) for _ in range(1000)]
    tabs = one_table([B(12, 12, samples)])
    st = O.pcg64_state6(31337)
    lat, _ = O.sample_pcg64(tabs, np.full(10_000, 12), np.full(10_000, 12), np.zeros(10_000), 500, state6=st)
    assert hashlib.sha256(lat.tobytes()).hexdigest() == fixtures["variance_seq_sha256"]


def test_token_fill_matches_reference(c1_trace):
    t = c1_trace
    ids, fin = O.token_fill(t["tok_is_prefill"], t["tok_chunk"], t["tok_progress"], t["tok_prompt_len"],
                            t["tok_generated"], t["tok_target"])
    assert np.array_equal(ids, t["tok_ids"])
    assert np.array_equal(fin, t["tok_fin"])


def test_pairwise_sum_matches_numpy():
    rng = np.random.default_rng(5)
    for n in list(range(0, 300)) + [1000, 4097, 70000]:
        a = rng.random(n) * np.exp(rng.normal(0, 8, n))
        assert O.pairwise_sum(a) == a.sum()


def test_distance_examples():
    assert O.distance((3, 3), (3, 3), (1, 10), (1, 10)) == 0.0
    assert abs(O.distance((51, 6), (101, 11), (1, 101), (1, 11)) - math.sqrt(0.5)) < 1e-12
    assert abs(O.distance((10, 9), (20, 4), (0, 100), (4, 4)) - 0.1) < 1e-12


def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32 R=10
    assert O.philox4x32_10([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert O.philox4x32_10([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert O.philox4x32_10([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == [
        0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_pcg64_words_match_numpy():
    st = O.pcg64_state6(987)
    w = O.pcg64_words(st, 1000)
    assert np.array_equal(w, np.random.PCG64(987).random_raw(1000))


def test_explicit_mode_equals_pcg_mode_given_same_words(c1_tables, c1_trace):
    """EXPLICIT mode feeds the same draw routine: with the words a PCG64 stream
    hands out (in numpy's consumption order), results equal the PCG64 replay."""
    n = 2000
    qt, qc, qp = c1_trace["tt"][:n], c1_trace["conc"][:n], c1_trace["phase"][:n]
    st = O.pcg64_state6(77)
    lat_pcg, sidx_pcg = O.sample_pcg64(c1_tables, qt, qc, qp, 32, state6=st)
    off, bkt, dist, prob, cdf, tid = O.pools(c1_tables, qt, qc, qp, 32)
    bg = np.random.PCG64(77)
    buf = {"has": False, "v": 0}

    def next32():
        if buf["has"]:
            buf["has"] = False
            return buf["v"]
        w = int(bg.random_raw())
        buf["has"], buf["v"] = True, w >> 32
        return w & 0xFFFFFFFF

    usel = np.zeros(n, np.uint64)
    uidx = np.zeros(n, np.uint32)
    for i in range(n):
        usel[i] = int(bg.random_raw())
        u = (int(usel[i]) >> 11) * (1.0 / 9007199254740992.0)
        j = int(np.searchsorted(cdf[off[i]:off[i + 1]], u, side="right"))
        t = c1_tables[tid[i]]
        b = bkt[off[i] + j]
        nn = int(t.off[b + 1] - t.off[b])
        if nn > 1:
            uidx[i] = next32()
            assert (int(uidx[i]) * nn) & 0xFFFFFFFF >= (2**32 - nn) % nn  # no rejection in this window
    lat_ex, sidx_ex = O.sample_batch(c1_tables, qt, qc, qp, 32, mode="explicit", u_sel=usel, u_idx=uidx)
    assert np.array_equal(sidx_ex, sidx_pcg)
    assert np.array_equal(lat_ex, lat_pcg)


def test_threads_do_not_change_results(c1_tables):
    from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama

    qt, qc, qp = queries_llama(20_000, 3)
    us, ui = explicit_uniforms(20_000, 4)
    a = O.sample_batch(c1_tables, qt, qc, qp, 32, mode="explicit", u_sel=us, u_idx=ui, threads=1)
    b = O.sample_batch(c1_tables, qt, qc, qp, 32, mode="explicit", u_sel=us, u_idx=ui, threads=4)
    assert np.array_equal(a[1], b[1])
    c = O.sample_batch(c1_tables, qt, qc, qp, 32, mode="philox", seed=9, threads=3)
    d = O.sample_batch(c1_tables, qt, qc, qp, 32, mode="philox", seed=9, threads=1)
    assert np.array_equal(c[1], d[1])


def test_build_rejects_invalid_records():
    tt = np.array([2, 3, 0, 5])
    conc = np.array([2, 3, 1, 5])
    with pytest.raises(O.BuildError) as e:
        O.build(tt, conc, np.zeros(4), np.full(4, 0.01))
    assert e.value.index == 2 and e.value.code == 2
    with pytest.raises(O.BuildError) as e:
        O.build(np.array([2, 2]), np.array([2, 3]), np.zeros(2), np.full(2, 0.01))
    assert e.value.index == 1 and e.value.code == 4
    with pytest.raises(O.BuildError) as e:
        O.build(np.array([2, 2]), np.array([2, 2]), np.zeros(2), np.array([0.1, float("nan")]))
    assert e.value.index == 1 and e.value.code == 5


# ----------------------------------------- bench configs: C2 and C3 (reference-made goldens)
def _big_tables(gen, g):
    from conftest import records_sha, soa_digest
    from paper_2605_00616_b200.workloads import records_llama, records_sparse

    rec = (records_llama if gen == "c2" else records_sparse)(1_000_000, 0)
    assert records_sha(*rec) == str(g["records_sha256"]), "generator drifted from the golden records"
    tabs = O.build(*rec, canonical=True)
    assert [soa_digest(t.tt, t.conc, t.off, t.samples) for t in tabs] == [str(x) for x in g["canon_digest"]]
    return tabs


def test_c2_oracle_matches_reference(c2_golden):
    """C2 (1M-record Llama-shaped pack): table digests, pools + probabilities of
    2,000 bench-workload keys and 500 out-of-range keys, and the reference
    LatencyOracle's 10,000-draw PCG64 stream with its final state."""
    from conftest import check_full_pools, pool_digests

    g = c2_golden
    tabs = _big_tables("c2", g)
    off, bkt, dist, prob, cdf, tid = O.pools(tabs, g["key_tt"], g["key_conc"], g["key_phase"], 32)
    assert np.array_equal(pool_digests(off, bkt, dist, prob, tid, tabs), g["pool_digest"])
    check_full_pools(off, bkt, dist, prob, tid, tabs, g, "pool_")
    st = O.pcg64_state6(0)
    lat, _ = O.sample_pcg64(tabs, g["seq_tt"], g["seq_conc"], g["seq_phase"], 32, state6=st)
    assert np.array_equal(lat, g["lat_seq"])
    assert st.tolist() == g["final_state"].tolist()


@pytest.mark.parametrize("floor", [32, 256])
def test_c3_oracle_matches_reference(c3_golden, floor):
    """C3 (sparse long-context, 1M records): pools of 800 bench-workload keys and
    200 out-of-range keys at M = 32 and 256."""
    from conftest import check_full_pools, pool_digests

    g = c3_golden
    tabs = _big_tables("c3", g)
    off, bkt, dist, prob, cdf, tid = O.pools(tabs, g["key_tt"], g["key_conc"], g["key_phase"], floor)
    assert np.array_equal(pool_digests(off, bkt, dist, prob, tid, tabs), g[f"m{floor}_digest"])
    check_full_pools(off, bkt, dist, prob, tid, tabs, g, f"m{floor}_")
