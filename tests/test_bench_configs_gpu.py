"""The CUDA path at the bench configs against goldens the reference made (B200 only).

C2 (BASELINE configs[1]) and C3 (configs[2]) goldens come from the unmodified
reference (tests/golden/make_golden_big.py); tests/test_oracle_cpu.py pins the
CPU restatement to the same files.  Here the GPU build, the GPU pools and the
device PCG64 replay are compared with them directly, and a 1M-query contiguous
window of the exact bench workload (explicit uniforms) with the CPU oracle.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import emu_oracle as O
from conftest import check_full_pools, pool_digests, records_sha, soa_digest
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, build_pack_arrays
from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, records_llama, records_sparse

pytestmark = pytest.mark.gpu


def _pack(gen, g):
    rec = (records_llama if gen == "c2" else records_sparse)(1_000_000, 0)
    assert records_sha(*rec) == str(g["records_sha256"])
    pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)  # GPU build
    soas = pack.soas()
    assert [soa_digest(s.tt, s.conc, s.off, s.samples) for s in soas] == [str(x) for x in g["canon_digest"]]
    return pack, soas, rec


@pytest.fixture(scope="module")
def c2(c2_golden):
    return _pack("c2", c2_golden)


def test_c2_pools_match_reference(c2, c2_golden):
    pack, soas, _ = c2
    g = c2_golden
    orc = LatencyOracle(pack, OracleConfig(reliability_floor=32))
    off, bkt, dist, prob, cdf, tid = orc.pools(g["key_tt"], g["key_conc"], g["key_phase"])
    assert np.array_equal(pool_digests(off, bkt, dist, prob, tid, soas), g["pool_digest"])
    check_full_pools(off, bkt, dist, prob, tid, soas, g, "pool_")


def test_c2_pcg64_stream_matches_reference(c2, c2_golden):
    """The reference LatencyOracle's first 10,000 bench-workload draws (seed 0),
    replayed on the device: half batched, half through the per-step call."""
    pack, _, _ = c2
    g = c2_golden
    orc = LatencyOracle(pack, OracleConfig(reliability_floor=32, rng_seed=0))
    n = 5000
    lat, _ = orc.sample_batch(g["seq_tt"][:n], g["seq_conc"][:n], g["seq_phase"][:n], rng="pcg64")
    lat = np.asarray(lat.cpu() if hasattr(lat, "cpu") else lat)
    steps = [orc(int(a), int(b), int(c)) for a, b, c in zip(g["seq_tt"][n:], g["seq_conc"][n:], g["seq_phase"][n:])]
    assert np.array_equal(np.concatenate([lat, np.array(steps)]), g["lat_seq"])
    st = orc.rng_state()
    s = st["state"]
    assert [s["state"] >> 64, s["state"] & (2**64 - 1), s["inc"] >> 64, s["inc"] & (2**64 - 1), st["has_uint32"],
            st["uinteger"]] == g["final_state"].tolist()


def test_c2_bench_workload_window_matches_oracle(c2):
    """bench.py's exact step (10M queries of queries_llama(10M, 1), explicit
    uniforms explicit_uniforms(10M, 1000), cold cache) on the device; the
    contiguous window [4M, 5M) checked query by query against the CPU oracle."""
    pack, soas, _ = c2
    Q = 10_000_000
    qt, qc, qp = queries_llama(Q, 1)
    us, ui = explicit_uniforms(Q, 1000)
    orc = LatencyOracle(pack, OracleConfig(reliability_floor=32))
    d = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    lat, sidx = orc.sample_batch(d(qt), d(qc), d(qp), rng="explicit", u_sel=d(us.view(np.int64)),
                                 u_idx=d(ui.view(np.int32)), seed=1)
    lo, hi = 4_000_000, 5_000_000
    tabs = [O.Table(s.tt, s.conc, s.off, s.samples) for s in soas]
    want_lat, want_sidx = O.sample_batch(tabs, qt[lo:hi], qc[lo:hi], qp[lo:hi], 32, mode="explicit",
                                         u_sel=us[lo:hi], u_idx=ui[lo:hi], threads=16)
    assert np.array_equal(sidx[lo:hi].cpu().numpy(), want_sidx)
    assert np.array_equal(lat[lo:hi].cpu().numpy(), want_lat)


@pytest.fixture(scope="module")
def c3(c3_golden):
    return _pack("c3", c3_golden)


@pytest.mark.parametrize("floor", [32, 256])
def test_c3_pools_match_reference(c3, c3_golden, floor):
    pack, soas, _ = c3
    g = c3_golden
    orc = LatencyOracle(pack, OracleConfig(reliability_floor=floor))
    off, bkt, dist, prob, cdf, tid = orc.pools(g["key_tt"], g["key_conc"], g["key_phase"])
    assert np.array_equal(pool_digests(off, bkt, dist, prob, tid, soas), g[f"m{floor}_digest"])
    check_full_pools(off, bkt, dist, prob, tid, soas, g, f"m{floor}_")


def test_c4_100m_build_matches_oracle():
    """Config 4 at full size: the 100M-record canonical 3-table build (records
    from the device generator G, the bench_configs c4 input) against the CPU
    restatement of build_pack + save_pack's order, table by table (digest of
    keys, offsets and samples)."""
    from paper_2605_00616_b200.capture import records_device
    from paper_2605_00616_b200.device import DeviceTables

    dev = records_device(100_000_000, seed=100)
    got = DeviceTables.build(*dev, canonical=True).to_host()
    rec = [d.cpu().numpy() for d in dev]
    del dev
    torch.cuda.empty_cache()
    want = O.build(*rec, canonical=True)
    for g, w in zip(got, want):
        assert len(g.tt) == len(w.tt) and len(g.samples) == len(w.samples) == int(w.off[-1])
        assert soa_digest(g.tt, g.conc, g.off, g.samples) == soa_digest(w.tt, w.conc, w.off, w.samples)
