"""Small runs of every round-2 path, each checked against the CPU oracle, for compute-sanitizer:
cold bitmap dedupe + tile tier, warm k_sweep with a miss list, the small-batch group route,
the two-pass warm path, the sparse group tier at M = 256, the onesweep build, the host pipeline."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import torch
import emu_oracle as O  # checker only
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, build_pack_arrays
from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, queries_sparse, records_llama, records_sparse

def check(orc, tabs, qt, qc, qp, floor, tag, host=False):
    us, ui = explicit_uniforms(len(qt), 9)
    if host:
        lat, sidx = orc.sample_batch(qt, qc, qp, rng="explicit", u_sel=us, u_idx=ui, seed=1)
    else:
        lat, sidx = orc.sample_batch(*(torch.as_tensor(a, device="cuda") for a in (qt, qc, qp)), rng="explicit",
                                     u_sel=torch.as_tensor(us.view(np.int64), device="cuda"),
                                     u_idx=torch.as_tensor(ui.view(np.int32), device="cuda"), seed=1)
        lat, sidx = lat.cpu().numpy(), sidx.cpu().numpy()
    lo, so = O.sample_batch(tabs, qt, qc, qp, floor, mode="explicit", u_sel=us, u_idx=ui, seed=1, threads=8)
    ok = np.array_equal(sidx, so) and np.array_equal(lat, lo)
    print(tag, "ok" if ok else "MISMATCH", flush=True)
    assert ok

n = int(os.environ.get("N", 60_000))
rec = records_llama(n, 0)  # onesweep build (several tiles per pass) + segmentation
pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
tabs = O.build(*rec, canonical=True)
for g, w in zip(pack.soas(), tabs):
    assert np.array_equal(g.tt, w.tt) and np.array_equal(g.off, w.off) and np.array_equal(g.samples, w.samples)
print("build ok", flush=True)
orc = LatencyOracle(pack, OracleConfig(reliability_floor=32))
qt, qc, qp = queries_llama(40_000, 1)
check(orc, tabs, qt, qc, qp, 32, "cold bitmap + tile tier")
qt2, qc2, qp2 = queries_llama(40_000, 2)
qt2[::5] += 3000  # out-of-grid / hash keys among them
check(orc, tabs, qt2, qc2, qp2, 32, "warm, misses")          # two-pass (many new keys last time) or sweep
check(orc, tabs, qt2, qc2, qp2, 32, "warm, no misses")       # decided from the last chunk
qt3, qc3, qp3 = queries_llama(40_000, 3)
check(orc, tabs, qt3, qc3, qp3, 32, "warm, few new keys")    # small-batch group route
orc.flush()
check(orc, tabs, qt3, qc3, qp3, 32, "host pipeline", host=True)
srec = records_sparse(n, 0)
spack = build_pack_arrays(*srec, num_gpu_blocks=1000, canonical=True)
stabs = O.build(*srec, canonical=True)
sorc = LatencyOracle(spack, OracleConfig(reliability_floor=256))
st, sc, sp = queries_sparse(3_000, 1)
check(sorc, stabs, st, sc, sp, 256, "sparse M=256 group tier")
print("all paths ok")
