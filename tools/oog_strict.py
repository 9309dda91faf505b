"""Strict out-of-grid pool repro: every round's pools vs the CPU oracle (not vs round 0).

Env: N keys (20000), ROUNDS (20), GEN=llama|sparse, FLOOR (32), MODE=pools|sample,
EMU_LIB_PATH=<libemu_b200_check.so> to count device invariant failures.
"""
import ctypes, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import emu_oracle as O  # checker only
from paper_2605_00616_b200 import LatencyOracle, OracleConfig, build_pack_arrays, _lib
from paper_2605_00616_b200.workloads import records_llama, records_sparse

gen = os.environ.get("GEN", "llama")
floor = int(os.environ.get("FLOOR", 32))
n = int(os.environ.get("N", 20000))
rounds = int(os.environ.get("ROUNDS", 20))
rec = (records_sparse if gen == "sparse" else records_llama)(1_000_000, 3)
pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
tabs = O.build(*rec, canonical=True)
rng = np.random.default_rng(int(os.environ.get("SEED", 5)))
hi_t = 140_000 if gen == "sparse" else 3000
kt = rng.integers(-10, hi_t, n).astype(np.int32)
kc = rng.integers(-3, 300, n).astype(np.int32)
kp = rng.integers(0, 2, n).astype(np.uint8)
t0 = time.time()
cache = "/tmp/oog_want_%s_%d_%d_%s.npz" % (gen, floor, n, os.environ.get("SEED", 5))
if os.path.exists(cache):
    z = np.load(cache)
    want = [z["a%d" % i] for i in range(6)]
else:
    want = O.pools(tabs, kt, kc, kp, floor)
    np.savez(cache, **{"a%d" % i: a for i, a in enumerate(want)})
print("oracle pools %.1fs" % (time.time() - t0), flush=True)
# the sample path (cache mode): 200k draws over the same keys, explicit uniforms
Qs = int(os.environ.get("QS", 200_000))
qi = rng.integers(0, n, Qs)
us = rng.integers(0, 2**63, Qs, dtype=np.uint64)
ui = rng.integers(0, 2**32, Qs, dtype=np.uint64).astype(np.uint32)
want_s = O.sample_batch(tabs, kt[qi], kc[qi], kp[qi], floor, mode="explicit", u_sel=us, u_idx=ui, threads=8)
chk = getattr(_lib.lib(), "emu_check_read", None)
bad_rounds = 0
for r in range(rounds):
    orc = LatencyOracle(pack, OracleConfig(reliability_floor=floor))
    try:
        got = orc.pools(kt, kc, kp)
        err = None
    except Exception as e:  # noqa: BLE001
        got, err = None, str(e)
    nchk = -1
    if chk is not None:
        v = ctypes.c_ulonglong(0)
        chk(ctypes.byref(v))
        nchk = int(v.value)
    ok = err is None and all(np.array_equal(a, b) for a, b in zip(got[:5], want[:5]))
    if ok:
        try:
            lat, sidx = orc.sample_batch(kt[qi], kc[qi], kp[qi], rng="explicit", u_sel=us, u_idx=ui)
            ok = np.array_equal(lat, want_s[0]) and np.array_equal(sidx, want_s[1])
            if not ok:
                err = "sample_batch differs at %d queries" % int((sidx != want_s[1]).sum())
        except Exception as e:  # noqa: BLE001
            ok, err = False, "sample_batch: " + str(e)
    if not ok:
        bad_rounds += 1
        msg = err
        if err is None:
            K0, K1 = np.diff(want[0]), np.diff(got[0])
            bad = np.flatnonzero(K0 != K1)
            msg = "K differs for %d keys; first %s" % (len(bad), [(int(kt[i]), int(kc[i]), int(kp[i]), int(K0[i]), int(K1[i])) for i in bad[:6]])
        print("round", r, "MISMATCH", msg, "checks", nchk, flush=True)
    else:
        print("round", r, "ok checks", nchk, flush=True)
    del orc
print("STRICT", gen, "N", n, "rounds", rounds, "bad", bad_rounds)
sys.exit(1 if bad_rounds else 0)
