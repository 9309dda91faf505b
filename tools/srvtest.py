import os, sys, subprocess
code = r'''
import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from paper_2605_00616_b200 import OracleConfig, OracleQuery, sample_latency
from paper_2605_00616_b200.profile import Bucket, StepPhase
from test_reference_suite_gpu import make_pack, anchored
near = [Bucket(600, 50, [0.010] * 10), Bucket(700, 50, [0.020] * 10), Bucket(900, 50, [0.040] * 10)]
pack = make_pack(anchored(near), [])
cfg = OracleConfig(reliability_floor=30, shepard_power=2.0)
g = np.random.default_rng(20240810)
seq = [sample_latency(pack, OracleQuery(500, 50, StepPhase.DECODE_ONLY), cfg, g) for _ in range(100_000)]
np.save(sys.argv[1], np.array(seq))
'''
for env in ("1", "0"):
    subprocess.run([sys.executable, "-c", code, f"/tmp/seq{env}.npy"], env=dict(os.environ, EMU_STEP_SERVER=env), check=True)
import numpy as np
a, b = np.load("/tmp/seq1.npy"), np.load("/tmp/seq0.npy")
d = np.flatnonzero(a != b)
print("mismatches", len(d), "first", d[:10], a[d[:5]], b[d[:5]])
