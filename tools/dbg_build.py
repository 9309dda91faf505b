"""Small GPU table build checked against the oracle (for compute-sanitizer runs)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import emu_oracle as O
from paper_2605_00616_b200 import build_pack_arrays
from paper_2605_00616_b200.workloads import records_llama
n = int(os.environ.get("N", 20000))
rec = records_llama(n, 0)
pack = build_pack_arrays(*rec, num_gpu_blocks=1000, canonical=True)
want = O.build(*rec, canonical=True)
for g, w in zip(pack.soas(), want):
    print(np.array_equal(g.tt, w.tt), np.array_equal(g.off, w.off), np.array_equal(g.samples, w.samples))
