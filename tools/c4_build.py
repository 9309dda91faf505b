"""One warm-up + N canonical 100M-record table builds (config 4 input), for ncu."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2605_00616_b200.capture import records_device
from paper_2605_00616_b200.device import DeviceTables
dev = records_device(int(os.environ.get("N", 100_000_000)), seed=100)
for _ in range(int(os.environ.get("BUILDS", 2))):
    t = DeviceTables.build(*dev, canonical=True)
    del t
torch.cuda.synchronize()
