"""candidate_batch timing in isolation and after corner_batch (bench order)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G
raw = G.generate_raw(G.config_c3())
print("alone", bench.candidate_batch(raw, 0, 1, steps=6)["ms_per_batch"])
flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | _lib.RUN_GRAPH
dev = ws.DeviceDesign(raw, n_corners=2)
for _ in range(5):
    dev.run(flags)
print("after main dev", bench.candidate_batch(raw, 0, 1, steps=6)["ms_per_batch"])
print("corner batch", bench.corner_batch(raw, 0, 1, flags, steps=6)["ms_per_batch"])
print("after corner batch", bench.candidate_batch(raw, 0, 1, steps=6)["ms_per_batch"])
