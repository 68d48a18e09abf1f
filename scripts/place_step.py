"""One C3 placement step (wire RC + fwd/bwd pass + position gradients) after
one warm-up step; for ncu launch lists / captures of the placement kernels.
python scripts/place_step.py [n_steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import generator as G, placement as PL

raw = G.generate_raw(G.config_c3())
pl = PL.synthetic_placement(raw, seed=3)
dev = ws.DeviceDesign(raw)
timer = PL.PlacementTimer(dev, pl, graph=False)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    print(timer.step())
torch.cuda.synchronize()
