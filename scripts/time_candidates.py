"""16 placement candidates of C3 in one ws_run (wire + pass + fused sweep,
blockIdx.y = candidate), graph replay: ms per batch (library WS_LIB).
python scripts/time_candidates.py [n]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import generator as G, placement as PL

NC = int(sys.argv[1]) if len(sys.argv) > 1 else 16
raw = G.generate_raw(G.config_c3())
pl = PL.synthetic_placement(raw, seed=3)
dev = ws.DeviceDesign(raw, n_corners=NC)
timers = []
for c in range(NC):
    rng = np.random.default_rng(2000 + c)
    xy = pl.xy + 0.5 * rng.standard_normal(pl.cell_xy.shape)[pl.cell_of_pin]
    timers.append(PL.PlacementTimer(dev, PL.Placement(xy, pl.res0, pl.cap0, pl.wire, pl.cell_of_pin, pl.cell_xy,
                                                      pl.pin_offset), corner=c))
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(5):
        dev.run(timers[0].flags, corner=0, n_corners=NC, gamma=timers[0].gamma, stream=st)
    ts = []
    for _ in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        dev.run(timers[0].flags, corner=0, n_corners=NC, gamma=timers[0].gamma, stream=st)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
print(os.path.basename(os.environ.get("WS_LIB", "default")), f"{NC} candidates: {np.median(ts):.3f} ms per batch",
      flush=True)
