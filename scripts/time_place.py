"""C3 placement step timing: pass alone vs wire + pass + position gradients
(CUDA events, graph replay, L2 flushed between steps)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G, placement as PL

raw = G.generate_raw(G.config_c3())
pl = PL.synthetic_placement(raw, seed=3)
dev = ws.DeviceDesign(raw)
timer = PL.PlacementTimer(dev, pl)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
base = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | _lib.RUN_GRAPH
for name, f in (("pass", base), ("wire+pass", base | _lib.RUN_WIRE),
                ("wire+pass+posgrad", base | _lib.RUN_WIRE | _lib.RUN_POSGRAD)):
    for _ in range(3):
        dev.run(f)
    ts = []
    for _ in range(20):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dev.run(f)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{name:20s} {ts[len(ts) // 2]:.4f} ms  launches {dev.last_launch_count()}")
