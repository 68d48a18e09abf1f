"""Pass time vs nets per level at fixed depth 60 (fused+graph): is the level
period set by the work per level or by a fixed latency?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

f = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | _lib.RUN_GRAPH
for cells in (40000, 80000, 160000, 315000, 630000, 1260000):
    cfg = G.GeneratorConfig(num_cells=cells, fanout=G.power_law(2.0, 64), depth_target=60, seed=7)
    raw = G.generate_raw(cfg)
    dev = ws.DeviceDesign(raw)
    for _ in range(3):
        dev.run(f)
    ts = []
    for _ in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dev.run(f)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    tasks = dev.topology("level_ptr")
    print(f"cells {cells:8d} pins {raw.n_pins:8d} levels {dev.n_levels} pass {ts[7]:.4f} ms "
          f"per level-step {ts[7] * 1e3 / (2 * dev.n_levels):.2f} us")
    dev.close()
