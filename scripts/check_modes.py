"""Time each run mode on C3 and check its results against the fused per-level mode."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

raw = G.generate_raw(G.config_c3() if len(sys.argv) < 2 else getattr(G, "config_" + sys.argv[1])())
dev = ws.DeviceDesign(raw)
base = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
FIELDS = ("arrival", "required", "slack", "lse_arrival", "d_arc", "d_edge", "adjoint")
dev.run(base | _lib.RUN_FUSED)
torch.cuda.synchronize()
ref = {f: dev.get(f) for f in FIELDS}
refs = dev.summary()
s = torch.cuda.current_stream()
for name, fl in [("fused", base | _lib.RUN_FUSED), ("fused+graph", base | _lib.RUN_FUSED | _lib.RUN_GRAPH),
                 ("persistent", base | _lib.RUN_PERSISTENT),
                 ("persistent+graph", base | _lib.RUN_PERSISTENT | _lib.RUN_GRAPH),
                 ("streams+graph", base | _lib.RUN_TWO_STREAM | _lib.RUN_GRAPH),
                 ("hard persistent", _lib.RUN_HARD | _lib.RUN_PERSISTENT)]:
    for f in FIELDS:
        dev.tensor(f).zero_()
    for _ in range(3):
        dev.run(fl)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        dev.run(fl, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ok = all(np.array_equal(dev.get(f), ref[f]) for f in (FIELDS if fl & _lib.RUN_LSE else FIELDS[:3]))
    print(f"{name:18s} {np.median(ts):8.4f} ms (min {min(ts):.4f})  results equal: {ok}  launches {dev.last_launch_count()}  summary {dev.summary() == refs}")
