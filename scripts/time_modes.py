"""Quick A/B timing: median ms/pass of C3 in the given run modes with the
library named by WS_LIB.  python scripts/time_modes.py fused+graph persistent"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

MODES = {"fused": _lib.RUN_FUSED, "fused+graph": _lib.RUN_FUSED | _lib.RUN_GRAPH,
         "persistent": _lib.RUN_PERSISTENT, "streams+graph": _lib.RUN_TWO_STREAM | _lib.RUN_GRAPH}
raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw)
base = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
out = []
for m in sys.argv[1:] or ["fused+graph"]:
    f = base | MODES[m]
    for _ in range(5):
        dev.run(f)
    ts = []
    for _ in range(30):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dev.run(f)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    out.append(f"{m} {ts[len(ts) // 2]:.4f}")
print(os.environ.get("WS_LIB", "default"), " | ".join(out))
