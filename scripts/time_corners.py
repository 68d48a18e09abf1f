"""ms per pass of n corners batched in one ws_run (C5 corner values), library WS_LIB.
python scripts/time_corners.py 1 4 16"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G
from bench import corner_values

raw = G.generate_raw(G.config_c3())
ns = [int(x) for x in sys.argv[1:]] or [1, 16]
dev = ws.DeviceDesign(raw, n_corners=max(ns))
for k in range(max(ns)):
    dev.set_values(k, **corner_values(raw, k))
f = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | _lib.RUN_GRAPH
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
out = []
for n in ns:
    for _ in range(3):
        dev.run(f, corner=0, n_corners=n)
    ts = []
    for _ in range(10):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dev.run(f, corner=0, n_corners=n)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    out.append(f"{n}: {ts[len(ts) // 2]:.3f} ms ({ts[len(ts) // 2] / n:.3f}/corner)")
print(os.environ.get("WS_LIB", "default"), " | ".join(out))
