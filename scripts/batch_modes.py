"""16-corner batch time per run mode (library WS_LIB): fused lockstep vs the
persistent kernel.  python scripts/batch_modes.py [n_corners]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G
from bench import corner_values

NC = int(sys.argv[1]) if len(sys.argv) > 1 else 16
raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw, n_corners=NC)
for k in range(NC):
    dev.set_values(k, **corner_values(raw, k))
base = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_GRAPH
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
for name, f in (("fused", base | _lib.RUN_FUSED), ("persistent", base | _lib.RUN_PERSISTENT)):
    try:
        with torch.cuda.stream(st):
            for _ in range(3):
                dev.run(f, corner=0, n_corners=NC, stream=st)
            ts = []
            for _ in range(10):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                dev.run(f, corner=0, n_corners=NC, stream=st)
                b.record(st)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
        ts.sort()
        print(f"{os.environ.get('WS_LIB', 'default')} {name} n={NC}: {ts[5]:.3f} ms ({ts[5] / NC:.3f}/corner)", flush=True)
    except Exception as e:  # noqa: BLE001
        print(name, "failed:", e)
