"""RC scheme ablation on C3: the streaming
(member, cond) RC kernel vs the CTE-scheme kernel; RC-only and whole-pass
times (CUDA events, median of 20)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

raw = G.generate_raw(G.config_c3())
for scheme in (sys.argv[1:] or ["flat", "cte", "pin"]):
    os.environ["WS_RC_SCHEME"] = scheme
    dev = ws.DeviceDesign(raw)
    out = []
    for name, f in (("pass", _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | _lib.RUN_GRAPH),
                    ("timed-seq", _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_TIMED)):
        ts, rc = [], []
        for i in range(21):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dev.run(f)
            b.record()
            torch.cuda.synchronize()
            if i:
                ts.append(a.elapsed_time(b))
                if f & _lib.RUN_TIMED:
                    rc.append(sum(ms for k, lv, ms in dev.kernel_times() if k == 0))
        ts.sort()
        out.append(f"{name} {ts[10]:.4f} ms")
        if rc:
            rc.sort()
            out.append(f"RC kernel {rc[10] * 1e3:.1f} us")
    print(scheme, " | ".join(out))
    dev.close()
