"""A/B one library build (WS_LIB): C3 parity against the oracle (hard pass
bit-exact, gradients <= 1e-4) plus C3 single-pass and 16-corner-batch
timings (fused + graph, L2 flushed between passes).
python scripts/ab_variants.py [--no-check] [--batch N]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G
from bench import corner_values

NB = int(sys.argv[sys.argv.index("--batch") + 1]) if "--batch" in sys.argv else 16
raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw, n_corners=max(NB, 1))
for k in range(1, NB):
    dev.set_values(k, **corner_values(raw, k))
f = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | _lib.RUN_GRAPH
name = os.path.basename(os.environ.get("WS_LIB", "default"))
st = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")


def timeit(n, reps=15):
    with torch.cuda.stream(st):
        for _ in range(3):
            dev.run(f, corner=0, n_corners=n, stream=st)
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            dev.run(f, corner=0, n_corners=n, stream=st)
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


ok = "unchecked"
if "--no-check" not in sys.argv:
    from oracle import oracle as O
    gamma = dev.run(f, corner=0, n_corners=1, stream=st)
    torch.cuda.synchronize()
    ofl = O.flatten_raw(raw)
    ost = O.run_engine(ofl)
    bad = [x for x in ("load", "net_delay", "impulse", "slew", "arrival", "required", "slack", "arc_delay")
           if not np.array_equal(dev.get(x), getattr(ost, x))]
    og = O.timing_gradients(ofl, ost, gamma=gamma)
    for x in ("lse_arrival", "arc_weights", "d_arc", "d_edge", "adjoint"):
        a, b = dev.get(x), getattr(og, x)
        if not np.allclose(a, b, rtol=1e-4, atol=1e-12 * max(1.0, float(np.abs(b).max()))):
            bad.append(x)
    tns, wns, loss = dev.summary()
    if tns != O.tns(ost, ofl) or wns != O.wns(ost, ofl):
        bad.append("tns/wns")
    ok = "parity OK" if not bad else "PARITY FAIL " + ",".join(bad)
t1 = timeit(1)
tb = timeit(NB, reps=8) if NB > 1 else float("nan")
print(f"{name:40s} {ok:12s} C3 {t1:.4f} ms/pass | {NB}-corner batch {tb:.3f} ms ({tb / NB:.3f}/corner) "
      f"launches {dev.last_launch_count()}", flush=True)
