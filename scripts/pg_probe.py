"""Per-phase timing of the fused position-gradient backward levels (WS_PROBE
build; profiling only).  One C3 placement step (graph off) with probes:
WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so python scripts/pg_probe.py
stamps: 0 start | 1 records+prefetch issue | 2 pdl_wait | 5 member phase |
        6 bwd net phase + sweep member terms | 7 sweep net records | 3 end"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G, placement as PL

STRIDE = 8 * 2048      # Launcher::PROBE_STRIDE: 2048 blocks x 8 stamps per launch
raw = G.generate_raw(G.config_c3())
pl = PL.synthetic_placement(raw, seed=3)
dev = ws.DeviceDesign(raw)
timer = PL.PlacementTimer(dev, pl, graph=False)
for _ in range(3):
    timer.step()
torch.cuda.synchronize()
n_launch = 130
probe = torch.zeros(n_launch * STRIDE, dtype=torch.int64, device="cuda")
_lib.lib().ws_set_probe(dev._h, ctypes.c_void_p(probe.data_ptr()))
probe.zero_()
timer.step()
torch.cuda.synchronize()
P = probe.view(n_launch, 2048, 8).cpu().numpy().astype(np.int64)
order = [0, 1, 2, 5, 6, 7, 3]
acc = []
for i in range(n_launch):
    b = P[i][P[i][:, 0] > 0]
    if not len(b) or not (b[:, 5] > 0).any():
        continue
    b = b[b[:, 5] > 0]
    t0 = b[:, 0].min()
    ph = [(b[:, order[k + 1]] - b[:, order[k]]) / 1e3 for k in range(len(order) - 1)]
    acc.append([np.median(x) for x in ph] + [np.max(x) for x in ph] + [(b[:, 3].max() - t0) / 1e3, len(b)])
A = np.array(acc)
names = ["rec", "wait", "members", "bwdnet+pgM", "pgB", "pgC+D"]
k = len(names)
print(f"{len(A)} PG backward launches; per launch, median over levels:")
print("  median block phase (us): " + " ".join(f"{n}={v:.2f}" for n, v in zip(names, np.median(A[:, :k], axis=0))))
print("  slowest block phase (us): " + " ".join(f"{n}={v:.2f}" for n, v in zip(names, np.median(A[:, k:2 * k], axis=0))))
print(f"  launch span (first start -> last end) {np.median(A[:, 2 * k]):.2f} us, blocks {np.median(A[:, 2 * k + 1]):.0f}")
