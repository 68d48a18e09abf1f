"""Block timeline of the fused (per-level PDL) pass (WS_PROBE build; profiling only).

WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so python scripts/fused_probe.py
Per launch and block: 0 start | 1 records loaded | 2 PDL wait released | 3 end | 4 SM id.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw)
flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED
for _ in range(3):
    dev.run(flags)
torch.cuda.synchronize()
STRIDE = 8 * 2048
NL = 130
probe = torch.zeros(NL * STRIDE, dtype=torch.int64, device="cuda")
_lib.lib().ws_set_probe(dev._h, ctypes.c_void_p(probe.data_ptr()))
for _ in range(2):
    probe.zero_()
    dev.run(flags)
    torch.cuda.synchronize()
P = probe.cpu().numpy().reshape(NL, 2048, 8)
L = dev.n_levels
launches = []
for i in range(NL):
    nb = int((P[i, :, 0] > 0).sum())
    if nb:
        launches.append((i, nb))
t0 = min(P[i, :nb, 0].min() for i, nb in launches)
rows = []
for i, nb in launches:
    a = (P[i, :nb, :4].astype(np.float64) - t0) / 1e3
    rows.append((i, nb, a))
print(f"{len(rows)} probed launches")
gaps = []
for (i, nb, a), (i2, nb2, b) in zip(rows, rows[1:]):
    gaps.append((b[:, 0].min() - a[:, 3].max(),       # next first start - this last end
                 b[:, 2].min() - a[:, 3].max(),       # next first wait release - this last end
                 b[:, 2].max() - a[:, 3].max(),       # next last wait release - this last end
                 np.median(b[:, 1] - b[:, 0]),        # next prologue (start -> records)
                 np.median(a[:, 3] - a[:, 2]),        # this body (median)
                 a[:, 3].max() - a[:, 2].min(),       # this span from first release to last end
                 (b[:, 0] > a[:, 3].max()).mean()))   # fraction of next blocks starting after this last end
g = np.array(gaps)
names = ["next first start - last end", "next first release - last end", "next last release - last end",
         "next prologue p50", "body p50", "release->last end span", "frac next blocks starting late"]
for k, n in enumerate(names):
    print(f"{n:36s} mean {g[:, k].mean():7.2f}  p50 {np.median(g[:, k]):7.2f}  max {g[:, k].max():7.2f}")
span = rows[-1][2][:, 3].max() - rows[0][2][:, 0].min()
print(f"probed span {span:.1f} us over {len(rows)} launches")
for i, nb, a in rows[30:34] + rows[90:94]:
    print(f"launch {i:3d} blocks {nb:3d}: start [{a[:,0].min():8.1f},{a[:,0].max():8.1f}] rec p50 {np.median(a[:,1]-a[:,0]):5.2f} "
          f"release [{a[:,2].min():8.1f},{a[:,2].max():8.1f}] end [{a[:,3].min():8.1f},{a[:,3].max():8.1f}] body p50 {np.median(a[:,3]-a[:,2]):5.2f} max {np.max(a[:,3]-a[:,2]):5.2f}")
