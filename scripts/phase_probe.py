"""Per-block phase timing of the level kernels (WS_PROBE build; profiling only).

WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so python scripts/phase_probe.py
Each level-kernel launch i of the pass stamps globaltimer at its phase
boundaries into probe[i]; this prints, per kernel kind, the mean duration of
each phase and the launch-to-launch spacing.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

STRIDE = 8 * 2048
raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw)
mode = sys.argv[1] if len(sys.argv) > 1 else "fused"
flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
flags |= {"fused": _lib.RUN_FUSED, "streams": _lib.RUN_TWO_STREAM, "seq": 0}[mode]
for _ in range(3):
    dev.run(flags)
torch.cuda.synchronize()
n_launch = 140
probe = torch.zeros(n_launch * STRIDE, dtype=torch.int64, device="cuda")
_lib.lib().ws_set_probe(dev._h, ctypes.c_void_p(probe.data_ptr()))
for _ in range(2):
    probe.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dev.run(flags)
    e1.record()
    torch.cuda.synchronize()
print(f"mode {mode}: pass {e0.elapsed_time(e1):.3f} ms, {dev.last_launch_count()} launches")
P = probe.view(n_launch, 2048, 8).cpu().numpy().astype(np.int64)
t_all = P[P > 0].min()
rows = []
for i in range(n_launch):
    blk = P[i]
    used = blk[:, 0] > 0
    if not used.any():
        continue
    b = blk[used]
    nst = int((b[0] > 0).sum())
    d = np.diff(b[:, :nst], axis=1) / 1e3
    rows.append((i, used.sum(), (b[:, 0].min() - t_all) / 1e3, (b[:, nst - 1].max() - t_all) / 1e3,
                 d.mean(axis=0)))
for i, nb, s, e, d in rows[:3] + rows[58:62] + rows[-3:]:
    print(f"launch {i:3d}: {nb:4d} blocks  start {s:8.2f}us end {e:8.2f}us  span {e - s:6.2f}  phases "
          + " ".join(f"{x:5.2f}" for x in d))
spans = np.array([r[3] - r[2] for r in rows])
gaps = np.array([rows[k + 1][2] - rows[k][3] for k in range(len(rows) - 1)])
print(f"{len(rows)} probed launches: mean span {spans.mean():.2f} us, mean gap to next start {gaps.mean():.2f} us")
