"""Per-block phase timing of the level kernels (WS_PROBE build; profiling only).

WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so python scripts/phase_probe.py [mode]
Launch i of the pass stamps globaltimer at its phase boundaries into
probe[i]; printed: per kernel kind the mean time between consecutive stamps,
the launch span and the gap between launches.
stamps: 0 start | 1 records (+LUT staging) | 2 pdl_wait | 3 end of the block

"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

STRIDE = 8 * 2048      # Launcher::PROBE_STRIDE: 2048 blocks x 8 stamps per launch
raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw)
mode = sys.argv[1] if len(sys.argv) > 1 else "fused"
flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
flags |= {"fused": _lib.RUN_FUSED, "streams": _lib.RUN_TWO_STREAM, "seq": 0}[mode]
for _ in range(3):
    dev.run(flags)
torch.cuda.synchronize()
n_launch = 130
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
    b = P[i][P[i][:, 0] > 0]
    if not len(b):
        continue
    nst = int((b[0] > 0).sum())
    d = np.diff(b[:, :nst], axis=1) / 1e3
    rows.append((i, len(b), (b[:, 0].min() - t_all) / 1e3, (b[:, nst - 1].max() - t_all) / 1e3,
                 d.mean(axis=0), np.median(b[:, 0] - b[:, 0].min()) / 1e3))
for i, nb, s, e, d, st in rows[:2] + rows[30:32] + rows[62:64] + rows[90:92]:
    print(f"launch {i:3d}: {nb:4d} blk start {s:8.2f} end {e:8.2f} span {e - s:6.2f} "
          f"blk-start-p50 {st:5.2f} | " + " ".join(f"{x:5.2f}" for x in d))
spans = np.array([r[3] - r[2] for r in rows])
step = np.array([rows[k + 1][3] - rows[k][3] for k in range(len(rows) - 1)])
print(f"{len(rows)} probed launches: mean span {spans.mean():.2f} us, mean end-to-end step {step.mean():.2f} us")
fw = [r for r in rows if r[0] >= 2 and r[0] < 62]
bw = [r for r in rows if r[0] >= 62]
if fw:
    print("fwd mean phases:", " ".join(f"{x:5.2f}" for x in np.mean([r[4] for r in fw], axis=0)))
if bw:
    print("bwd mean phases:", " ".join(f"{x:5.2f}" for x in np.mean([r[4] for r in bw], axis=0)))
