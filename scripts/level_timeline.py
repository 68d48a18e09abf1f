"""Critical path of the level launches of one fused C3 pass (WS_PROBE build):
for each level launch, relative to the previous launch's last block end T:
how many blocks started after T, the PDL release lag (first wait release -
T), and the phases of the last-finishing block.
WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so python scripts/level_timeline.py"""
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
flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED
torch.cuda.set_stream(torch.cuda.Stream())
s = torch.cuda.current_stream()
for _ in range(3):
    dev.run(flags, stream=s)
torch.cuda.synchronize()
n_launch = dev.last_launch_count() + 2
probe = torch.zeros(n_launch * STRIDE, dtype=torch.int64, device="cuda")
_lib.lib().ws_set_probe(dev._h, ctypes.c_void_p(probe.data_ptr()))
dev.run(flags, stream=s)
torch.cuda.synchronize()
P = probe.view(n_launch, 2048, 8).cpu().numpy().astype(np.int64)
L = dev.n_levels
rows = []
prev_end = None
for i in range(1, 2 * L + 1):
    b = P[i][P[i][:, 0] > 0]
    if not len(b):
        continue
    st, rec, rel, end = (b[:, k].astype(np.float64) for k in (0, 1, 2, 3))
    if prev_end is not None:
        late = int((st > prev_end).sum())
        lag = (rel.min() - prev_end) / 1e3
        j = int(np.argmax(end))
        early = st < prev_end - 5000        # started > 5 us before the previous level's end
        lateb = st > prev_end - 2000        # started in its last 2 us
        rows.append(("fwd" if i <= L else "bwd", len(b), late, lag, (st[j] - prev_end) / 1e3,
                     (rec[j] - st[j]) / 1e3, (rel[j] - max(rec[j], prev_end)) / 1e3, (end[j] - rel[j]) / 1e3,
                     (end.max() - prev_end) / 1e3, np.median(end - rel) / 1e3,
                     np.median((rec - st)[early]) / 1e3 if early.any() else np.nan,
                     np.median((rec - st)[lateb]) / 1e3 if lateb.any() else np.nan,
                     int(early.sum()), int(lateb.sum()),
                     np.median((st - prev_end) / 1e3)))
    prev_end = end.max()
for kind in ("fwd", "bwd"):
    R = np.array([r[1:] for r in rows if r[0] == kind], dtype=np.float64)
    m = np.median(R, axis=0)
    print(f"{kind}: blocks {m[0]:.0f}, started after the previous level's end {m[1]:.0f}, "
          f"PDL release lag {m[2]:.2f} us | last-finishing block: start {m[3]:+.2f}, records {m[4]:.2f}, "
          f"wait after records {m[5]:.2f}, body {m[6]:.2f} | level step {m[7]:.2f} us, median body {m[8]:.2f}")
    m2 = np.nanmedian(R[:, 9:], axis=0)
    print(f"   records phase: blocks started >5 us before the previous end {m2[2]:.0f} (median {m2[0]:.2f} us), "
          f"in its last 2 us {m2[3]:.0f} (median {m2[1]:.2f} us); median start {m2[4]:+.2f} us")
