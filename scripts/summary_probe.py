"""k_summary phase timeline (WS_PROBE build): per block 0 start | 1 leaves done |
2 after the done-counter atomic | 3 end (last block)."""
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
probe = torch.zeros(130 * 8 * 2048, dtype=torch.int64, device="cuda")
_lib.lib().ws_set_probe(dev._h, ctypes.c_void_p(probe.data_ptr()))
dev.run(flags)
torch.cuda.synchronize()
P = probe.cpu().numpy().reshape(130, 2048, 8)
i = dev.last_launch_count() - 1
A = P[i]
nb = int((A[:, 0] > 0).sum())
A = A[:nb, :4].astype(np.float64)
t0 = A[:, 0].min()
A = (A - t0) / 1e3
A[A < -1e6] = np.nan
print(f"launch {i}: {nb} blocks")
print("start  min/max %.2f %.2f" % (np.nanmin(A[:, 0]), np.nanmax(A[:, 0])))
print("leaves done p50/max %.2f %.2f" % (np.nanmedian(A[:, 1]), np.nanmax(A[:, 1])))
print("after atomic max %.2f" % np.nanmax(A[:, 2]))
print("end (last block) %.2f" % np.nanmax(A[:, 3]))
