"""Per-level timeline of the persistent pass kernel (WS_PROBE build; profiling only).

WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so python scripts/persist_probe.py
stamps per (level, block): 0 level start (barrier left) | 1 tasks done | 2 next records prefetched
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
flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_PERSISTENT
for _ in range(3):
    dev.run(flags)
torch.cuda.synchronize()
L = dev.n_levels
probe = torch.zeros(2 * 2 * L * 2048 * 4 + 2048 * 4, dtype=torch.int64, device="cuda")
_lib.lib().ws_set_probe(dev._h, ctypes.c_void_p(probe.data_ptr()))
for _ in range(2):
    probe.zero_()
    dev.run(flags)
    torch.cuda.synchronize()
flat = probe.cpu().numpy().astype(np.int64)
A = flat[: 2 * L * 2048 * 4].reshape(2 * L, 2048, 4)
ncta = int((A[0, :, 0] > 0).sum())
P = A[:, :ncta, :3]
B = flat[2 * L * 2048 * 4:4 * L * 2048 * 4].reshape(2 * L, 2048, 4)[:, :ncta]
t0 = P[P > 0].min()
start = (P[:, :, 0] - t0) / 1e3
done = (P[:, :, 1] - t0) / 1e3
pref = (P[:, :, 2] - t0) / 1e3
print(f"{ncta} blocks, {2 * L} levels, pass span {(pref.max() - start.min()):.1f} us")
for name, rng in (("fwd", range(0, L)), ("bwd", range(2 * L - 1, L - 1, -1))):
    work = np.array([np.median(done[li] - start[li]) for li in rng])
    worst = np.array([np.max(done[li] - start[li]) for li in rng])
    prefetch = np.array([np.median(pref[li] - done[li]) for li in rng])
    lv = list(rng)
    bar = np.array([start[lv[i + 1]].min() - pref[lv[i]].max() for i in range(len(lv) - 1)])
    skew = np.array([start[li].max() - start[li].min() for li in rng])
    print(f"{name}: per level  task p50 {work.mean():5.2f} us  task max {worst.mean():5.2f} us  "
          f"prefetch {prefetch.mean():5.2f} us  barrier(last arrive->first leave) {bar.mean():5.2f} us  "
          f"start skew {skew.mean():5.2f} us")

# task-body phases (block 0's first task of each level): start -> gathered -> arc -> net -> done
bs = B.astype(np.float64)
st = P[:, :, 0].astype(np.float64)
dn = P[:, :, 1].astype(np.float64)
for name, rng in (("fwd", range(0, L)), ("bwd", range(L, 2 * L))):
    rows = []
    for li in rng:
        ok = (bs[li, :, 0] > 0)
        if not ok.any():
            continue
        g = bs[li, ok, 0] - st[li, ok]
        a = bs[li, ok, 1] - bs[li, ok, 0]
        if name == "fwd":
            n = bs[li, ok, 2] - bs[li, ok, 1]
            e = dn[li, ok] - bs[li, ok, 2]
            rows.append((np.median(g), np.median(a), np.median(n), np.median(e)))
        else:
            e = dn[li, ok] - bs[li, ok, 1]
            rows.append((np.median(g), np.median(a), np.median(e)))
    if not rows:
        print(f"{name}: no body stamps (nonzero B entries: {(B > 0).sum()})")
        continue
    r = np.mean(rows, axis=0) / 1e3
    label = "gathers | arc | net+LSE | weights+members" if name == "fwd" else "gathers | members | nets"
    print(f"{name} body phases ({label}): " + " ".join(f"{x:5.2f}" for x in r) + " us")

K = flat[4 * L * 2048 * 4:].reshape(2048, 4)[:ncta].astype(np.float64)
ev = cuda_ms = None
s0 = K[:, 0].min()
print("kernel phases (us from first block start): start max %.1f | RC done p50 %.1f max %.1f | fwd done max %.1f | bwd done max %.1f" % (
    (K[:, 0].max() - s0) / 1e3, (np.median(K[:, 1]) - s0) / 1e3, (K[:, 1].max() - s0) / 1e3,
    (K[:, 2].max() - s0) / 1e3, (K[:, 3].max() - s0) / 1e3))
st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
st.record(); dev.run(flags); en.record(); torch.cuda.synchronize()
print("one pass (probe build, events): %.1f us" % (st.elapsed_time(en) * 1e3))
