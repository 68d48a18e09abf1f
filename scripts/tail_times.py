"""Warm per-launch deltas (RUN_TIMED sequential pass) of the non-level kernels on C3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw)
f = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_TIMED
for _ in range(3):
    dev.run(f)
kt = dev.kernel_times()
names = {0: "net_rc", 1: "fwd", 2: "bwd", 3: "lse", 4: "grad", 5: "other"}
print("first entries:", [(names[k], l, round(ms * 1e3, 1)) for k, l, ms in kt[:3]])
print("last entries:", [(names[k], l, round(ms * 1e3, 1)) for k, l, ms in kt[-4:]])
import collections
agg = collections.defaultdict(float)
for k, l, ms in kt:
    agg[names[k]] += ms
print({k: round(v * 1e3, 1) for k, v in agg.items()})
