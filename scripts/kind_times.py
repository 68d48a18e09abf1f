"""Per-kind event times of one fused C3 pass (WS_RUN_TIMED: an event after
every launch, which serialises the PDL overlap): library WS_LIB.
python scripts/kind_times.py"""
import os
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw)
f = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | _lib.RUN_TIMED
for _ in range(3):
    dev.run(f)
acc = defaultdict(list)
for _ in range(5):
    dev.run(f)
    torch.cuda.synchronize()
    per = defaultdict(float)
    for kind, level, ms in dev.kernel_times():
        per[kind] += ms
    for k, v in per.items():
        acc[k].append(v)
names = {0: "rc", 1: "fwd", 2: "bwd", 5: "tail"}
print(os.path.basename(os.environ.get("WS_LIB", "default")),
      " ".join(f"{names.get(k, k)}={np.median(v):.3f}ms" for k, v in sorted(acc.items())))
