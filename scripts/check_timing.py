"""Reproduce bench.py's timed loop for one mode and cross-check with host wall time."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw)
flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | int(sys.argv[1])
stream = torch.cuda.current_stream()
flush = torch.empty(2 * 126 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for _ in range(3):
    dev.run(flags, stream=stream)
torch.cuda.synchronize()
for use_flush in (False, True):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(10):
        if use_flush:
            flush.fill_(i)
        evs[i][0].record(stream)
        dev.run(flags, stream=stream)
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / 10
    per = [a.elapsed_time(b) for a, b in evs]
    print(f"flush={use_flush}: event ms/step {sum(per)/10:.4f}  wall ms/step {wall:.4f}  per {['%.3f' % x for x in per[:4]]}")
