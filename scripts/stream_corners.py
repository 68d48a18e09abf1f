"""C5 16-corner batch: lockstep (one ws_run over 16 corners) vs S concurrent
streams each running 16/S corners (independent level chains interleave on
the GPU).  python scripts/stream_corners.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G
from bench import corner_values

NC = 16
raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw, n_corners=NC)
for k in range(NC):
    dev.set_values(k, **corner_values(raw, k))
f = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | _lib.RUN_GRAPH
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
main = torch.cuda.Stream()


def one(S):
    per = NC // S
    streams = [torch.cuda.Stream() for _ in range(S)]
    def go():
        ev = torch.cuda.Event()
        ev.record(main)
        ends = []
        for i, st in enumerate(streams):
            st.wait_event(ev)
            dev.run(f, corner=i * per, n_corners=per, stream=st)
            e = torch.cuda.Event()
            e.record(st)
            ends.append(e)
        for e in ends:
            main.wait_event(e)
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        with torch.cuda.stream(main):
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        go()
        b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for S in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8, 16]:
    ms = one(S)
    print(f"streams={S:2d} corners/stream={NC // S:2d}: {ms:.3f} ms per 16-corner batch ({NC / ms * 1e3:.0f} corners/s)",
          flush=True)
