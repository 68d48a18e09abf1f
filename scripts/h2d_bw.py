"""Pinned H2D bandwidth: one stream vs chunks over several streams (138 MB)."""
import torch

n = 137871360 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunks = [(i * n // ns, (i + 1) * n // ns) for i in range(ns)]
    ts = []
    for it in range(6):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s, (a, b) in zip(streams, chunks):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        if it:
            ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(f"{ns} streams: {ms:.3f} ms, {n * 8 / ms / 1e6:.1f} GB/s")
