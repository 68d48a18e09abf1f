"""One graph-replayed C3 fused pass inside a cudaProfilerStart/Stop range,
for ncu range replay (per-pass DRAM traffic of the real, PDL-overlapped
pass):

ncu --replay-mode range --profile-from-start off --cache-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --csv --log-file gpurun_out/traffic_range_r02.csv python scripts/pass_range.py [graph]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

graph = len(sys.argv) < 2 or sys.argv[1] != "nograph"
raw = G.generate_raw(G.config_c3())
dev = ws.DeviceDesign(raw)
flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | (_lib.RUN_GRAPH if graph else 0)
torch.cuda.set_stream(torch.cuda.Stream())
s = torch.cuda.current_stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
for _ in range(3):
    dev.run(flags, stream=s)
flush.fill_(1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
dev.run(flags, stream=s)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("pass launches", dev.last_launch_count(), "summary", dev.summary())
