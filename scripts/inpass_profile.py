"""Per-kernel-class in-pass time of the fused C3 pass -> profiles/inpass_<R>.json.

WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so python scripts/inpass_profile.py r02 [launches.csv]

The WS_PROBE build stamps %globaltimer at the start and end of every block
of every level kernel.  Because of programmatic dependent launch the level
kernels overlap (level l+1's prologue runs under level l), so serialised
per-kernel durations (ncu, CUDA events between launches) over-count.  Here a
level launch's in-pass share is its critical-path increment: the time from
the previous level launch's last block end to its own last block end; the
first level launch's increment starts at the RC kernel's end, taken as the
first level launch's last block end minus its own span.  The RC kernel and
the tail (k_fin_summary) are not probed: their durations come from the ncu
launch list of the same pass (serialised, ~= in-pass: RC streams alone,
the tail runs after the last level).  The classes are then compared with the
pass's CUDA-event time.
"""
import csv
import ctypes
import json
import os
import statistics
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

R = sys.argv[1] if len(sys.argv) > 1 else "r02"
STRIDE = 8 * 2048       # Launcher::PROBE_STRIDE
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
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
passes = []
for it in range(7):
    probe.zero_()
    flush.fill_(it)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    dev.run(flags, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    P = probe.view(n_launch, 2048, 8).cpu().numpy().astype(np.int64)
    ends, spans, idx = [], [], []
    for i in range(1, 2 * dev.n_levels + 1):      # launch 0 is RC; 1..L forward, L+1..2L backward
        b = P[i][P[i][:, 0] > 0]
        if not len(b):
            continue
        # slots: 0 start | 1 records | 2 PDL wait released | 3 end | 4 SM id
        idx.append(i)
        ends.append(b[:, 3].max())
        spans.append((b[:, 3].max() - b[:, 0].min()) / 1e3)
    passes.append((e0.elapsed_time(e1) * 1e3, ends, spans))
L = dev.n_levels
# launches probed in order: L forward levels then L backward levels
tot_us = statistics.median(p[0] for p in passes)
fw, bw = [], []
for t_us, ends, spans in passes:
    assert len(ends) == 2 * L, (len(ends), L)
    inc = [spans[0]] + [(ends[i] - ends[i - 1]) / 1e3 for i in range(1, len(ends))]
    fw.append(sum(inc[:L]))
    bw.append(sum(inc[L:]))
rc_us = tail_us = None
if len(sys.argv) > 2 and os.path.exists(sys.argv[2]):
    rows = list(csv.reader(open(sys.argv[2])))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    sc = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    rcs, tails = [], []
    for r in rows[hi + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        v = float(r[vi].replace(",", "")) * sc.get(r[ui], 1.0)
        if "k_rc_flat" in r[ki]:
            rcs.append(v)
        elif "k_fin_summary" in r[ki]:
            tails.append(v)
    rc_us = statistics.median(rcs) if rcs else None
    tail_us = statistics.median(tails) if tails else None
fwd_us, bwd_us = statistics.median(fw), statistics.median(bw)
classes = [
    {"kernel": "k_fwd<1,1> (fwd + LSE level)", "launches_per_pass": L, "in_pass_us": round(fwd_us, 1),
     "avg_step_us": round(fwd_us / L, 2), "share": round(fwd_us / tot_us, 4)},
    {"kernel": "k_bwd<1,1> (bwd + grad level)", "launches_per_pass": L, "in_pass_us": round(bwd_us, 1),
     "avg_step_us": round(bwd_us / L, 2), "share": round(bwd_us / tot_us, 4)},
]
if rc_us is not None:
    classes.append({"kernel": "k_rc_flat (+free pins)", "launches_per_pass": 1, "in_pass_us": round(rc_us, 1),
                    "share": round(rc_us / tot_us, 4), "source": "ncu launch list (serialised)"})
if tail_us is not None:
    classes.append({"kernel": "k_fin_summary", "launches_per_pass": 1, "in_pass_us": round(tail_us, 1),
                    "share": round(tail_us / tot_us, 4), "source": "ncu launch list (serialised)"})
ssum = sum(c["in_pass_us"] for c in classes)
out = {"round": R, "what": "in-pass time per kernel class of one fused C3 pass (no graph): level launches "
                          "from WS_PROBE globaltimer block stamps as critical-path increments, RC and "
                          "tail from the ncu launch list; median of 7 passes",
       "pass_us_cuda_events": round(tot_us, 1), "classes_sum_us": round(ssum, 1),
       "classes_over_pass": round(ssum / tot_us, 4), "classes": classes}
for d in ("profiles", "gpurun_out"):     # gpurun_out/ is what travels back from a GPU box
    os.makedirs(os.path.join(HERE, d), exist_ok=True)
    json.dump(out, open(os.path.join(HERE, d, f"inpass_{R}.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
