"""profiles/traffic_<R>.json from gpurun_out/traffic_apprange_<R>.csv: the DRAM
bytes of ONE graph-replayed fused C3 pass measured by ncu app-range replay
(scripts/pass_range.py; ncu --replay-mode app-range --cache-control none)."""
import csv
import json
import os
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r02"
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(open(os.path.join(HERE, "gpurun_out", f"traffic_apprange_{R}.csv"))))
hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
h = rows[hi]
vals = {r[h.index("Metric Name")]: float(r[h.index("Metric Value")].replace(",", ""))
        for r in rows[hi + 1:] if len(r) > h.index("Metric Value")}
B = 1034449488          # SURVEY.md §8(d) B_fwdbwd(C3)
rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
out = {"round": R,
       "what": "DRAM bytes of ONE graph-replayed fused C3 pass (122 launches, PDL-overlapped as in the "
               "bench): ncu --replay-mode app-range --cache-control none over a cudaProfilerStart/Stop "
               "range around one ws_run (scripts/pass_range.py); reads + writes of the whole pass",
       "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "bytes_per_pass": int(rd + wr),
       "algorithmic_bytes_per_pass": B, "traffic_over_algorithmic": round((rd + wr) / B, 3),
       "range_duration_us_under_profiler": round(vals.get("gpu__time_duration.sum", 0) / 1e3, 1),
       "command": "ncu --replay-mode app-range --cache-control none --clock-control none --metrics "
                  "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum python "
                  "scripts/pass_range.py"}
json.dump(out, open(os.path.join(HERE, "profiles", f"traffic_{R}.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
