"""profiles/traffic_<R>.json from gpurun_out/traffic_<R>.csv (ncu dram bytes
of every kernel of one C3 pass).  python scripts/traffic_json.py r01"""
import collections
import csv
import json
import os
import sys

R = sys.argv[1]
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(open(os.path.join(HERE, "gpurun_out", f"traffic_{R}.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1}
TIME = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
per = collections.defaultdict(lambda: {"launches": set(), "dram_bytes": 0.0, "time_us_cold_serialized": 0.0})
units = set()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki]
    d = per[name]
    d["launches"].add(r[ii])
    v = float(r[vi].replace(",", ""))
    units.add(r[ui])
    if r[mi].startswith("dram__bytes"):
        d["dram_bytes"] += v * BYTES.get(r[ui], 1)
    elif r[mi] == "gpu__time_duration.sum":
        d["time_us_cold_serialized"] += v * TIME.get(r[ui], 1.0)
pk = {k: {"launches": len(v["launches"]), "dram_bytes": int(v["dram_bytes"]),
          "time_us_cold_serialized": round(v["time_us_cold_serialized"], 1)} for k, v in per.items()}
tot = sum(v["dram_bytes"] for v in pk.values())
alg = 1034449488
out = {"round": R,
       "what": "DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of every kernel of ONE C3 "
               "fwd+bwd pass (fused mode), ncu --clock-control none, cold caches per kernel",
       "bytes_per_pass": tot, "algorithmic_bytes_per_pass": alg,
       "traffic_over_algorithmic": round(tot / alg, 3), "per_kernel": pk, "units_seen": sorted(units)}
json.dump(out, open(os.path.join(HERE, "profiles", f"traffic_{R}.json"), "w"), indent=1)
print(tot, round(tot / alg, 3), {k: v["launches"] for k, v in pk.items()})
