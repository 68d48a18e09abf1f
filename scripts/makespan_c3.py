"""Makespan model (the reference's own) on measured C3 kernel costs vs the
measured passes -> stdout JSON."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), HERE]
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import generator as G
from makespan_ref import makespan_report

raw = G.generate_raw(G.config_c3())
flat = ws.flatten(raw)
out = {}
for gran in (1, 10):
    rep = makespan_report(flat, granularity=gran, repeats=5)
    out[f"granularity_{gran}"] = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in rep.items()}
print(json.dumps(out, indent=1))
