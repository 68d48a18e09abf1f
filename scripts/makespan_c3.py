"""Makespan model on measured C3 kernel costs vs measured passes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import fusion as F, generator as G

raw = G.generate_raw(G.config_c3())
flat = ws.flatten(raw)
out = {}
for gran in (1, 10):
    rep = F.makespan_report(flat, cfg=F.FusionConfig(granularity=gran), repeats=5)
    out[f"granularity_{gran}"] = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in rep.items()}
print(json.dumps(out, indent=1))
