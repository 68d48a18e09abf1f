"""Small-design passes in every run mode (+ placement, ingest, timed) for
compute-sanitizer: python scripts/sanitize_run.py"""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G, placement as PL

for topo in ("star", "random_tree"):
    raw = G.generate_raw(G.GeneratorConfig(num_cells=600, fanout=G.power_law(2.0, 150), depth_target=6,
                                           seed=5, net_topology=topo))
    dev = ws.DeviceDesign(raw, n_corners=2)
    base = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
    outs = []
    for extra in (0, _lib.RUN_FUSED, _lib.RUN_TWO_STREAM, _lib.RUN_PERSISTENT, _lib.RUN_FUSED | _lib.RUN_GRAPH,
                  _lib.RUN_TIMED):
        dev.run(base | extra, corner=0, n_corners=2)
        outs.append(dev.get("adjoint"))
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    pl = PL.synthetic_placement(raw, seed=1)
    timer = PL.PlacementTimer(dev, pl)
    timer.step()
    timer.step(pl.xy + 0.1)
    dev.run(_lib.RUN_WIRE | base | _lib.RUN_POSGRAD, corner=1)
    # the fused sweep (k_bwd<..., PG>, cp.async prologue) vs the stand-alone one
    fused = base | _lib.RUN_FUSED | _lib.RUN_WIRE | _lib.RUN_POSGRAD
    dev.run(fused, corner=0, n_corners=2)
    a = dev.get("d_xy", 1)
    os.environ["WS_PG_SWEEP"] = "stream"
    dev.run(fused, corner=0, n_corners=2)
    del os.environ["WS_PG_SWEEP"]
    assert np.array_equal(a, dev.get("d_xy", 1))
    print(topo, dev.summary(), float(np.abs(timer.grad_xy()).max()))
    dev.close()
d = tempfile.mkdtemp()
ws.save_raw(os.path.join(d, "x.npz"), raw)
dev = ws.DeviceDesign.from_file(os.path.join(d, "x.npz"))
dev.run(_lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED)
dev.close()
print("sanitize run ok")
