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
# corner batches: 8 corners in the fused mode = two half batches on two
# streams (the split), the batch level kernels, star-net root loads folded
# in the RC member blocks, the in-kernel corner sum; then 8 placement
# candidates (fused sweep, split) — bitwise against the lockstep batch
from paper_2603_28381_b200.corners import corner_values
raw = G.generate_raw(G.GeneratorConfig(num_cells=600, fanout=G.power_law(2.0, 150), depth_target=6, seed=5))
outs = []
for split in ("8", "0"):
    os.environ["WS_SPLIT"] = split
    dev = ws.DeviceDesign(raw, n_corners=8)
    del os.environ["WS_SPLIT"]
    for k in range(8):
        dev.set_values(k, **corner_values(raw, k))
    dev.run(_lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | _lib.RUN_CORNER_SUM, corner=0,
            n_corners=8)
    o = [dev.get("d_arc_sum")] + [dev.get("adjoint", k) for k in range(8)]
    timers = [PL.PlacementTimer(dev, PL.synthetic_placement(raw, seed=30 + k), corner=k, graph=False)
              for k in range(8)]
    dev.run(PL.PlacementTimer.FLAGS, corner=0, n_corners=8)
    o += [dev.get("d_xy", k) for k in range(8)]
    outs.append(o)
    dev.close()
assert all(np.array_equal(x, y) for x, y in zip(*outs))
print("batch split ok")
d = tempfile.mkdtemp()
ws.save_raw(os.path.join(d, "x.npz"), raw)
dev = ws.DeviceDesign.from_file(os.path.join(d, "x.npz"))
dev.run(_lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED)
dev.close()
print("sanitize run ok")
