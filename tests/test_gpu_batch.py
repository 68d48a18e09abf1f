"""Corner batches vs single-corner runs.

A batch of nc corners runs every level kernel once with blockIdx.y = corner
(the batch's corners sit at a uniform stride in HBM, alloc_corners), with
the occupancy-tuned level-kernel variants for nc >= 4.  Every TimingState and
GradientState field and the summary are bitwise those of single-corner runs;
WS_RUN_CORNER_SUM's sum_k d_arc / sum_k d_edge (the batch objective's
gradient) is the corner-order sum, bitwise the sequential numpy sum of the
corners, in every run mode.
"""

import numpy as np
import pytest
import torch

from golden_util import G_FIELDS, ST_FIELDS, load, raw_of
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G
from paper_2603_28381_b200.corners import corner_values

pytestmark = pytest.mark.gpu

FUSED = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED


def _batch_vs_single(raw, nc, loss="hinge"):
    dev = ws.DeviceDesign(raw, n_corners=nc)
    for k in range(nc):
        dev.set_values(k, **corner_values(raw, k))
    dev.run(FUSED | _lib.RUN_CORNER_SUM, corner=0, n_corners=nc, loss=loss)
    batch = [{f: dev.get(f, k) for f in ST_FIELDS + G_FIELDS} for k in range(nc)]
    sums = [dev.summary(k) for k in range(nc)]
    dsum = {f: dev.get(f) for f in ("d_arc_sum", "d_edge_sum")}
    assert dev.last_launch_count() > 0
    # the sequential mode (per-level kernels, blockIdx.y = corner) gives the same
    dev.run(_lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_CORNER_SUM, corner=0,
            n_corners=nc, loss=loss)
    for f in dsum:
        assert np.array_equal(dev.get(f), dsum[f]), f
    tot = {"d_arc_sum": batch[0]["d_arc"].copy(), "d_edge_sum": batch[0]["d_edge"].copy()}
    for b in batch[1:]:
        tot["d_arc_sum"] += b["d_arc"]
        tot["d_edge_sum"] += b["d_edge"]
    for f in dsum:
        assert np.array_equal(dsum[f], tot[f]), f
    for k in range(nc):
        dev.run(FUSED, corner=k, n_corners=1, loss=loss)
        for f in ST_FIELDS + G_FIELDS:
            assert np.array_equal(dev.get(f, k), batch[k][f], equal_nan=True), (nc, k, f)
        assert dev.summary(k) == sums[k]
    dev.close()


@pytest.mark.parametrize("name", ["edge_kinds", "multi_out", "gen_multi_out_tree", "gen_heavy_1500",
                                  "gen_tree_1200", "kat_diamond", "kat_flat_nets"])
@pytest.mark.parametrize("nc", [2, 3, 5, 8, 16])
def test_batch_bitwise_single(name, nc):
    _batch_vs_single(raw_of(load(name)), nc)


@pytest.mark.parametrize("nc", [4, 16])
def test_batch_softplus_wide_nets(nc):
    cfg = G.GeneratorConfig(num_cells=2500, fanout=G.power_law(1.1, 260), depth_target=5,
                            max_cell_inputs=180, seed=11, net_topology="random_tree")
    _batch_vs_single(G.generate_raw(cfg), nc, loss="softplus")


def test_batch_graph_replay_c1():
    raw = G.generate_raw(G.config_c1())
    _batch_vs_single(raw, 16)
    dev = ws.DeviceDesign(raw, n_corners=16)
    for k in range(16):
        dev.set_values(k, **corner_values(raw, k))
    dev.run(FUSED | _lib.RUN_CORNER_SUM, corner=0, n_corners=16)
    ref = dev.get("d_arc_sum"), dev.get("arrival", 15)
    for _ in range(3):
        dev.run(FUSED | _lib.RUN_CORNER_SUM | _lib.RUN_GRAPH, corner=0, n_corners=16)
    assert np.array_equal(dev.get("d_arc_sum"), ref[0]) and np.array_equal(dev.get("arrival", 15), ref[1])
    dev.close()


def _with_env(var, val, fn):
    import os
    old = os.environ.get(var)
    os.environ[var] = val
    try:
        return fn()
    finally:
        if old is None:
            del os.environ[var]
        else:
            os.environ[var] = old


@pytest.mark.parametrize("nc", [5, 8, 16])
def test_batch_split_streams_bitwise(nc):
    """Fused batches of >= WS_SPLIT corners run as two half batches on the
    context's two streams (the default for >= 8); every field, the summaries
    and the batch gradient sum equal the lockstep batch (WS_SPLIT=0)."""
    raw = raw_of(load("gen_heavy_1500"))

    def run(split):
        def go():
            dev = ws.DeviceDesign(raw, n_corners=nc)
            for k in range(nc):
                dev.set_values(k, **corner_values(raw, k))
            for _ in range(2):     # the second run replays the captured graph
                dev.run(FUSED | _lib.RUN_GRAPH | _lib.RUN_CORNER_SUM, corner=0, n_corners=nc)
            out = [{f: dev.get(f, k) for f in ST_FIELDS + G_FIELDS} for k in range(nc)]
            out.append({f: dev.get(f) for f in ("d_arc_sum", "d_edge_sum")})
            out.append([dev.summary(k) for k in range(nc)])
            dev.close()
            return out
        return _with_env("WS_SPLIT", split, go)

    a, b = run("0"), run("4")
    for k in range(nc + 1):
        for f in a[k]:
            assert np.array_equal(a[k][f], b[k][f], equal_nan=True), (k, f)
    assert a[-1] == b[-1]
