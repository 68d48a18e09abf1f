"""The fusion pipeline's kernel graph and dependency discipline, and the
reference's makespan model on MEASURED kernel costs.

The makespan simulator is the reference's own (scripts/makespan_ref.py
imports the unmodified stasim.fusion); this package only builds the same
KernelGraph (checked against the reference's here) and measures the costs.
"""

import os
import sys

import numpy as np
import pytest

import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import fusion as F
from paper_2603_28381_b200 import generator as G

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "scripts"))
from makespan_ref import makespan_report, reference_fusion  # noqa: E402

KINDS = ("net_rc", "cell_delay_at", "slack_bwd", "lse_fwd", "grad_bwd")
RF = reference_fusion()
needs_ref = pytest.mark.skipif(RF is None, reason="reference not installed")


@needs_ref
@pytest.mark.parametrize("L,g", [(1, 1), (3, 1), (7, 2), (12, 5), (60, 10), (13, 20)])
def test_kernel_graph_matches_reference(L, g):
    rng = np.random.default_rng(L * 31 + g)
    costs = {(k, li): float(rng.uniform(0, 3)) for li in range(L) for k in KINDS}
    ours, ref = F.build_kernel_graph(L, costs, g), RF.build_kernel_graph(L, costs, g)
    assert ours.sta_order == ref.sta_order and ours.grad_order == ref.grad_order
    assert [(e.src, e.dst) for e in ours.edges] == [(e.src, e.dst) for e in ref.edges]
    for kid, k in ours.kernels.items():
        r = ref.kernels[kid]
        assert (k.stream, k.kind, k.level, k.cost) == (r.stream, r.kind, r.level, r.cost)
    assert ours.is_acyclic()
    # the reference's own scheduler accepts our graph's structure and costs
    fus = RF.schedule_fused(RF.build_kernel_graph(L, costs, g))
    assert RF.check_schedule(ref, fus) == []


def test_kernel_graph_validation():
    with pytest.raises(ValueError):
        F.build_kernel_graph(3, {}, 1)
    with pytest.raises(ValueError):
        F.build_kernel_graph(3, None, 0)
    with pytest.raises(ValueError):
        F.Kernel("x", F.STA_STREAM, "lse_fwd", 0, 1.0)
    with pytest.raises(ValueError):
        F.Kernel("x", F.GRAD_STREAM, "lse_fwd", 0, -1.0)


@pytest.mark.gpu
def test_dependency_violation_raises():
    """fusion.py:307-312 / test_fusion.py:198-209: a kernel whose
    dependency never executed is refused, nothing is launched."""
    raw = G.generate_raw(G.GeneratorConfig(num_cells=200, depth_target=4, seed=3))
    run = F.PipelineRun(ws.flatten(raw))
    g = F.build_kernel_graph(run.flat.n_levels, None, 1)
    with pytest.raises(F.FusionError):
        run.execute(g.kernels["lse_fwd:0"], ["cell_delay_at:0"])
    assert run.done == set()
    run.execute(g.kernels["net_rc:0"], [])
    with pytest.raises(F.FusionError):
        run.execute(g.kernels["cell_delay_at:1"], ["net_rc:1"])


@pytest.mark.gpu
@pytest.mark.parametrize("gran", [1, 3, 10])
def test_execute_graph_bitwise_sequential(gran):
    """Kernel by kernel through the dependency discipline == one ws_run."""
    from golden_util import G_FIELDS, ST_FIELDS, load, raw_of
    for name in ("edge_kinds", "multi_out", "gen_tree_1200"):
        flat = ws.flatten(raw_of(load(name)))
        cfg = F.FusionConfig(granularity=gran)
        st, gs = F.execute_graph(flat, cfg=cfg)
        st2, gs2, _ = F.execute_sequential(flat, cfg=cfg)
        for f in ST_FIELDS:
            assert np.array_equal(getattr(st, f), getattr(st2, f), equal_nan=True), (name, f)
        for f in G_FIELDS:
            assert np.array_equal(getattr(gs, f), getattr(gs2, f)), (name, f)
        assert gs.loss == gs2.loss


@needs_ref
@pytest.mark.gpu
def test_measured_costs_feed_the_reference_model():
    raw = G.generate_raw(G.config_c1())
    flat = ws.flatten(raw)
    rep = makespan_report(flat, repeats=3)
    assert rep["problems"] == []
    # calibrated costs: the sequential model reproduces the measured pass
    assert abs(rep["model_sequential_ms"] - rep["measured_sequential_ms"]) <= \
        1e-9 * rep["measured_sequential_ms"]
    assert rep["model_fused_ms"] <= rep["model_sequential_ms"] + 1e-9
    assert rep["fitted_contention"] is None or rep["fitted_contention"] >= 1.0
    costs = F.measured_kernel_costs(ws.engine.DeviceDesign(raw), flat.n_levels, repeats=1)
    assert all(v >= 0 for v in costs.values())
    assert sum(costs[("cell_delay_at", li)] for li in range(flat.n_levels)) > 0
