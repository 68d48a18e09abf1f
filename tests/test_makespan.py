"""The reference's two-lane makespan model (fusion.py:163-265), restated in
paper_2603_28381_b200.fusion, and its validation on MEASURED kernel costs
(SURVEY.md §8(f) rank 3).  CPU: the model's known answers on abstract cost
tables (the reference's test_fusion.py examples: sta 10 / grad 5 per level).
GPU: per-kernel CUDA-event costs of a sequential pass feed build_kernel_graph;
the schedules are valid and the sequential model reproduces the measured
sequential pass."""

import numpy as np
import pytest

import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import fusion as F
from paper_2603_28381_b200 import generator as G

KINDS = ("net_rc", "cell_delay_at", "slack_bwd", "lse_fwd", "grad_bwd")


def costs_table(n, sta=10.0, grad=5.0):
    c = {(k, li): 0.0 for li in range(n) for k in KINDS}
    for li in range(n):
        c[("cell_delay_at", li)] = sta
        c[("lse_fwd", li)] = grad
    return c


def test_sequential_sums_costs():
    g = F.build_kernel_graph(3, costs_table(3), granularity=1)
    assert F.schedule_sequential(g).makespan == 45.0
    g0 = F.build_kernel_graph(3, costs_table(3, grad=0.0), granularity=1)
    assert F.schedule_sequential(g0).makespan == 30.0


def test_fused_two_lane_example():
    g = F.build_kernel_graph(3, costs_table(3), granularity=1)
    r = F.schedule_fused(g)
    assert [r.finish(f"lse_fwd:{i}") for i in range(3)] == [15.0, 25.0, 35.0]
    assert r.makespan == 35.0 and F.check_schedule(g, r) == []
    g0 = F.build_kernel_graph(4, costs_table(4, sta=7.0, grad=0.0), granularity=1)
    assert F.schedule_fused(g0).makespan == F.schedule_sequential(g0).makespan == 28.0


def test_contention_stretches_overlap():
    g = F.build_kernel_graph(3, costs_table(3, grad=9.0), granularity=1)
    base, slow = F.schedule_fused(g, 1.0), F.schedule_fused(g, 2.0)
    assert base.makespan == 39.0 and slow.makespan > base.makespan
    assert F.check_schedule(g, slow) == []


def test_fused_never_slower_random():
    rng = np.random.default_rng(4)
    for _ in range(40):
        L = int(rng.integers(1, 20))
        c = {(k, li): (float(rng.uniform(0, 5)) if rng.random() > 0.2 else 0.0)
             for li in range(L) for k in KINDS}
        g = F.build_kernel_graph(L, c, granularity=int(rng.integers(1, 8)))
        assert g.is_acyclic()
        s, f = F.schedule_sequential(g), F.schedule_fused(g)
        assert f.makespan <= s.makespan + 1e-12
        assert F.check_schedule(g, f) == [] and F.check_schedule(g, s) == []
        assert 0.0 <= f.overlap_fraction <= 1.0


def test_check_schedule_flags_violations():
    g = F.build_kernel_graph(2, costs_table(2), granularity=1)
    r = F.schedule_fused(g)
    rec = [dict(x) for x in r.records]
    for x in rec:
        if x["id"] == "lse_fwd:0":
            x["start"] = 0.0           # before cell_delay_at:0 finishes
    bad = F.ScheduleResult(rec, r.makespan, 0, 0, 0, 0)
    assert any("event violated" in p for p in F.check_schedule(g, bad))


@pytest.mark.gpu
def test_measured_costs_feed_the_model():
    raw = G.generate_raw(G.config_c1())
    flat = ws.flatten(raw)
    rep = F.makespan_report(flat, repeats=3)
    assert rep["problems"] == []
    # calibrated costs: the sequential model reproduces the measured pass
    assert abs(rep["model_sequential_ms"] - rep["measured_sequential_ms"]) <= \
        1e-9 * rep["measured_sequential_ms"]
    assert rep["model_fused_ms"] <= rep["model_sequential_ms"] + 1e-9
    assert rep["fitted_contention"] is None or rep["fitted_contention"] >= 1.0
    costs = F.measured_kernel_costs(ws.engine.DeviceDesign(raw), flat.n_levels, repeats=1)
    assert all(v >= 0 for v in costs.values())
    assert sum(costs[("cell_delay_at", li)] for li in range(flat.n_levels)) > 0
