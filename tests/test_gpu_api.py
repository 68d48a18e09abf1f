"""The reference's oracle-level API on the device:
run_reference in both reduce modes, propagate_arrival / propagate_required,
finite_diff_check, and the design checks in front of ws_create."""

import numpy as np
import pytest

from golden_util import ST_FIELDS, load, raw_of
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import generator as G

pytestmark = pytest.mark.gpu

SEQ = ["edge_kinds", "gen_tree_1200", "gen_heavy_1500", "multi_out", "gen_uniform_tree"]


@pytest.mark.parametrize("name", SEQ)
def test_run_reference_modes_bit_exact(name):
    """run_reference(flat) is the reference's sequential mode (np.add.reduceat
    root loads: first + pairwise rest); "tree"/8 is run_engine."""
    g = load(name)
    flat = ws.flatten(raw_of(g))
    sq = ws.run_reference(flat)
    for f in ST_FIELDS:
        assert np.array_equal(getattr(sq, f), g["sq_" + f], equal_nan=True), f
    tr = ws.run_reference(flat, reduce_mode="tree", reduce_width=8)
    for f in ST_FIELDS:
        assert np.array_equal(getattr(tr, f), g["st_" + f], equal_nan=True), f
    with pytest.raises(ValueError):
        ws.run_reference(flat, reduce_mode="bogus")


@pytest.mark.parametrize("name", ["edge_kinds", "multi_out", "gen_c1_star", "gen_tree_1200"])
def test_propagate_arrival_required(name):
    g = load(name)
    flat = ws.flatten(raw_of(g))
    st = ws.TimingState.init(flat)
    for f in ("load", "net_delay", "impulse"):
        setattr(st, f, g["st_" + f].copy())
    ws.propagate_arrival(flat, st)
    for f in ("arrival", "slew", "arc_delay"):
        assert np.array_equal(getattr(st, f), g["st_" + f]), f
    ws.propagate_required(flat, st)
    for f in ("required", "slack"):
        assert np.array_equal(getattr(st, f), g["st_" + f]), f


@pytest.mark.parametrize("loss", ["hinge", "softplus"])
def test_finite_diff_check(loss):
    """diff.py:339-474 with the reference's own bar (test_diff.py:128-145:
    max rel < 1e-4): device analytic d_arc / d_edge vs central differences of
    the extended-precision loss."""
    for name in ("kat_chain5_viol", "multi_out", "edge_kinds"):
        rep = ws.finite_diff_check(ws.flatten(raw_of(load(name))), loss=loss)
        assert rep.n_coords > 0 and rep.loss_kind == loss
        if rep.n_significant:
            assert rep.max_rel_error < 1e-4, (name, str(rep))
    for seed in (11, 12, 13):
        raw = G.generate_raw(G.GeneratorConfig(num_cells=25, fanout=G.uniform(1, 4), depth_target=5,
                                               seed=seed))
        rep = ws.finite_diff_check(ws.flatten(raw), loss=loss)
        assert rep.n_significant > 0 and rep.max_rel_error < 1e-4, str(rep)
        assert not rep.epsilon_dominated


def test_finite_diff_flags():
    """test_diff.py:148-161: a design without violations has zero gradients
    and zero loss changes; a huge epsilon is flagged epsilon-dominated."""
    from test_design_api import chain
    d = chain(4)
    d.cells = [ws.Cell([ws.TimingArc(a.from_pin, a.to_pin,
                                     [ws.Lut2D([0.0], [0.0], [[0.01]])] * 4, a.slew_luts)])
               for c in d.cells for a in c.arcs]
    d.endpoints = [ws.Endpoint(d.endpoints[0].pin, 100.0)]
    d.clock_period = 100.0
    rep = ws.finite_diff_check(ws.flatten(d))
    assert rep.max_abs_error <= 1e-9
    raw = G.generate_raw(G.GeneratorConfig(num_cells=20, fanout=G.uniform(1, 3), depth_target=5, seed=14))
    flat = ws.flatten(raw)
    small = ws.finite_diff_check(flat)
    big = ws.finite_diff_check(flat, epsilon=0.5 * flat.clock_period)
    assert not small.epsilon_dominated and big.epsilon_dominated
    assert big.max_abs_error > small.max_abs_error
    with pytest.raises(ValueError):
        ws.finite_diff_check(flat, epsilon=-1.0)


def test_invalid_designs_never_reach_the_kernels():
    raw = raw_of(load("gen_tree_1200"))
    # a member listed before its parent
    mp = raw.mem_parent_pin.copy()
    k = int(np.flatnonzero(raw.mem_parent_pin != raw.net_root[np.searchsorted(raw.net_mptr, np.arange(len(mp)), side="right") - 1])[0])
    mp[k] = raw.mem_pin[k + 1] if k + 1 < len(mp) else raw.mem_pin[k]
    bad = raw_of(load("gen_tree_1200"))
    bad.mem_parent_pin = mp
    with pytest.raises(ws.DesignSemanticsError):
        ws.flatten(bad)
    # a pin that is a member of two nets
    bad2 = raw_of(load("gen_c1_star"))
    mp2 = bad2.mem_pin.copy()
    mp2[1] = mp2[0]
    bad2.mem_pin = mp2
    with pytest.raises(ws.DesignSemanticsError):
        ws.DeviceDesign(bad2)
