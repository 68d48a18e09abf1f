"""The workload generator port reproduces the reference generator bit for bit
(generator.py:205-359): same pins, arcs, LUT pool, RC values and seeds."""

import os
import sys

import numpy as np
import pytest

from golden_util import load, raw_of
from paper_2603_28381_b200 import generator as G

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
RAW_FIELDS = ("net_root", "net_mptr", "mem_pin", "mem_parent_pin", "mem_res", "mem_cap",
              "root_cap", "arc_from", "arc_to", "arc_dlut", "arc_slut", "lut_s_ptr",
              "lut_l_ptr", "lut_t_ptr", "lut_s_flat", "lut_l_flat", "lut_t_flat", "pi_pin",
              "pi_arrival", "pi_slew", "ep_pin", "ep_required")

GOLDEN_CFGS = {
    "gen_c1_star": dict(num_cells=2500, fanout=G.power_law(2.0, 64), depth_target=12, seed=7),
    "gen_tree_1200": dict(num_cells=1200, fanout=G.power_law(2.0, 64), depth_target=9, seed=1,
                          net_topology="random_tree"),
    "gen_heavy_1500": dict(num_cells=1500, fanout=G.power_law(2.0, 512), depth_target=8, seed=901),
    "gen_single_in": dict(num_cells=400, fanout=G.fixed(2), depth_target=6, seed=3,
                          max_cell_inputs=1, net_topology="random_tree"),
    "gen_uniform_tree": dict(num_cells=300, fanout=G.uniform(1, 9), depth_target=7, seed=5,
                             net_topology="random_tree"),
}


def same(a, b):
    for f in RAW_FIELDS:
        x, y = getattr(a, f), getattr(b, f)
        assert x.shape == y.shape and np.array_equal(x, y), f
    assert a.n_pins == b.n_pins and a.clock_period == b.clock_period


@pytest.mark.parametrize("name", sorted(GOLDEN_CFGS))
def test_port_matches_reference_fixture(name):
    g = load(name)
    same(G.generate_raw(G.GeneratorConfig(**GOLDEN_CFGS[name])), raw_of(g))


def test_config_validation():
    with pytest.raises(ValueError):
        G.GeneratorConfig(num_cells=0)
    with pytest.raises(ValueError):
        G.GeneratorConfig(num_cells=3, depth_target=4)
    with pytest.raises(ValueError):
        G.GeneratorConfig(num_cells=10, net_topology="mesh")
    with pytest.raises(ValueError):
        G.FanoutDist("zipf")


def test_deterministic():
    cfg = G.GeneratorConfig(num_cells=500, seed=11)
    same(G.generate_raw(cfg), G.generate_raw(cfg))


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "stasim")),
                    reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("kw", [
    dict(num_cells=700, fanout=("fixed", 1), depth_target=7, seed=4),      # coverage bumps
    dict(num_cells=900, fanout=("uniform", 2, 6), depth_target=10, seed=21, net_topology="random_tree"),
    dict(num_cells=1000, fanout=("power_law", 2.0, 512), depth_target=5, seed=8, max_cell_inputs=2),
    dict(num_cells=300, fanout=("power_law", 1.5, 32), depth_target=3, seed=2, lut_grid_size=1),
])
def test_port_matches_live_reference(kw):
    sys.path.insert(0, REF)
    try:
        import stasim
    finally:
        sys.path.remove(REF)
    from paper_2603_28381_b200.netlist import design_to_raw
    fk = kw.pop("fanout")
    mk = {"fixed": (stasim.fixed, G.fixed), "uniform": (stasim.uniform, G.uniform),
          "power_law": (stasim.power_law, G.power_law)}[fk[0]]
    d = stasim.generate_design(stasim.GeneratorConfig(fanout=mk[0](*fk[1:]), **kw))
    r = G.generate_raw(G.GeneratorConfig(fanout=mk[1](*fk[1:]), **kw))
    same(design_to_raw(d), r)
    assert d.meta["fanout_bumps"] == r.meta["fanout_bumps"]
