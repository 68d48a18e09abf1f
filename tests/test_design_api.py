"""Host-side API of the drop-in (SURVEY §8(b) re-exports): validation and
its error types, the JSON document, the scalar LUT / per-net RC oracle
functions and the level-schedule checker — against the reference's own
tests (test_netlist.py, test_sta.py) and, where it is installed here,
against the reference itself on the same inputs."""

import os
import sys

import numpy as np
import pytest

import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import design_io as D, generator as G
from paper_2603_28381_b200.netlist import (Cell, Design, Endpoint, Lut2D, Net, PrimaryInput,
                                           TimingArc)

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
have_ref = os.path.isdir(os.path.join(REF, "stasim"))
needs_ref = pytest.mark.skipif(not have_ref, reason="reference not built")


def ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import stasim
    return stasim


def const_lut(v):
    return Lut2D(np.array([0.0]), np.array([0.0]), np.array([[float(v)]]))


def const_arc(f, t, d, s=1e-12):
    return TimingArc(f, t, [const_lut(d) for _ in range(4)], [const_lut(s) for _ in range(4)])


def zero_net(root, members, parents=None):
    m = len(members)
    return Net(root, list(members), list(parents) if parents else [root] * m, np.zeros((m, 4)),
               np.zeros((m, 4)), np.zeros(4))


def chain(n):
    names, nets, cells, root = ["pi"], [], [], 0
    for i in range(n - 1):
        names += [f"b{i}.in", f"b{i}.out"]
        nets.append(zero_net(root, [len(names) - 2]))
        cells.append(Cell([const_arc(len(names) - 2, len(names) - 1, 1.0)]))
        root = len(names) - 1
    names.append("po")
    nets.append(zero_net(root, [len(names) - 1]))
    return Design(names, cells, nets, [PrimaryInput(0, 0.0, 1e-12)], [Endpoint(len(names) - 1, 1.0)], 1.0)


# ---- validate (test_netlist.py:29-68)

def test_validate_not_topological():
    net = Net(0, [1, 2], [2, 0], np.zeros((2, 4)), np.zeros((2, 4)), np.zeros(4))
    d = Design(["r", "a", "b"], [], [net], [PrimaryInput(0, 0.0, 1e-12)],
               [Endpoint(1, 1.0), Endpoint(2, 1.0)], 1.0)
    v = ws.validate(d)
    assert [x.kind for x in v] == ["non-tree-net"] and "not in topological order" in v[0].message


def test_validate_parent_two_cycle():
    net = Net(0, [1, 2], [2, 1], np.zeros((2, 4)), np.zeros((2, 4)), np.zeros(4))
    d = Design(["r", "a", "b"], [], [net], [PrimaryInput(0, 0.0, 1e-12)],
               [Endpoint(1, 1.0), Endpoint(2, 1.0)], 1.0)
    assert [x.kind for x in ws.validate(d)].count("non-tree-net") == 1


def test_validate_combinational_loop():
    d = Design(["a.out", "b.in", "b.out", "a.in"], [Cell([const_arc(3, 0, 1.0)]), Cell([const_arc(1, 2, 1.0)])],
               [zero_net(0, [1]), zero_net(2, [3])], [], [], 1.0)
    assert any(x.kind == "cyclic" and "cycle" in x.message for x in ws.validate(d))


def test_validate_clean_and_every_kind():
    assert ws.validate(chain(4)) == []
    d = chain(3)
    d.nets[0].member_res[0, 1] = -1.0                                 # bad-value
    d.cells[0].arcs.append(const_arc(3, 3, 1.0))                      # self loop
    d.cells.append(Cell([const_arc(1, 2, 1.0)]))                      # second cell drives pin 2
    d.primary_inputs.append(PrimaryInput(0, 0.0, 1e-12))              # PI listed twice
    d.endpoints.append(Endpoint(4, float("nan")))                     # non-finite RAT
    d.clock_period = -1.0
    kinds = {x.kind for x in ws.validate(d)}
    assert {"bad-value", "bad-arc", "multi-driver"} <= kinds
    d2 = chain(3)
    d2.nets[1].member_pins.append(9)
    d2.nets[1].member_parents.append(2)
    d2.nets[1].member_res = np.zeros((2, 4))
    d2.nets[1].member_caps = np.zeros((2, 4))
    assert [x.kind for x in ws.validate(d2)] == ["dangling-ref"]
    lut = Lut2D(np.array([1.0, 0.0]), np.array([0.0]), np.array([[0.0], [1.0]]))
    d3 = chain(2)
    d3.cells[0].arcs[0].delay_luts[2] = lut
    assert any(x.kind == "bad-lut" and "strictly increasing" in x.message for x in ws.validate(d3))
    d4 = chain(2)
    d4.pin_names += ["x", "y", "z"]
    d4.nets.append(zero_net(4, [5]))                                  # root x undriven, y dangles
    d4.cells.append(Cell([const_arc(6, 2, 1.0)]))                     # z sources an arc, no value
    kinds = [x.kind for x in ws.validate(d4)]
    assert "undriven-root" in kinds and "dangling-pin" in kinds and "undriven-pin" in kinds


def test_lut_checks():
    good = Lut2D(np.array([0.0, 1.0]), np.array([0.0, 1.0]), np.array([[0.0, 1.0], [2.0, 3.0]]))
    assert good.check() == []
    assert any("strictly increasing" in p for p in
               Lut2D(np.array([1.0, 0.0]), np.array([0.0]), np.array([[0.0], [1.0]])).check())
    assert any("shape" in p for p in Lut2D(np.array([0.0]), np.array([0.0]), np.array([[0.0, 1.0]])).check())


def test_engine_invariants_refuse_before_the_kernels():
    """flatten / DeviceDesign raise DesignSemanticsError for inputs the
    device build cannot honour (tree order, multiple drivers, axis order)."""
    net = Net(0, [1, 2], [2, 0], np.zeros((2, 4)), np.zeros((2, 4)), np.zeros(4))
    d = Design(["r", "a", "b"], [], [net], [PrimaryInput(0, 0.0, 1e-12)],
               [Endpoint(1, 1.0), Endpoint(2, 1.0)], 1.0)
    with pytest.raises(ws.DesignSemanticsError) as e:
        D.check_engine_invariants(ws.design_to_raw(d))
    assert e.value.violations[0].kind == "non-tree-net"
    d2 = chain(2)
    d2.cells[0].arcs[0].slew_luts[3] = Lut2D(np.array([2.0, 1.0]), np.array([0.0]), np.array([[1.0], [2.0]]))
    with pytest.raises(ValueError):
        D.check_engine_invariants(ws.design_to_raw(d2))
    D.check_engine_invariants(G.generate_raw(G.config_c1()))


def test_raw_and_object_validation_agree_on_generated():
    d = G.generate_design(G.GeneratorConfig(num_cells=400, depth_target=6, seed=9,
                                            net_topology="random_tree"))
    assert ws.validate(d) == [] and ws.validate(ws.design_to_raw(d)) == []


# ---- JSON document (test_netlist.py:116-134)

def test_serialize_round_trip_byte_identical():
    d = chain(4)
    text = ws.serialize_design(d)
    again = ws.parse_design(text)
    assert ws.design_equal(d, again) and ws.serialize_design(again) == text
    assert ws.serialize_design(d) == ws.serialize_design(chain(4))


def test_parse_rejects_garbage():
    with pytest.raises(ws.DesignFormatError):
        ws.parse_design("not json at all {")
    with pytest.raises(ws.DesignFormatError):
        ws.parse_design("{}")
    bad = ws.serialize_design(chain(3)).replace('"parent": 0', '"parent": 4', 1)
    with pytest.raises(ws.DesignSemanticsError):
        ws.parse_design(bad)


@needs_ref
def test_documents_interchange_with_the_reference():
    R = ref()
    d = R.generate_design(R.GeneratorConfig(num_cells=300, depth_target=5, seed=11))
    text = R.serialize_design(d)
    ours = ws.parse_design(text)
    assert ws.serialize_design(ours) == text                   # byte for byte
    assert R.serialize_design(R.parse_design(ws.serialize_design(ours))) == text


# ---- scalar oracle functions (sta.py:103-202) vs the reference

@needs_ref
def test_interpolate_lut_and_net_rc_match_reference():
    R = ref()
    import stasim.sta as RS
    d = R.generate_design(R.GeneratorConfig(num_cells=200, depth_target=4, seed=2,
                                            net_topology="random_tree"))
    rng = np.random.default_rng(1)
    for cell in d.cells[:60]:
        for lut in cell.arcs[0].delay_luts + cell.arcs[0].slew_luts:
            for _ in range(3):
                s, l = rng.uniform(-1e-11, 4e-10), rng.uniform(-1e-15, 2e-13)
                assert ws.interpolate_lut(lut, s, l) == RS.interpolate_lut(lut, s, l)
    for net in d.nets[:120]:
        a, b = ws.compute_net_loads(net), RS.compute_net_loads(net)
        assert np.array_equal(a, b)
        da, db = ws.compute_net_delays(net, a), RS.compute_net_delays(net, b)
        assert np.array_equal(da, db)
        assert np.array_equal(ws.compute_net_impulses(net, a, da), RS.compute_net_impulses(net, b, db))


@needs_ref
def test_check_schedule_matches_reference():
    R = ref()
    import stasim.sta as RS
    from stasim.flatten import LevelSchedule
    d = R.generate_design(R.GeneratorConfig(num_cells=300, depth_target=6, seed=5))
    fl = R.flatten(d)
    assert ws.check_schedule(d, fl.schedule) == [] == RS.check_schedule(d, fl.schedule)
    flat_nets = np.concatenate(fl.schedule.levels)
    bad = LevelSchedule([flat_nets], np.zeros(len(d.nets), dtype=np.int64))
    assert len(ws.check_schedule(d, bad)) == len(RS.check_schedule(d, bad)) > 0
    dup = LevelSchedule(fl.schedule.levels + [fl.schedule.levels[0]], fl.schedule.level_of)
    assert any("appear" in p for p in ws.check_schedule(d, dup))
