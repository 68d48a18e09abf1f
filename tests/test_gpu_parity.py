"""GPU parity against the reference's own outputs (golden fixtures).

Every call goes through the C-ABI library (libwarpstar_b200.so).  Bars
(north_star): levels / CSR / FlatDesign indices bit-exact; the hard pass
(load, net_delay, impulse, slew, arrival, required, slack, arc_delay) and
TNS/WNS bit-exact with the reference's run_engine (the contract is 1e-5
relative; we hold bit-exactness); gradients within 1e-4 relative.
"""

import copy

import numpy as np
import pytest

from golden_util import G_FIELDS, ST_FIELDS, grad_close, load, max_rel, names, raw_of
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200.netlist import raw_to_design

pytestmark = pytest.mark.gpu
CASES = names()

_flats = {}


def flat_of(name):
    if name not in _flats:
        _flats[name] = ws.flatten(raw_of(load(name)))
    return _flats[name]


@pytest.mark.parametrize("name", CASES)
def test_device_flatten_bit_exact(name):
    g = load(name)
    flat = flat_of(name)
    for k, v in g.items():
        if k.startswith("flat_"):
            got = getattr(flat, k[5:])
            assert got.shape == v.shape and np.array_equal(got, v), k
    lv = flat.schedule.levels
    assert np.array_equal(np.concatenate(lv) if lv else np.zeros(0, np.int64), g["levels_nets"])
    assert np.array_equal(flat.schedule.level_of, g["level_of"])
    csr = ws.build_csr(raw_of(g))
    assert np.array_equal(csr.pin_list, g["csr_pin_list"])
    assert np.array_equal(csr.net_index, g["csr_net_index"])


@pytest.mark.parametrize("name", CASES)
def test_run_engine_bit_exact(name):
    g = load(name)
    flat = flat_of(name)
    st = ws.run_engine(flat)
    for f in ST_FIELDS:
        assert np.array_equal(getattr(st, f), g["st_" + f]), (f, max_rel(getattr(st, f), g["st_" + f]))
    assert ws.tns(st, flat) == g["tns"]
    assert ws.wns(st, flat) == g["wns"]


@pytest.mark.parametrize("name", CASES)
def test_timing_gradients(name):
    g = load(name)
    flat = flat_of(name)
    st = ws.run_engine(flat)
    gs = ws.timing_gradients(flat, cfg=ws.LseConfig(float(g["gamma"])), state=st)
    for f in G_FIELDS:
        assert grad_close(getattr(gs, f), g["g_" + f]), (f, max_rel(getattr(gs, f), g["g_" + f]))
    assert gs.loss == pytest.approx(float(g["g_loss"]), rel=1e-12, abs=1e-300)
    if "gs_loss" in g:
        gp = ws.timing_gradients(flat, cfg=ws.LseConfig(float(g["gamma"])), loss="softplus", state=st)
        for f in G_FIELDS:
            assert grad_close(getattr(gp, f), g["gs_" + f]), f
        assert gp.loss == pytest.approx(float(g["gs_loss"]), rel=1e-12)


@pytest.mark.parametrize("name", CASES)
def test_fused_modes_bit_identical(name):
    """fused (both modes) == sequential == run_engine + timing_gradients,
    bitwise (test_fusion.py:166-188)."""
    g = load(name)
    flat = flat_of(name)
    cfg = dict(gamma=float(g["gamma"]))
    seq = ws.execute_sequential(flat, cfg=ws.FusionConfig(**cfg))
    for mode in ("interleaved", "threads"):
        for gran in (1, 3, 10):
            fus = ws.execute_fused(flat, cfg=ws.FusionConfig(mode=mode, granularity=gran, **cfg))
            for f in ST_FIELDS:
                assert np.array_equal(getattr(fus[0], f), getattr(seq[0], f)), (mode, f)
            for f in G_FIELDS:
                assert np.array_equal(getattr(fus[1], f), getattr(seq[1], f)), (mode, f)
            assert fus[1].loss == seq[1].loss
    st = ws.run_engine(flat)
    gd = ws.timing_gradients(flat, cfg=ws.LseConfig(float(g["gamma"])), state=st)
    for f in ST_FIELDS:
        assert np.array_equal(getattr(seq[0], f), getattr(st, f)), f
    for f in G_FIELDS:
        assert np.array_equal(getattr(seq[1], f), getattr(gd, f)), f


@pytest.mark.parametrize("name", CASES)
def test_legacy_level_shims_bit_exact(name):
    """run_engine(flat, kernels=get_backend("cuda")) drives the per-level
    C-ABI shims (the reference's raw kernel ABI) — bit-identical
    (test_backends.py:28-39)."""
    g = load(name)
    flat = flat_of(name)
    st = ws.run_engine(flat, kernels=ws.get_backend("cuda"))
    for f in ST_FIELDS:
        assert np.array_equal(getattr(st, f), g["st_" + f]), f


@pytest.mark.parametrize("name", ["gen_c1_star", "gen_tree_1200", "edge_kinds"])
@pytest.mark.parametrize("w", [1, 2, 4, 16, 32])
def test_reduce_width_matches_oracle(name, w):
    from oracle import oracle as O
    from golden_util import raw_ns
    g = load(name)
    flat = flat_of(name)
    st = ws.run_engine(flat, reduce_width=w)
    ofl = O.flatten_raw(raw_ns(g))
    ost = O.run_engine(ofl, reduce_width=w)
    for f in ST_FIELDS:
        assert np.array_equal(getattr(st, f), getattr(ost, f)), f


def test_object_model_input_and_value_substitution():
    """flatten() of an object-model Design equals flatten() of its arrays;
    the copy.copy(flat) value-substitution workflow."""
    g = load("gen_c1_star")
    raw = raw_of(g)
    flat = ws.flatten(raw_to_design(raw))
    st = ws.run_engine(flat)
    for f in ST_FIELDS:
        assert np.array_equal(getattr(st, f), g["st_" + f]), f
    f2 = copy.copy(flat)
    f2.mem_res = flat.mem_res * 1.1
    st2 = ws.run_engine(f2)
    from oracle import oracle as O
    from golden_util import raw_ns
    ns = raw_ns(g)
    ns.mem_res = ns.mem_res * 1.1
    ost = O.run_engine(O.flatten_raw(ns))
    for f in ST_FIELDS:
        assert np.array_equal(getattr(st2, f), getattr(ost, f)), f
    # and the original flat still gives the original values
    st3 = ws.run_engine(flat)
    assert np.array_equal(st3.arrival, g["st_arrival"])


def test_tns_wns_kats():
    """test_sta.py:357-391 on the device summary kernels."""
    flat = flat_of("kat_flat_nets")
    st = ws.run_engine(flat)
    st.slack[flat.ep_pin[:3], 2] = [3.0, -2.0, -5.0]
    st.slack[flat.ep_pin[:3], 3] = [3.0, 0.0, 1.0]
    st.slack[flat.ep_pin[3:], 2:4] = 1.0
    assert ws.tns(st, flat) == -7.0
    assert ws.wns(st, flat) == -5.0
    f2 = copy.copy(flat)
    f2.ep_pin = np.zeros(0, dtype=np.int64)
    f2.ep_required = np.zeros((0, 4))
    assert ws.wns(st, f2) == float("inf")
    assert ws.tns(st, f2) == 0.0


def test_cycle_error_names_root_of_lowest_stuck_net():
    from oracle import oracle as O
    from golden_util import raw_ns
    g = load("kat_diamond")
    ns = raw_ns(g)
    # close a loop: the merge net's sink drives the top buffer's input arc
    ns.arc_from = ns.arc_from.copy()
    ns.arc_from[0] = 8          # po feeds b (net 3 -> net 1 -> net 3)
    with pytest.raises(O.OracleCycleError) as oe:
        O.flatten_raw(ns)
    raw = raw_of(g)
    raw.arc_from = ns.arc_from.astype(np.int32)
    with pytest.raises(ws.CycleError) as de:
        ws.flatten(raw)
    assert de.value.pin == oe.value.pin


def test_chain_kats():
    """Chain / two-input / tie-break known answers (test_sta.py:223-270,
    test_diff.py:74-125) on the device path."""
    for name in ("kat_chain6", "kat_chain5_viol", "kat_chain2_req", "kat_two_input", "kat_tie_break"):
        g = load(name)
        flat = flat_of(name)
        st = ws.run_engine(flat)
        assert np.array_equal(st.arrival, g["st_arrival"])
    st = ws.run_engine(flat_of("kat_two_input"))
    assert st.arrival[4, 2] == 6.0 and st.arrival[4, 0] == 5.0
    st = ws.run_engine(flat_of("kat_tie_break"))
    assert np.all(st.slew[4] == 1e-12)
    gs = ws.timing_gradients(flat_of("kat_chain5_viol"))
    assert gs.loss > 0
    np.testing.assert_allclose(gs.d_arc, 1.0, rtol=1e-9)
    np.testing.assert_allclose(gs.d_edge, 1.0, rtol=1e-9)
    flat = flat_of("kat_chain6")
    gl = ws.forward_lse_arrival(flat, state=ws.run_engine(flat))
    assert np.array_equal(gl.lse_arrival, ws.run_engine(flat).arrival[:, 2:4])


@pytest.mark.parametrize("name", CASES)
def test_persistent_pass_bit_identical(name):
    """One cooperative kernel for the whole pass == the per-level kernels."""
    from paper_2603_28381_b200 import _lib
    flat = flat_of(name)
    dev = flat.dev
    ws.run_engine(flat)   # uploads the flat's values
    base = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
    dev.run(base | _lib.RUN_FUSED)
    ref = {f: dev.get(f) for f in ST_FIELDS + G_FIELDS}
    ref_sum = dev.summary()
    for flags in (base | _lib.RUN_PERSISTENT, base | _lib.RUN_PERSISTENT | _lib.RUN_GRAPH):
        dev.run(flags)
        for f in ST_FIELDS + G_FIELDS:
            assert np.array_equal(dev.get(f), ref[f]), (flags, f)
        assert dev.summary() == ref_sum
    dev.run(_lib.RUN_HARD | _lib.RUN_PERSISTENT)
    for f in ST_FIELDS:
        assert np.array_equal(dev.get(f), ref[f]), f
    assert dev.summary()[:2] == ref_sum[:2]


def test_graph_replay_bit_identical():
    g = load("gen_c1_star")
    flat = flat_of("gen_c1_star")
    dev = flat.dev
    from paper_2603_28381_b200 import _lib
    flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED
    dev.run(flags)
    a = {f: dev.get(f) for f in ST_FIELDS + G_FIELDS}
    for _ in range(3):
        dev.run(flags | _lib.RUN_GRAPH)
    for f in ST_FIELDS + G_FIELDS:
        assert np.array_equal(dev.get(f), a[f]), f
    for f in ST_FIELDS:
        assert np.array_equal(a[f], g["st_" + f]), f


def test_graph_replay_follows_gamma_and_loss():
    """The graph cache keys on the pass shape, not on gamma: a placement /
    annealing loop that changes gamma every call re-uses the executable (its
    kernel parameters updated in place) and still gets the new gamma's
    results; more shapes than the cache holds evict the oldest."""
    from paper_2603_28381_b200 import _lib
    flat = flat_of("gen_c1_star")
    dev = flat.dev
    base = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED
    g0 = 0.01 * flat.clock_period
    for i, gamma in enumerate(g0 * np.linspace(0.5, 2.0, 12)):
        loss = "softplus" if i % 3 == 2 else "hinge"
        dev.run(base | _lib.RUN_GRAPH, gamma=gamma, loss=loss)
        got = dev.get("d_arc"), dev.summary()
        dev.run(base, gamma=gamma, loss=loss)
        assert np.array_equal(dev.get("d_arc"), got[0]) and dev.summary() == got[1], (i, gamma)
    for gran in range(1, 20):      # 19 shapes > the 16-entry cache
        dev.run(base | _lib.RUN_GRAPH, gamma=g0, granularity=gran)
    dev.run(base, gamma=g0)
    ref = dev.get("lse_arrival")
    dev.run(base | _lib.RUN_GRAPH, gamma=g0, granularity=1)
    assert np.array_equal(dev.get("lse_arrival"), ref)
