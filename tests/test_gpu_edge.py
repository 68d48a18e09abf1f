"""Edge shapes on the device vs the CPU oracle, every run mode:

* wide nets (> TASK_A = 128 in-arcs: single-net TK_WIDE tasks) and big RC
  trees (> TASK_M = 128 members: TK_LOOP tasks) next to chunked big star nets;
* a design with no nets at all (every pin free), with and without endpoints;
* a NaN endpoint requirement (the reference's np.minimum.at / maximum.at
  merges are NaN-sticky).
The hard pass must be bit-exact (NaN positions included), gradients within
north_star's 1e-4, modes bitwise equal, position gradients within 1e-9.
"""

import numpy as np
import pytest

from golden_util import G_FIELDS, ST_FIELDS, grad_close
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G, placement as PL
from paper_2603_28381_b200.netlist import RawDesign
from oracle import oracle as O

pytestmark = pytest.mark.gpu

BASE = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
MODES = {"fused": BASE | _lib.RUN_FUSED, "persistent": BASE | _lib.RUN_PERSISTENT,
         "streams": BASE | _lib.RUN_TWO_STREAM, "sequential": BASE}


def _check_modes(raw, gamma=None):
    flat = O.flatten_raw(raw)
    st = O.run_engine(flat)
    g = 0.01 * flat.clock_period if gamma is None else gamma
    gr = O.timing_gradients(flat, st, gamma=g)
    dev = ws.DeviceDesign(raw)
    ref = None
    for name, flags in MODES.items():
        dev.run(flags, gamma=g)
        got = {f: dev.get(f) for f in ST_FIELDS + G_FIELDS}
        for f in ST_FIELDS:
            assert np.array_equal(got[f], getattr(st, f), equal_nan=True), (name, f)
        for f in G_FIELDS:
            assert grad_close(got[f], getattr(gr, {"lse_arrival": "lse_arrival"}.get(f, f))), (name, f)
        tns, wns, loss = dev.summary()
        ot, ow = O.tns(st, flat), O.wns(st, flat)
        assert (tns == ot or (np.isnan(tns) and np.isnan(ot))) and \
               (wns == ow or (np.isnan(wns) and np.isnan(ow))), name
        if ref is None:
            ref = got
        else:
            for f in ref:
                assert np.array_equal(ref[f], got[f], equal_nan=True), (name, f)
    dev.close()
    return flat


def test_wide_nets_and_big_rc_trees():
    cfg = G.GeneratorConfig(num_cells=2500, fanout=G.power_law(1.1, 260), depth_target=5,
                            max_cell_inputs=180, seed=11, net_topology="random_tree")
    raw = G.generate_raw(cfg)
    flat = O.flatten_raw(raw)
    assert int(flat.net_a.max()) > 128, "no TK_WIDE net"
    assert int(flat.net_m.max()) > 128, "no TK_LOOP / chunked net"
    _check_modes(raw)
    # position gradients on the same shapes
    pl = PL.synthetic_placement(raw, seed=2)
    dev = ws.DeviceDesign(raw)
    PL.PlacementTimer(dev, pl).step()
    res, cap = O.wire(flat, pl.xy, pl.res0, pl.cap0, pl.wire.r_unit, pl.wire.c_unit)
    f2 = O.with_values(flat, mem_res=res, mem_cap=cap)
    st2 = O.run_engine(f2)
    pg = O.position_gradients(f2, st2, O.timing_gradients(f2, st2), pl.xy, pl.wire.r_unit,
                              pl.wire.c_unit)
    assert grad_close(dev.get("d_xy"), pg.d_xy, rtol=1e-9)
    assert grad_close(dev.get("d_cap"), pg.d_cap, rtol=1e-9)
    dev.close()


def _empty_raw(with_endpoints):
    lut = dict(lut_s_ptr=np.array([0, 2]), lut_l_ptr=np.array([0, 2]), lut_t_ptr=np.array([0, 4]),
               lut_s_flat=np.array([1e-12, 2e-12]), lut_l_flat=np.array([1e-15, 2e-15]),
               lut_t_flat=np.array([1e-11, 2e-11, 3e-11, 4e-11]))
    z4 = np.zeros((0, 4))
    ep = np.array([1, 3], np.int32) if with_endpoints else np.zeros(0, np.int32)
    epr = (np.array([[0.0, 0.0, 5e-12, 5e-12], [0.0, 0.0, -1e-12, 2e-12]]) if with_endpoints
           else np.zeros((0, 4)))
    return RawDesign(n_pins=5, clock_period=1e-10, net_root=np.zeros(0, np.int32),
                     net_mptr=np.zeros(1, np.int64), mem_pin=np.zeros(0, np.int32),
                     mem_parent_pin=np.zeros(0, np.int32), mem_res=z4, mem_cap=z4, root_cap=z4,
                     arc_from=np.zeros(0, np.int32), arc_to=np.zeros(0, np.int32),
                     arc_dlut=np.zeros((0, 4), np.int32), arc_slut=np.zeros((0, 4), np.int32),
                     pi_pin=np.array([0, 1], np.int32),
                     pi_arrival=np.array([[1e-12, 1e-12, 2e-12, 2e-12], [0, 0, 3e-12, 4e-12]]),
                     pi_slew=np.full((2, 4), 2e-12), ep_pin=ep, ep_required=epr,
                     **lut).normalized()


@pytest.mark.parametrize("with_endpoints", [True, False])
def test_design_without_nets(with_endpoints):
    raw = _empty_raw(with_endpoints)
    _check_modes(raw)
    dev = ws.DeviceDesign(raw)
    dev.run(BASE | _lib.RUN_FUSED)
    tns, wns, loss = dev.summary()
    if not with_endpoints:
        assert tns == 0.0 and wns == float("inf") and loss == 0.0
    dev.close()


def test_nan_endpoint_requirement():
    raw = G.generate_raw(G.GeneratorConfig(num_cells=300, depth_target=5, seed=4))
    epr = np.array(raw.ep_required, dtype=np.float64)
    epr[0, 2] = np.nan                         # late rise of the first endpoint entry
    epr[1, 1] = np.nan                         # early fall of the second
    raw.ep_required = epr
    _check_modes(raw.normalized())


@pytest.mark.parametrize("name", ["multi_out", "gen_multi_out_tree", "gen_multi_out_50k"])
def test_multi_out_arcs_every_mode(name):
    """Pins with 2+ out-arcs (multi-output cells, a free PI and a feedthrough
    root fanning out into several cells, out-arcs landing in nets of
    different levels): the required-time fold and the gather-form adjoint
    over out-arcs 2+ (diff.py:236-241 scatters them with np.add.at) in every
    run mode, against the oracle and the reference's own outputs."""
    from golden_util import load, raw_of
    g = load(name)
    raw = raw_of(g)
    flat = _check_modes(raw, gamma=float(g["gamma"]))
    assert int(np.diff(flat.mem_out_ptr).max()) >= 2
    dev = ws.DeviceDesign(raw)
    for flags in MODES.values():
        dev.run(flags, gamma=float(g["gamma"]))
        for f in ST_FIELDS:
            assert np.array_equal(dev.get(f), g["st_" + f]), f
        for f in G_FIELDS:
            assert grad_close(dev.get(f), g["g_" + f]), f
    if "gs_loss" in g:
        dev.run(MODES["fused"], gamma=float(g["gamma"]), loss="softplus")
        for f in G_FIELDS:
            assert grad_close(dev.get(f), g["gs_" + f]), f
    dev.close()


def test_lut_pool_beyond_16_bit_ids():
    """A design whose every arc owns its tables (the reference's
    conftest.const_arc style: LUTs deduplicated by object identity only):
    more than 65535 pooled LUTs, same results as the shared-pool design."""
    from golden_util import load, raw_of
    g = load("gen_multi_out_50k")
    raw = raw_of(g)
    A = raw.n_arcs
    ids = np.concatenate([raw.arc_dlut, raw.arc_slut], axis=1).reshape(-1)      # 8 per arc
    assert 8 * A > 65535

    def pack(ptr, flat):
        lens = np.diff(ptr)[ids]
        new_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        new_flat = np.concatenate([flat[ptr[i]:ptr[i + 1]] for i in ids])
        return new_ptr, new_flat
    kw = {}
    for ax in ("s", "l", "t"):
        kw[f"lut_{ax}_ptr"], kw[f"lut_{ax}_flat"] = pack(np.asarray(getattr(raw, f"lut_{ax}_ptr")),
                                                      np.asarray(getattr(raw, f"lut_{ax}_flat")))
    own = np.arange(8 * A, dtype=np.int64).reshape(A, 8)
    big = RawDesign(**{**{f: getattr(raw, f) for f in raw.__dataclass_fields__ if f != "meta"}, **kw,
                       "arc_dlut": own[:, :4], "arc_slut": own[:, 4:]}).normalized()
    assert big.n_luts == 8 * A
    dev = ws.DeviceDesign(big)
    for flags in MODES.values():
        dev.run(flags, gamma=float(g["gamma"]))
        for f in ST_FIELDS:
            assert np.array_equal(dev.get(f), g["st_" + f]), f
        for f in G_FIELDS:
            assert grad_close(dev.get(f), g["g_" + f]), f
    dev.close()
