"""Pin the position-gradient oracle (oracle/sta_oracle.c: orc_wire,
orc_posgrad_level, orc_pos_reduce) by central finite differences.

The reference has no position model (SPEC.md non-goal), so there are no
golden vectors for this path.  The FD target is built only from
reference-restated functions: positions -> wire RC -> run_engine (bit-exact
to the reference, test_oracle_golden.py) -> timing_gradients loss.  The
analytic gradient must match it to 1e-6 relative on the largest
coordinates (observed ~1e-10) on star and RC-tree nets, both loss kinds, and
on the reference's edge-kind fixture (PI roots, feedthrough roots, free pins).
"""

import numpy as np
import pytest

from golden_util import load, raw_of
from oracle import oracle as O
from paper_2603_28381_b200 import generator as G
from paper_2603_28381_b200 import placement as PL


def _setup(raw, loss):
    pl = PL.synthetic_placement(raw, seed=1)
    flat = O.flatten_raw(raw)
    assert np.array_equal(O.parent_pins(flat), np.asarray(raw.mem_parent_pin, np.int64))
    ru, cu = pl.wire.r_unit, pl.wire.c_unit
    gamma = 0.01 * flat.clock_period
    res, cap = O.wire(flat, pl.xy, pl.res0, pl.cap0, ru, cu)
    f = O.with_values(flat, mem_res=res, mem_cap=cap)
    st = O.run_engine(f)
    gr = O.timing_gradients(f, st, gamma=gamma, loss=loss)
    pg = O.position_gradients(f, st, gr, pl.xy, ru, cu)
    return pl, flat, gamma, res, cap, gr, pg


def _fd_xy(pl, flat, gamma, loss, fi, eps):
    xp = pl.xy.copy().ravel()
    xm = xp.copy()
    xp[fi] += eps
    xm[fi] -= eps
    lf = lambda x: O.placed_loss(flat, x.reshape(-1, 2), pl.res0, pl.cap0, pl.wire.r_unit,
                                 pl.wire.c_unit, gamma, loss)
    return (lf(xp) - lf(xm)) / (2 * eps)


def _check_xy(raw, loss, n_top=8, eps=1e-2):
    pl, flat, gamma, res, cap, gr, pg = _setup(raw, loss)
    g = pg.d_xy.ravel()
    assert np.all(np.isfinite(g))
    assert np.abs(g).max() > 0, "design has no position sensitivity"
    for fi in np.argsort(-np.abs(g))[:n_top]:
        fd = _fd_xy(pl, flat, gamma, loss, fi, eps)
        assert abs(fd - g[fi]) <= 1e-6 * abs(g[fi]), (fi, fd, g[fi])
    # coordinates the analytic gradient calls flat are flat
    zeros = np.flatnonzero(g == 0)
    for fi in zeros[:: max(1, len(zeros) // 3)][:3]:
        fd = _fd_xy(pl, flat, gamma, loss, fi, eps)
        assert abs(fd) <= 1e-9 * np.abs(g).max(), (fi, fd)
    return pg


@pytest.mark.parametrize("topo", ["star", "random_tree"])
@pytest.mark.parametrize("loss", ["hinge", "softplus"])
def test_position_gradient_fd(topo, loss):
    cfg = G.GeneratorConfig(num_cells=300, fanout=G.power_law(2.0, 16), depth_target=8, seed=3,
                            net_topology=topo)
    _check_xy(G.generate_raw(cfg), loss)


def test_position_gradient_fd_edge_kinds():
    raw = raw_of(load("edge_kinds"))
    _check_xy(raw, "softplus", n_top=6, eps=1e-3)


@pytest.mark.parametrize("topo", ["star", "random_tree"])
def test_rc_gradient_fd(topo):
    """d_res / d_cap against FD of the loss in the RC values themselves."""
    cfg = G.GeneratorConfig(num_cells=200, fanout=G.power_law(2.0, 12), depth_target=6, seed=5,
                            net_topology=topo)
    raw = G.generate_raw(cfg)
    pl, flat, gamma, res, cap, gr, pg = _setup(raw, "hinge")

    def loss_of(r, c):
        f = O.with_values(flat, mem_res=r, mem_cap=c)
        return O.timing_gradients(f, O.run_engine(f), gamma=gamma).loss

    for name, arr, grad in (("res", res, pg.d_res), ("cap", cap, pg.d_cap)):
        for fi in np.argsort(-np.abs(grad).ravel())[:4]:
            k, j = divmod(int(fi), 2)
            h = 1e-6 * arr[k, 2 + j]
            up, dn = arr.copy(), arr.copy()
            up[k, 2 + j] += h
            dn[k, 2 + j] -= h
            args = (up, cap) if name == "res" else (res, up)
            argm = (dn, cap) if name == "res" else (res, dn)
            fd = (loss_of(*args) - loss_of(*argm)) / (2 * h)
            assert abs(fd - grad[k, j]) <= 1e-6 * abs(grad[k, j]), (name, k, j, fd, grad[k, j])


def test_interp_grad_matches_fd():
    raw = G.generate_raw(G.GeneratorConfig(num_cells=50, depth_target=3, seed=1))
    flat = O.flatten_raw(raw)
    s_ax = flat.lut_s_flat[flat.lut_s_ptr[0]:flat.lut_s_ptr[1]]
    l_ax = flat.lut_l_flat[flat.lut_l_ptr[0]:flat.lut_l_ptr[1]]
    rng = np.random.default_rng(0)
    for _ in range(20):
        qs = rng.uniform(s_ax[0], s_ax[-1])
        ql = rng.uniform(l_ax[0], l_ax[-1])
        ds, dl = O.interp_grad(flat, 0, qs, ql)
        hs, hl = 1e-7 * qs, 1e-7 * ql
        fs = (O.interpolate(flat, 0, qs + hs, ql) - O.interpolate(flat, 0, qs - hs, ql)) / (2 * hs)
        fl = (O.interpolate(flat, 0, qs, ql + hl) - O.interpolate(flat, 0, qs, ql - hl)) / (2 * hl)
        assert abs(ds - fs) <= 1e-6 * abs(fs) and abs(dl - fl) <= 1e-6 * abs(fl)
    # outside the table: clamped, flat
    ds, dl = O.interp_grad(flat, 0, s_ax[-1] * 2, l_ax[0] / 2)
    assert ds == 0.0 and dl == 0.0


def test_wire_model_identity_and_lengths():
    raw = G.generate_raw(G.GeneratorConfig(num_cells=100, depth_target=4, seed=2))
    flat = O.flatten_raw(raw)
    pl = PL.synthetic_placement(raw, seed=4)
    res, cap = O.wire(flat, pl.xy, pl.res0, pl.cap0, np.zeros(4), np.zeros(4))
    assert np.array_equal(res, pl.res0) and np.array_equal(cap, pl.cap0)
    res, cap = O.wire(flat, pl.xy, pl.res0, pl.cap0, pl.wire.r_unit, pl.wire.c_unit)
    ln = PL.member_lengths(raw, pl.xy)
    assert np.allclose(res, pl.res0 + ln[:, None] * pl.wire.r_unit[None, :], rtol=1e-15)
    # calibration keeps the mean RC of the generated design
    assert np.allclose(res.mean(axis=0), np.asarray(raw.mem_res).mean(axis=0), rtol=1e-12)
    assert np.allclose(cap.mean(axis=0), np.asarray(raw.mem_cap).mean(axis=0), rtol=1e-12)


@pytest.mark.parametrize("name", ["kat_chain6", "kat_diamond", "kat_two_input", "kat_tie_break",
                                  "kat_flat_nets", "gen_tree_1200", "gen_heavy_1500",
                                  "gen_single_in", "gen_uniform_tree", "multi_out",
                                  "gen_multi_out_tree"])
def test_position_gradient_fd_golden_designs(name):
    """FD pinning on the reference's own test designs (the golden fixtures'
    netlists, softplus loss so every endpoint contributes)."""
    raw = raw_of(load(name))
    pl, flat, gamma, res, cap, gr, pg = _setup(raw, "softplus")
    g = pg.d_xy.ravel()
    if not np.abs(g).max() > 0:
        pytest.skip("no position sensitivity in this design")
    for fi in np.argsort(-np.abs(g))[:4]:
        fd = _fd_xy(pl, flat, gamma, "softplus", fi, 1e-3)
        assert abs(fd - g[fi]) <= 1e-5 * abs(g[fi]), (name, fi, fd, g[fi])
