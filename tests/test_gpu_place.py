"""GPU parity of the position model and position gradients (ws_place.cu,
WS_RUN_WIRE | WS_RUN_POSGRAD) against the CPU oracle, which
test_place_oracle.py pins by finite differences.

Through the C ABI: the wire RC (mem_res / mem_cap written by k_wire) and the
hard pass on it are bit-exact; d_slew, d_root_cap, d_res, d_cap, d_len and
d_xy follow the oracle's operation order except for the member sums of the
root-slew terms (a fixed warp-shuffle order); with the LSE exp/log ulps that
is the only source of difference.  They are held to 1e-9 relative (with a
1e-9 x max floor), five orders tighter than north_star's 1e-4 bar; d_xy
sums signed edge terms, so ulp-level input differences can grow by the
cancellation factor.
"""

import numpy as np
import pytest

from golden_util import ST_FIELDS, grad_close, load, raw_of
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G, placement as PL
from oracle import oracle as O

pytestmark = pytest.mark.gpu

PG_FIELDS = (("d_slew", "d_slew"), ("d_root_cap", "d_root_cap"), ("d_res", "d_res"),
             ("d_cap", "d_cap"), ("d_len", "g_len"), ("d_xy", "d_xy"))


def oracle_place(raw, pl, loss="hinge"):
    flat = O.flatten_raw(raw)
    res, cap = O.wire(flat, pl.xy, pl.res0, pl.cap0, pl.wire.r_unit, pl.wire.c_unit)
    f = O.with_values(flat, mem_res=res, mem_cap=cap)
    st = O.run_engine(f)
    gr = O.timing_gradients(f, st, gamma=0.01 * flat.clock_period, loss=loss)
    pg = O.position_gradients(f, st, gr, pl.xy, pl.wire.r_unit, pl.wire.c_unit)
    return flat, res, cap, st, gr, pg


def check(dev, corner, raw, pl, loss="hinge", rtol=1e-9):
    flat, res, cap, st, gr, pg = oracle_place(raw, pl, loss)
    t_res = dev.value_tensor("mem_res", corner).cpu().numpy()
    t_cap = dev.value_tensor("mem_cap", corner).cpu().numpy()
    assert np.array_equal(t_res, res) and np.array_equal(t_cap, cap)
    for f in ST_FIELDS:
        assert np.array_equal(dev.get(f, corner), getattr(st, f)), f
    tns, wns, lossv = dev.summary(corner)
    assert tns == O.tns(st, flat) and wns == O.wns(st, flat)
    assert abs(lossv - gr.loss) <= 1e-9 * abs(gr.loss)
    for name, oname in PG_FIELDS:
        a, b = dev.get(name, corner), getattr(pg, oname)
        if not grad_close(a, b, rtol=rtol):
            d = np.abs(a - b)
            i = int(np.argmax(d / np.maximum(np.abs(b), 1e-9 * np.abs(b).max())))
            raise AssertionError(f"{name}: worst rel {d.flat[i] / max(abs(b.flat[i]), 1e-300):.3e} "
                                 f"at {i} ({a.flat[i]!r} vs {b.flat[i]!r}), max|b| {np.abs(b).max():.3e}")
    return pg


def gen(n, topo="star", seed=3):
    return G.generate_raw(G.GeneratorConfig(num_cells=n, fanout=G.power_law(2.0, 16),
                                            depth_target=8, seed=seed, net_topology=topo))


@pytest.mark.parametrize("topo", ["star", "random_tree"])
@pytest.mark.parametrize("loss", ["hinge", "softplus"])
def test_place_step_matches_oracle(topo, loss):
    raw = gen(600, topo)
    pl = PL.synthetic_placement(raw, seed=2)
    dev = ws.DeviceDesign(raw)
    timer = PL.PlacementTimer(dev, pl, loss=loss)
    timer.step()
    check(dev, 0, raw, pl, loss)
    dev.close()


def test_place_edge_kinds():
    raw = raw_of(load("edge_kinds"))
    pl = PL.synthetic_placement(raw, seed=5)
    dev = ws.DeviceDesign(raw)
    PL.PlacementTimer(dev, pl, loss="softplus").step()
    check(dev, 0, raw, pl, "softplus")
    dev.close()


def test_place_c1_graph_replay_new_positions():
    """Graph-captured steps with changing positions equal fresh oracle runs."""
    raw = G.generate_raw(G.config_c1())
    pl = PL.synthetic_placement(raw, seed=7)
    dev = ws.DeviceDesign(raw)
    timer = PL.PlacementTimer(dev, pl, graph=True)
    rng = np.random.default_rng(11)
    for it in range(3):
        xy = pl.xy + rng.normal(0.0, 2.0, pl.xy.shape) * (it > 0)
        timer.step(xy)
        pl2 = PL.Placement(xy=xy, res0=pl.res0, cap0=pl.cap0, wire=pl.wire,
                           cell_of_pin=pl.cell_of_pin, cell_xy=pl.cell_xy, pin_offset=pl.pin_offset)
        check(dev, 0, raw, pl2)
    dev.close()


def test_place_corners_independent():
    raw = gen(400, "random_tree", seed=9)
    pa = PL.synthetic_placement(raw, seed=1)
    pb = PL.synthetic_placement(raw, seed=2)
    dev = ws.DeviceDesign(raw, n_corners=2)
    ta = PL.PlacementTimer(dev, pa, corner=0)
    tb = PL.PlacementTimer(dev, pb, corner=1)
    dev.run(PL.PlacementTimer.FLAGS, corner=0, n_corners=2)
    check(dev, 0, raw, pa)
    check(dev, 1, raw, pb)
    assert ta.corner == 0 and tb.corner == 1
    dev.close()


def test_place_identity_without_positions():
    """With the default model (xy = 0, wire = 0, base RC = the design's RC)
    RUN_WIRE reproduces the design's values: the pass equals run_engine."""
    raw = gen(300)
    dev = ws.DeviceDesign(raw)
    dev.run(_lib.RUN_WIRE | _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED
            | _lib.RUN_POSGRAD)
    st = O.run_engine(O.flatten_raw(raw))
    for f in ST_FIELDS:
        assert np.array_equal(dev.get(f), getattr(st, f)), f
    assert np.all(dev.get("d_xy") == 0.0)     # all positions equal: sign(0) = 0
    dev.close()


def test_posgrad_needs_grad_pass():
    raw = gen(100)
    dev = ws.DeviceDesign(raw)
    with pytest.raises(RuntimeError):
        dev.run(_lib.RUN_HARD | _lib.RUN_POSGRAD)
    dev.close()


def test_place_c3_full_size():
    """C3 (2.49M pins) placement step: hard pass bit-exact on the wire RC,
    position gradients vs the oracle."""
    raw = G.generate_raw(G.config_c3())
    pl = PL.synthetic_placement(raw, seed=3)
    dev = ws.DeviceDesign(raw)
    PL.PlacementTimer(dev, pl).step()
    pg = check(dev, 0, raw, pl)
    assert np.count_nonzero(pg.d_xy) > 0
    dev.close()


def test_place_c4_loop_c3():
    """C4: 200 graph-replayed placement invocations on C3 with perturbed
    cell positions (seed 1000 + t); invocations 0, 99 and 199 equal fresh
    oracle runs on the same coordinates."""
    raw = G.generate_raw(G.config_c3())
    pl = PL.synthetic_placement(raw, seed=3)
    dev = ws.DeviceDesign(raw)
    timer = PL.PlacementTimer(dev, pl)
    for t in range(200):
        rng = np.random.default_rng(1000 + t)
        xy = pl.xy + 0.5 * rng.standard_normal(pl.cell_xy.shape)[pl.cell_of_pin]
        timer.step(xy)
        if t in (0, 99, 199):
            check(dev, 0, raw, PL.Placement(xy=xy, res0=pl.res0, cap0=pl.cap0, wire=pl.wire,
                                            cell_of_pin=pl.cell_of_pin, cell_xy=pl.cell_xy,
                                            pin_offset=pl.pin_offset))
    dev.close()


def test_place_c2_heavy_tail():
    """C2 (995,808 pins, fanout up to 508; RC-tree variant off): the member
    rounds of big nets and the chunked pass tasks under the position model."""
    raw = G.generate_raw(G.config_c2())
    pl = PL.synthetic_placement(raw, seed=4)
    dev = ws.DeviceDesign(raw)
    PL.PlacementTimer(dev, pl, loss="softplus").step()
    check(dev, 0, raw, pl, "softplus")
    dev.close()


def test_place_c1_tree_persistent_pass_equivalence():
    """The position sweep after a fused pass equals the one after a
    sequential pass (the sweep reads only the finished pass state)."""
    raw = G.generate_raw(G.config_c1("random_tree"))
    pl = PL.synthetic_placement(raw, seed=8)
    dev = ws.DeviceDesign(raw, n_corners=2)
    for k in (0, 1):
        dev.set_values(k, res0=pl.res0, cap0=pl.cap0, wire=pl.wire.packed(), xy=pl.xy)
    base = _lib.RUN_WIRE | _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_POSGRAD
    dev.run(base | _lib.RUN_FUSED, corner=0)
    dev.run(base, corner=1)
    for f in ("d_xy", "d_res", "d_cap", "d_slew", "d_root_cap"):
        assert np.array_equal(dev.get(f, 0), dev.get(f, 1)), f
    check(dev, 0, raw, pl)
    dev.close()


def test_descend_reduces_the_timing_loss():
    """Gradient steps on cell positions (dL/dxy reduced to cells) lower the
    hinge-TNS loss of a C1 design."""
    raw = G.generate_raw(G.config_c1())
    pl = PL.synthetic_placement(raw, seed=5)
    dev = ws.DeviceDesign(raw)
    timer = PL.PlacementTimer(dev, pl)
    hist = PL.descend(timer, pl, steps=15, step_um=2.0)
    losses = [h[0] for h in hist]
    assert losses[-1] < losses[0]
    assert min(losses[1:]) < losses[0]
    dev.close()


@pytest.mark.parametrize("name", ["multi_out", "gen_multi_out_tree", "gen_multi_out_50k"])
@pytest.mark.parametrize("loss", ["hinge", "softplus"])
def test_place_multi_out_arcs(name, loss):
    """Position gradients on pins with several out-arcs (the slew adjoint
    gsa of every out-arc is summed into its source pin)."""
    raw = raw_of(load(name))
    pl = PL.synthetic_placement(raw, seed=7)
    dev = ws.DeviceDesign(raw)
    PL.PlacementTimer(dev, pl, loss=loss).step()
    check(dev, 0, raw, pl, loss)
    dev.close()


def _sweep_case(case):
    if case == "c1":
        return G.generate_raw(G.config_c1())
    if case == "tree":
        return gen(600, "random_tree")
    if case in ("edge_kinds", "multi_out", "gen_multi_out_tree"):
        return raw_of(load(case))
    topo = "star" if case == "big_star" else "random_tree"
    return G.generate_raw(G.GeneratorConfig(num_cells=2500, fanout=G.power_law(1.1, 300), depth_target=5,
                                            max_cell_inputs=180, seed=13, net_topology=topo))


@pytest.mark.parametrize("case", ["c1", "tree", "edge_kinds", "multi_out", "gen_multi_out_tree",
                                  "big_star", "big_tree"])
def test_fused_sweep_equals_stream_sweep(case, monkeypatch):
    """The fused mode runs the position-gradient sweep inside the backward
    level kernels (k_bwd<..., PG>); WS_PG_SWEEP=stream runs the stand-alone
    k_pg_mem / k_pg_level kernels on the second stream.  Same bodies
    (ws_pg.cuh), same order: bitwise equal, including chunked big star nets
    (> TASK_M members), TK_WIDE nets and TK_LOOP RC trees; the fused one also
    matches the oracle."""
    raw = _sweep_case(case)
    pl = PL.synthetic_placement(raw, seed=4)
    out = {}
    for mode in ("fused", "stream"):
        if mode == "stream":
            monkeypatch.setenv("WS_PG_SWEEP", "stream")
        else:
            monkeypatch.delenv("WS_PG_SWEEP", raising=False)
        dev = ws.DeviceDesign(raw)
        PL.PlacementTimer(dev, pl, graph=mode == "fused").step()
        out[mode] = {f: dev.get(f) for f, _ in PG_FIELDS}
        if mode == "fused" and case in ("c1", "big_star", "edge_kinds"):
            check(dev, 0, raw, pl)
        dev.close()
    for f, _ in PG_FIELDS:
        assert np.array_equal(out["fused"][f], out["stream"][f], equal_nan=True), f


@pytest.mark.parametrize("nc", [5, 16])
def test_place_candidate_batch_bitwise_single(nc):
    """A batch of nc placement candidates in one ws_run (k_wire, the pass and
    the fused sweep with blockIdx.y = candidate; the 4-block level-kernel
    variants for nc >= 4 outside the sweep) equals nc single-candidate runs
    bit for bit, chunked big star nets and wide nets included; candidate 0
    also matches the oracle."""
    raw = _sweep_case("big_star")
    pls = [PL.synthetic_placement(raw, seed=20 + k) for k in range(nc)]
    dev = ws.DeviceDesign(raw, n_corners=nc)
    timers = [PL.PlacementTimer(dev, pls[k], corner=k, graph=False) for k in range(nc)]
    dev.run(PL.PlacementTimer.FLAGS, corner=0, n_corners=nc)
    batch = [{f: dev.get(f, k) for f, _ in PG_FIELDS} for k in range(nc)]
    check(dev, 0, raw, pls[0])
    for k in range(nc):
        timers[k].step()
        for f, _ in PG_FIELDS:
            assert np.array_equal(dev.get(f, k), batch[k][f], equal_nan=True), (k, f)
    dev.close()


def test_place_candidate_batch_split_streams_bitwise():
    """Placement-candidate batches of >= WS_SPLIT candidates run as two half
    batches on two streams (fused sweep included): bitwise the lockstep
    batch (WS_SPLIT=0)."""
    import os
    raw = _sweep_case("big_star")
    nc = 8
    pls = [PL.synthetic_placement(raw, seed=40 + k) for k in range(nc)]

    def run(split):
        old = os.environ.get("WS_SPLIT")
        os.environ["WS_SPLIT"] = split
        try:
            dev = ws.DeviceDesign(raw, n_corners=nc)
        finally:
            if old is None:
                del os.environ["WS_SPLIT"]
            else:
                os.environ["WS_SPLIT"] = old
        timers = [PL.PlacementTimer(dev, pls[k], corner=k, graph=False) for k in range(nc)]
        dev.run(PL.PlacementTimer.FLAGS, corner=0, n_corners=nc)
        out = [{f: dev.get(f, k) for f, _ in PG_FIELDS} for k in range(nc)]
        dev.close()
        del timers
        return out

    a, b = run("0"), run("4")
    for k in range(nc):
        for f, _ in PG_FIELDS:
            assert np.array_equal(a[k][f], b[k][f], equal_nan=True), (k, f)
