"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (needs /root/reference, built into oracle/_ref by
oracle/build_ref.sh):

    python tests/golden/make_golden.py

For each case it stores, in tests/golden/<case>.npz:
  * the flat ingest arrays (inputs; ``raw_*``),
  * the reference's FlatDesign index arrays, level schedule and build_csr
    (``flat_*``, ``levels_ptr``/``levels_nets``, ``csr_*``),
  * the reference's run_engine TimingState (``st_*``; compiled backend, which
    test_backends.py:28-39 proves bit-identical to its Python kernels),
    tns/wns,
  * timing_gradients(flat, state=...) GradientState (``g_*``) for the hinge loss
    with the default gamma, plus ``gs_*`` for softplus on selected cases.

Designs: the reference test fixtures (conftest.py:36-127, test_sta.py:242-254),
hand-built root-kind edge cases, and reference-generator designs (C1 of
BASELINE.md plus a random_tree, a heavy-tail and a single-input variant).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.dont_write_bytecode = True
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
sys.path.insert(0, REPO)

import stasim  # noqa: E402  (the reference)
from stasim import (GeneratorConfig, generate_design, flatten, power_law, uniform,  # noqa: E402
                    fixed, build_csr, tns, wns, validate)
from stasim.netlist import (Cell, Design, Endpoint, Lut2D, Net, PrimaryInput,  # noqa: E402
                            TimingArc)
from stasim.warp import run_engine  # noqa: E402
from stasim.sta import run_reference  # noqa: E402
from stasim.diff import timing_gradients, LseConfig  # noqa: E402
from stasim.backend import backend_name  # noqa: E402

from paper_2603_28381_b200.netlist import design_to_raw  # noqa: E402

assert backend_name() == "compiled", "build the reference first: oracle/build_ref.sh"

RAW_FIELDS = ("net_root", "net_mptr", "mem_pin", "mem_parent_pin", "mem_res", "mem_cap",
              "root_cap", "arc_from", "arc_to", "arc_dlut", "arc_slut", "lut_s_ptr",
              "lut_l_ptr", "lut_t_ptr", "lut_s_flat", "lut_l_flat", "lut_t_flat", "pi_pin",
              "pi_arrival", "pi_slew", "ep_pin", "ep_required")
FLAT_FIELDS = ("net_ptr", "net_root", "root_cap", "root_kind", "mem_pin", "mem_parent_loc",
               "mem_res", "mem_cap", "mem_net", "mem_local", "lut_s_ptr", "lut_l_ptr",
               "lut_t_ptr", "lut_s_flat", "lut_l_flat", "lut_t_flat", "arc_from", "arc_to",
               "arc_dlut", "arc_slut", "net_in_ptr", "net_in_arc", "mem_out_ptr",
               "mem_out_arc", "net_m", "net_a", "net_o", "member_of_pin", "root_net_of_pin",
               "pi_pin", "pi_arrival", "pi_slew", "ep_pin", "ep_required", "is_endpoint")
ST_FIELDS = ("load", "net_delay", "impulse", "slew", "arrival", "required", "slack",
             "arc_delay")
G_FIELDS = ("lse_arrival", "arc_weights", "d_arc", "d_edge", "adjoint")
# fixtures that also store run_reference(flat) in its default "sequential" mode
SEQ_CASES = ("edge_kinds", "gen_tree_1200", "gen_heavy_1500", "multi_out", "gen_uniform_tree")


# --- reference test fixtures (restated builders; conftest.py:10-127) -------

def const_lut(v):
    return Lut2D(np.array([0.0]), np.array([0.0]), np.array([[float(v)]]))


def const_arc(f, t, delay, slew=1e-12):
    return TimingArc(f, t, [const_lut(delay) for _ in range(4)],
                     [const_lut(slew) for _ in range(4)])


def zero_net(root, members, parents=None):
    m = len(members)
    return Net(root=root, member_pins=list(members),
               member_parents=list(parents) if parents is not None else [root] * m,
               member_res=np.zeros((m, 4)), member_caps=np.zeros((m, 4)), root_cap=np.zeros(4))


def checked(d):
    v = validate(d)
    assert v == [], [str(x) for x in v]
    return d


def chain_design(n_nets, arc_delay=1.0, required=None, clock_period=1.0, pi_arrival=0.0):
    names, nets, cells, root = ["pi"], [], [], 0
    for i in range(n_nets - 1):
        names += [f"b{i}.in", f"b{i}.out"]
        sink, out = len(names) - 2, len(names) - 1
        nets.append(zero_net(root, [sink]))
        cells.append(Cell([const_arc(sink, out, arc_delay)]))
        root = out
    names.append("po")
    po = len(names) - 1
    nets.append(zero_net(root, [po]))
    req = required if required is not None else clock_period
    return checked(Design(names, cells, nets, [PrimaryInput(0, pi_arrival, 1e-12)],
                          [Endpoint(po, req)], clock_period))


def diamond_design(delay_top=1.0, delay_bot=1.0, merge_delays=(1.0, 1.0), clock_period=10.0):
    names = ["pi", "b.in", "c.in", "b.out", "c.out", "d.in1", "d.in2", "d.out", "po"]
    nets = [zero_net(0, [1, 2]), zero_net(3, [5]), zero_net(4, [6]), zero_net(7, [8])]
    cells = [Cell([const_arc(1, 3, delay_top)]), Cell([const_arc(2, 4, delay_bot)]),
             Cell([const_arc(5, 7, merge_delays[0]), const_arc(6, 7, merge_delays[1])])]
    return checked(Design(names, cells, nets, [PrimaryInput(0, 0.0, 1e-12)],
                          [Endpoint(8, clock_period)], clock_period))


def two_input_design(arrivals=(3.0, 5.0), delays=(2.0, 1.0), required=10.0, clock_period=10.0):
    names = ["pi0", "pi1", "g.in0", "g.in1", "g.out", "po"]
    nets = [zero_net(0, [2]), zero_net(1, [3]), zero_net(4, [5])]
    cells = [Cell([const_arc(2, 4, delays[0]), const_arc(3, 4, delays[1])])]
    return checked(Design(names, cells, nets,
                          [PrimaryInput(0, arrivals[0], 1e-12), PrimaryInput(1, arrivals[1], 1e-12)],
                          [Endpoint(5, required)], clock_period))


def flat_nets_design(member_counts, clock_period=1.0):
    names, nets, pis, eps = [], [], [], []
    for ni, m in enumerate(member_counts):
        root = len(names)
        names.append(f"n{ni}.r")
        sinks = []
        for k in range(m):
            sinks.append(len(names))
            names.append(f"n{ni}.s{k}")
        nets.append(zero_net(root, sinks))
        pis.append(PrimaryInput(root, 0.0, 1e-12))
        eps.extend(Endpoint(s, clock_period) for s in sinks)
    return checked(Design(names, [], nets, pis, eps, clock_period))


def tie_break_design():
    # test_sta.py:242-254
    names = ["pi0", "pi1", "g.in0", "g.in1", "g.out", "po"]
    nets = [zero_net(0, [2]), zero_net(1, [3]), zero_net(4, [5])]
    cells = [Cell([const_arc(2, 4, 1.0, slew=1e-12), const_arc(3, 4, 1.0, slew=5e-12)])]
    return checked(Design(names, cells, nets,
                          [PrimaryInput(0, 0.0, 1e-12), PrimaryInput(1, 0.0, 1e-12)],
                          [Endpoint(5, 10.0)], 10.0))


def edge_kinds_design():
    """Root-kind edge cases: a feedthrough root, a
    PI-rooted RC tree net, a PI that feeds an arc directly, duplicate
    endpoint entries on one pin, an endpoint root, and real 2x3 LUTs."""
    rng = np.random.default_rng(5)
    s_ax = np.array([1e-12, 2e-11, 2e-10])
    l_ax = np.array([1e-15, 1e-13])

    def lut(scale):
        return Lut2D(s_ax, l_ax, scale * (1e-11 + rng.uniform(0.5, 1.5, (3, 2)) * 1e-11))

    def arc(f, t):
        return TimingArc(f, t, [lut(1.0), lut(1.1), lut(1.0), lut(1.2)],
                         [lut(0.5), lut(0.6), lut(0.5), lut(0.7)])

    # pins
    names = ["pi0", "a", "b", "c", "g.out", "d", "e", "pi1", "h.in", "h.out", "q", "r"]
    pi0, a, b, c, gout, d, e, pi1, hin, hout, q, r = range(len(names))
    res = lambda m: rng.uniform(100, 2000, (m, 4))
    cap = lambda m: rng.uniform(0.5e-15, 5e-15, (m, 4))
    nets = [
        # PI-rooted tree net: pi0 -> a -> b, pi0 -> c
        Net(pi0, [a, b, c], [pi0, a, pi0], res(3), cap(3), rng.uniform(1e-15, 3e-15, 4)),
        # feedthrough: b roots a net with member d
        Net(b, [d], [b], res(1), cap(1), rng.uniform(1e-15, 3e-15, 4)),
        # g.out driven by arcs from c, d and pi1 (PI feeding an arc directly)
        Net(gout, [e, hin], [gout, e], res(2), cap(2), rng.uniform(1e-15, 3e-15, 4)),
        Net(hout, [q, r], [hout, hout], res(2), cap(2), rng.uniform(1e-15, 3e-15, 4)),
    ]
    cells = [Cell([arc(c, gout), arc(d, gout), arc(pi1, gout)]), Cell([arc(hin, hout)])]
    T = 2e-10
    pis = [PrimaryInput(pi0, [1e-12, 1e-12, 3e-12, 3e-12], 2e-12),
           PrimaryInput(pi1, [2e-12, 2e-12, 6e-12, 6e-12], 4e-12)]
    eps = [Endpoint(a, [0, 0, 0.8 * T, T]), Endpoint(e, [0, 0, T, T]), Endpoint(q, [0, 0, T, T]), Endpoint(r, [0, 0, T, T]),
           Endpoint(r, [1e-12, 0, 0.5 * T, 0.7 * T]), Endpoint(gout, [0, 0, 0.9 * T, T])]
    return checked(Design(names, cells, nets, pis, eps, T))


def multi_out_design():
    """Pins with more than one out-arc: a two-output cell
    whose input pins each drive 2 arcs, a free primary input (in no net)
    driving arcs into two cells, a feedthrough root that also sources arcs
    into two cells at different levels, a member whose two out-arcs land in
    nets of different levels, a 4-in-arc root (past the register fast path)
    and an endpoint member that also drives arcs."""
    rng = np.random.default_rng(11)
    s_ax = np.array([1e-12, 1.5e-11, 6e-11, 2e-10])
    l_ax = np.array([1e-15, 8e-15, 1e-13])

    def lut(scale):
        return Lut2D(s_ax, l_ax, scale * (1e-11 + rng.uniform(0.5, 1.5, (4, 3)) * 1e-11))

    def arc(f, t):
        return TimingArc(f, t, [lut(1.0), lut(1.1), lut(1.0), lut(1.2)],
                         [lut(0.5), lut(0.6), lut(0.5), lut(0.7)])

    names = ["pi0", "pi1", "x", "y", "z", "a.o1", "a.o2", "f", "g", "h", "k", "l", "b.out",
             "m", "n", "c.out", "d.out", "po1", "po2", "po3"]
    P = {nm: i for i, nm in enumerate(names)}
    res = lambda m: rng.uniform(100, 2000, (m, 4))
    cap = lambda m: rng.uniform(0.5e-15, 5e-15, (m, 4))
    rc = lambda: rng.uniform(1e-15, 3e-15, 4)

    def net(root, members, parents):
        m = len(members)
        return Net(P[root], [P[x] for x in members], [P[x] for x in parents], res(m), cap(m), rc())

    nets = [
        net("pi1", ["x", "y", "z"], ["pi1", "x", "pi1"]),         # PI-rooted tree net
        net("a.o1", ["f", "g"], ["a.o1", "a.o1"]),
        net("a.o2", ["h"], ["a.o2"]),
        net("f", ["k", "l"], ["f", "k"]),                          # feedthrough root (f in a.o1's net)
        net("b.out", ["m", "n"], ["b.out", "b.out"]),
        net("c.out", ["po1"], ["c.out"]),
        net("d.out", ["po2", "po3"], ["d.out", "po2"]),
    ]
    A = lambda f, t: arc(P[f], P[t])
    cells = [
        # two-output cell: x and pi0 -> a.o1, x and y -> a.o2
        Cell([A("x", "a.o1"), A("pi0", "a.o1"), A("x", "a.o2"), A("y", "a.o2")]),
        # 4 in-arcs, one from the free PI
        Cell([A("pi0", "b.out"), A("g", "b.out"), A("h", "b.out"), A("z", "b.out")]),
        Cell([A("f", "c.out"), A("k", "c.out"), A("m", "c.out")]),
        Cell([A("l", "d.out"), A("f", "d.out"), A("n", "d.out"), A("y", "d.out"), A("g", "d.out")]),
    ]
    T = 9e-11
    pis = [PrimaryInput(P["pi0"], [1e-12, 2e-12, 3e-12, 4e-12], 2e-12),
           PrimaryInput(P["pi1"], [2e-12, 2e-12, 5e-12, 6e-12], 3e-12)]
    eps = [Endpoint(P["po1"], [0, 0, 0.6 * T, 0.7 * T]), Endpoint(P["po2"], [0, 0, T, T]),
           Endpoint(P["po3"], [0, 0, 0.5 * T, T]), Endpoint(P["g"], [0, 0, 0.2 * T, 0.3 * T]),
           Endpoint(P["po3"], [1e-12, 0, 0.4 * T, 0.9 * T])]
    return checked(Design(names, cells, nets, pis, eps, T))


def add_multi_out_arcs(design, seed, frac=0.15, wide=(140,), loops=(4, 5, 6, 9, 12, 17)):
    """Mutate a generated design so that many pins drive several arcs: a
    fraction `frac` of the member pins gains an extra arc into the root of a
    net at a strictly higher level (added to the cell that already drives
    that root, so every target keeps a single driving cell; edges that go up
    in level cannot close a cycle).  Roots listed in `wide` / `loops` get that
    many extra in-arcs (the > 128 wide-net task and the > 3 in-arc loop)."""
    rng = np.random.default_rng(seed)
    flat = flatten(design)
    level_of = flat.schedule.level_of
    mem_net = {int(p): int(n) for p, n in zip(flat.mem_pin, flat.mem_net)}
    cell_of_root = {}
    for ci, cell in enumerate(design.cells):
        for a in cell.arcs:
            cell_of_root[a.to_pin] = ci
    roots = [(int(r), int(level_of[n])) for n, r in enumerate(flat.net_root)
             if int(r) in cell_of_root]
    roots.sort(key=lambda x: x[1])
    root_lv = np.array([lv for _, lv in roots])
    members = sorted(mem_net)

    def add(u, r):
        ci = cell_of_root[r]
        tmpl = design.cells[ci].arcs[0]
        design.cells[ci].arcs.append(TimingArc(u, r, list(tmpl.delay_luts), list(tmpl.slew_luts)))

    def targets_above(lv):
        i = int(np.searchsorted(root_lv, lv, side="right"))
        return roots[i:]

    for u in members:
        if rng.random() >= frac:
            continue
        up = targets_above(level_of[mem_net[u]])
        if up:
            add(u, up[int(rng.integers(len(up)))][0])
    top = roots[len(roots) // 2:]
    for k in list(wide) + list(loops):
        r, lv = top[int(rng.integers(len(top)))]
        cand = [u for u in members if level_of[mem_net[u]] < lv]
        for u in rng.choice(cand, size=min(k, len(cand)), replace=False):
            add(int(u), r)
    return checked(design)


def cases():
    out = [
        ("kat_chain6", chain_design(6, arc_delay=1.25), None, False),
        ("kat_chain5_viol", chain_design(5, arc_delay=1.0, required=2.0, clock_period=2.0), None, False),
        ("kat_chain2_req", chain_design(2, arc_delay=4.0, required=10.0, clock_period=10.0), None, False),
        ("kat_diamond", diamond_design(), 1.0, False),
        ("kat_two_input", two_input_design(), None, False),
        ("kat_flat_nets", flat_nets_design([2, 1, 3]), None, False),
        ("kat_tie_break", tie_break_design(), None, False),
        ("edge_kinds", edge_kinds_design(), None, True),
        ("gen_c1_star", generate_design(GeneratorConfig(
            num_cells=2500, fanout=power_law(2.0, 64), depth_target=12, seed=7)), None, True),
        ("gen_tree_1200", generate_design(GeneratorConfig(
            num_cells=1200, fanout=power_law(2.0, 64), depth_target=9, seed=1,
            net_topology="random_tree")), None, True),
        ("gen_heavy_1500", generate_design(GeneratorConfig(
            num_cells=1500, fanout=power_law(2.0, 512), depth_target=8, seed=901)), None, False),
        ("gen_single_in", generate_design(GeneratorConfig(
            num_cells=400, fanout=fixed(2), depth_target=6, seed=3, max_cell_inputs=1,
            net_topology="random_tree")), None, False),
        ("gen_uniform_tree", generate_design(GeneratorConfig(
            num_cells=300, fanout=uniform(1, 9), depth_target=7, seed=5,
            net_topology="random_tree")), None, True),
        ("multi_out", multi_out_design(), None, True),
        ("gen_multi_out_50k", add_multi_out_arcs(generate_design(GeneratorConfig(
            num_cells=12500, fanout=power_law(2.0, 64), depth_target=20, seed=13)), seed=13),
         None, False),
        ("gen_multi_out_tree", add_multi_out_arcs(generate_design(GeneratorConfig(
            num_cells=1500, fanout=power_law(2.0, 200), depth_target=10, seed=17,
            net_topology="random_tree")), seed=17, frac=0.3, wide=(130,), loops=(4, 7)),
         None, True),
    ]
    return out


def dump(name, design, gamma, softplus):
    raw = design_to_raw(design)
    flat = flatten(design)
    st = run_engine(flat, reduce_width=8)
    cfg = LseConfig(gamma) if gamma is not None else None
    gs = timing_gradients(flat, cfg=cfg, loss="hinge", state=st)
    arrs = {"n_pins": np.int64(design.n_pins), "clock_period": np.float64(design.clock_period),
            "gamma": np.float64(gs.gamma), "g_loss": np.float64(gs.loss),
            "tns": np.float64(tns(st, flat)), "wns": np.float64(wns(st, flat))}
    for f in RAW_FIELDS:
        arrs["raw_" + f] = getattr(raw, f)
    for f in FLAT_FIELDS:
        arrs["flat_" + f] = getattr(flat, f)
    lv = flat.schedule.levels
    arrs["levels_ptr"] = np.concatenate([[0], np.cumsum([len(x) for x in lv])]).astype(np.int64)
    arrs["levels_nets"] = (np.concatenate(lv) if lv else np.zeros(0)).astype(np.int64)
    arrs["level_of"] = flat.schedule.level_of
    csr = build_csr(design)
    arrs["csr_pin_list"] = csr.pin_list
    arrs["csr_net_index"] = csr.net_index
    for f in ST_FIELDS:
        arrs["st_" + f] = getattr(st, f)
    for f in G_FIELDS:
        arrs["g_" + f] = getattr(gs, f)
    if name in SEQ_CASES:
        # run_reference's default reduce mode (np.add.reduceat root loads)
        sq = run_reference(flat)
        for f in ST_FIELDS:
            arrs["sq_" + f] = getattr(sq, f)
    if softplus:
        gp = timing_gradients(flat, cfg=cfg, loss="softplus", state=st)
        arrs["gs_loss"] = np.float64(gp.loss)
        for f in G_FIELDS:
            arrs["gs_" + f] = getattr(gp, f)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrs)
    return design.n_pins


if __name__ == "__main__":
    total = 0
    only = set(sys.argv[1:])
    for name, d, gamma, sp in cases():
        if only and name not in only:
            continue
        n = dump(name, d, gamma, sp)
        sz = os.path.getsize(os.path.join(HERE, name + ".npz"))
        total += sz
        print(f"{name}: {n} pins, {sz / 1024:.0f} KiB")
    print(f"total {total / 1024:.0f} KiB")
