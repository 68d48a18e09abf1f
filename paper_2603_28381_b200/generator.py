"""Seeded synthetic netlist generator (workload source, not the timed path).

Produces the reference generator's designs bit for bit
(/root/reference/pkg/src/stasim/generator.py:205-359) but straight into the
flat ``RawDesign`` arrays the device ingests, without building 10^6 Python
objects.  Same PRNG plan: ``SeedSequence(seed).spawn(5)`` into Philox
sub-streams (generator.py:208-214); every draw is taken from the same stream
in the same order, so bulk draws (``rng.random(n)``, ``integers(size=n)``)
reproduce the reference's scalar calls exactly.  The one inherently
sequential part, spare-input wiring (generator.py:296-311), stays a scalar
loop.  Bit-identity with the reference is checked in
tests/test_generator_port.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .netlist import N_COND, RawDesign, pack_luts, raw_to_design

NOMINAL_STAGE_DELAY = 60e-12  # generator.py:26
N_CELL_CLASSES = 8            # generator.py:158


@dataclass
class FanoutDist:
    """fixed(k), uniform(lo, hi) or power_law(alpha, max) (generator.py:29-89)."""

    kind: str
    k: int = 1
    lo: int = 1
    hi: int = 1
    alpha: float = 2.0
    max: int = 1

    def __post_init__(self):
        if self.kind not in ("fixed", "uniform", "power_law"):
            raise ValueError(f"unknown fanout distribution {self.kind!r}")
        if self.kind == "fixed" and self.k < 1:
            raise ValueError("fixed fanout must be >= 1")
        if self.kind == "uniform" and not (1 <= self.lo <= self.hi):
            raise ValueError("uniform fanout needs 1 <= lo <= hi")
        if self.kind == "power_law" and not (self.alpha > 0 and self.max >= 1):
            raise ValueError("power_law fanout needs alpha > 0 and max >= 1")

    def sample(self, rng: np.random.Generator, n: int) -> np.ndarray:
        if self.kind == "fixed":
            return np.full(n, self.k, dtype=np.int64)
        if self.kind == "uniform":
            return rng.integers(self.lo, self.hi + 1, size=n, dtype=np.int64)
        support = np.arange(1, self.max + 1, dtype=np.float64)
        pmf = support ** (-self.alpha)
        pmf /= pmf.sum()
        return rng.choice(np.arange(1, self.max + 1, dtype=np.int64), size=n, p=pmf)

    def to_doc(self):
        if self.kind == "fixed":
            return {"kind": "fixed", "k": self.k}
        if self.kind == "uniform":
            return {"kind": "uniform", "lo": self.lo, "hi": self.hi}
        return {"kind": "power_law", "alpha": self.alpha, "max": self.max}


def fixed(k):
    return FanoutDist("fixed", k=k)


def uniform(lo, hi):
    return FanoutDist("uniform", lo=lo, hi=hi)


def power_law(alpha, max_fanout):
    return FanoutDist("power_law", alpha=alpha, max=max_fanout)


@dataclass
class GeneratorConfig:
    """Same fields, defaults and validation as generator.py:104-130."""

    num_cells: int
    fanout: FanoutDist = field(default_factory=lambda: power_law(2.0, 64))
    depth_target: int = 8
    lut_grid_size: int = 5
    seed: int = 0
    max_cell_inputs: int = 3
    clock_scale: float = 1.0
    net_topology: str = "star"

    def __post_init__(self):
        if self.num_cells < 1:
            raise ValueError("num_cells must be >= 1")
        if self.depth_target < 1:
            raise ValueError("depth_target must be >= 1")
        if self.depth_target > self.num_cells:
            raise ValueError(
                f"infeasible config: depth_target {self.depth_target} exceeds num_cells {self.num_cells}")
        if self.lut_grid_size < 1:
            raise ValueError("lut_grid_size must be >= 1")
        if self.max_cell_inputs < 1:
            raise ValueError("max_cell_inputs must be >= 1")
        if not (self.clock_scale > 0):
            raise ValueError("clock_scale must be > 0")
        if self.net_topology not in ("star", "random_tree"):
            raise ValueError(f"unknown net topology {self.net_topology!r}")

    def to_doc(self):
        return {"num_cells": self.num_cells, "fanout": self.fanout.to_doc(),
                "depth_target": self.depth_target, "lut_grid_size": self.lut_grid_size,
                "seed": self.seed, "max_cell_inputs": self.max_cell_inputs,
                "clock_scale": self.clock_scale, "net_topology": self.net_topology}


class _Table:
    __slots__ = ("slew_axis", "load_axis", "table")

    def __init__(self, s, l, t):
        self.slew_axis, self.load_axis, self.table = s, l, t


def _lut_library(rng, grid):
    """Per class: [rise_d, fall_d, rise_d, fall_d] delay and the matching
    slew tables; early/late share one table object (generator.py:161-195).
    Draw order per class: base, fall_ratio, s_coef, r_eff, cross, sl_base,
    sl_s_coef, sl_r_eff."""
    slew_axis = np.geomspace(1e-12, 2e-10, grid) if grid > 1 else np.array([5e-12])
    load_axis = np.geomspace(5e-16, 3e-13, grid) if grid > 1 else np.array([5e-15])
    lib = []
    for _ in range(N_CELL_CLASSES):
        base = rng.uniform(20e-12, 80e-12)
        fall_ratio = rng.uniform(0.95, 1.15)
        s_coef = rng.uniform(0.15, 0.35)
        r_eff = rng.uniform(100.0, 600.0)
        cross = rng.uniform(0.02, 0.08)
        sl_base = rng.uniform(2e-12, 8e-12)
        sl_s_coef = rng.uniform(0.1, 0.3)
        sl_r_eff = rng.uniform(50.0, 300.0)
        s_col = slew_axis[:, None]
        l_row = load_axis[None, :]
        cross_term = cross * base * (s_col / slew_axis[-1]) * (l_row / load_axis[-1])
        tabs = {}
        for edge, ratio in (("rise", 1.0), ("fall", fall_ratio)):
            d = ratio * base + s_coef * s_col + r_eff * l_row + cross_term
            s = ratio * sl_base + sl_s_coef * s_col + sl_r_eff * l_row
            tabs[edge] = (_Table(slew_axis, load_axis, d + 0 * l_row),
                          _Table(slew_axis, load_axis, s + 0 * l_row))
        lib.append(([tabs["rise"][0], tabs["fall"][0], tabs["rise"][0], tabs["fall"][0]],
                    [tabs["rise"][1], tabs["fall"][1], tabs["rise"][1], tabs["fall"][1]]))
    return lib


def _unif(lo, hi, u):
    """numpy's uniform(lo, hi) = lo + (hi - lo) * next_double."""
    return lo + (hi - lo) * u


def generate_raw(cfg: GeneratorConfig) -> RawDesign:
    """Deterministic design for cfg, as flat arrays (the reference's design
    for the same cfg, pin ids, arc order and values identical)."""
    ss = np.random.SeedSequence(cfg.seed)
    kids = ss.spawn(5)
    rng_fan = np.random.Generator(np.random.Philox(kids[0]))
    rng_wire = np.random.Generator(np.random.Philox(kids[1]))
    rng_rc = np.random.Generator(np.random.Philox(kids[2]))
    rng_lut = np.random.Generator(np.random.Philox(kids[3]))
    rng_pin = np.random.Generator(np.random.Philox(kids[4]))

    nc = cfg.num_cells
    depth = cfg.depth_target
    max_in = cfg.max_cell_inputs
    layer_sizes = [len(c) for c in np.array_split(np.arange(nc), depth)]
    layer_start = np.concatenate([[0], np.cumsum(layer_sizes)]).astype(np.int64)
    clock_period = cfg.clock_scale * depth * NOMINAL_STAGE_DELAY

    lib = _lut_library(rng_lut, cfg.lut_grid_size)
    cell_class = rng_lut.integers(0, N_CELL_CLASSES, size=nc)

    # pins 0..nc-1 are the cell outputs (generator.py:237-244)
    n_pins = nc
    cell_inputs = [[] for _ in range(nc)]

    # first-layer inputs are primary inputs (generator.py:247-256)
    l0 = layer_sizes[0]
    n_in0 = rng_wire.integers(1, max_in + 1, size=l0)
    n_pi = int(n_in0.sum())
    pi_pin = np.arange(n_pins, n_pins + n_pi, dtype=np.int64)
    pos = n_pins
    for c in range(l0):
        k = int(n_in0[c])
        cell_inputs[c].extend(range(pos, pos + k))
        pos += k
    n_pins = pos
    u = rng_pin.random(3 * n_pi).reshape(n_pi, 3) if n_pi else np.zeros((0, 3))
    base = _unif(0.0, 10e-12, u[:, 0])
    late = base + _unif(0.0, 5e-12, u[:, 1])
    pi_arrival = np.stack([base, base, late, late], axis=1)
    pi_slew = np.repeat(_unif(1e-12, 5e-12, u[:, 2])[:, None], N_COND, axis=1)

    fanouts = np.concatenate([cfg.fanout.sample(rng_fan, s) for s in layer_sizes])

    net_sinks = [[] for _ in range(nc)]
    ep_pins = []
    fanout_bumps = 0
    n_inputs = np.zeros(nc, dtype=np.int64)
    n_inputs[:l0] = n_in0
    n_inputs = n_inputs.tolist()
    for li in range(depth):
        d0, d1 = int(layer_start[li]), int(layer_start[li + 1])
        drivers = np.arange(d0, d1, dtype=np.int64)
        if li + 1 < depth:
            c0, c1 = int(layer_start[li + 1]), int(layer_start[li + 2])
        else:
            c0 = c1 = 0
        n_cons = c1 - c0
        conn = np.repeat(drivers, fanouts[d0:d1])
        rng_wire.shuffle(conn)
        conn = conn.tolist()
        while len(conn) < n_cons:  # coverage (generator.py:282-286)
            extra = int(rng_wire.choice(drivers))
            fanouts[extra] += 1
            conn.append(extra)
            fanout_bumps += 1
        order = np.arange(c0, c1, dtype=np.int64)
        rng_wire.shuffle(order)
        order = order.tolist()
        open_cells = []
        for j, c in enumerate(order):
            p = n_pins
            n_pins += 1
            cell_inputs[c].append(p)
            n_inputs[c] += 1
            net_sinks[conn[j]].append(p)
            if max_in > 1:
                open_cells.append(c)
        integers = rng_wire.integers
        for d in conn[len(order):]:
            c = -1
            while open_cells:
                pick = int(integers(0, len(open_cells)))
                oc = open_cells[pick]
                if n_inputs[oc] < max_in:
                    c = oc
                    break
                open_cells[pick] = open_cells[-1]
                open_cells.pop()
            p = n_pins
            n_pins += 1
            if c < 0:
                ep_pins.append(p)
            else:
                cell_inputs[c].append(p)
                n_inputs[c] += 1
            net_sinks[d].append(p)

    # arcs: cell order, input order (generator.py:316-320)
    n_in = np.asarray(n_inputs, dtype=np.int64)
    arc_from = np.fromiter((p for ins in cell_inputs for p in ins), dtype=np.int64,
                           count=int(n_in.sum()))
    arc_to = np.repeat(np.arange(nc, dtype=np.int64), n_in)
    arc_cls = cell_class[arc_to]
    # LUT pool in first-appearance order: per class [rise_d, rise_s, fall_d, fall_s]
    first = {}
    for k in arc_cls.tolist():
        if k not in first:
            first[k] = len(first)
            if len(first) == N_CELL_CLASSES:
                break
    luts = []
    cls_slot = np.zeros(N_CELL_CLASSES, dtype=np.int64)
    for k, slot in sorted(first.items(), key=lambda kv: kv[1]):
        dl, sl = lib[k]
        cls_slot[k] = len(luts)
        luts += [dl[0], sl[0], dl[1], sl[1]]
    base_id = cls_slot[arc_cls]
    arc_dlut = np.stack([base_id, base_id + 2, base_id, base_id + 2], axis=1)
    arc_slut = arc_dlut + 1
    s_ptr, l_ptr, t_ptr, s_flat, l_flat, t_flat = pack_luts(luts)

    # nets (generator.py:322-344)
    m_per = np.fromiter((len(s) for s in net_sinks), dtype=np.int64, count=nc)
    net_mptr = np.zeros(nc + 1, dtype=np.int64)
    np.cumsum(m_per, out=net_mptr[1:])
    M = int(net_mptr[-1])
    mem_pin = np.fromiter((p for s in net_sinks for p in s), dtype=np.int64, count=M)
    if cfg.net_topology == "star":
        mem_parent = np.repeat(np.arange(nc, dtype=np.int64), m_per)
        # per cell: 4 doubles per member (res rise, res fall factor, cap rise,
        # cap fall factor), then 2 for the root cap
        draws = 4 * m_per + 2
        u = rng_rc.random(int(draws.sum()))
        start = np.concatenate([[0], np.cumsum(draws)[:-1]])
        local = np.arange(M, dtype=np.int64) - np.repeat(net_mptr[:-1], m_per)
        mrow = np.repeat(start, m_per) + 4 * local
        res_r = _unif(100.0, 2000.0, u[mrow])
        res_f = res_r * _unif(0.95, 1.05, u[mrow + 1])
        cap_r = _unif(0.5e-15, 5e-15, u[mrow + 2])
        cap_f = cap_r * _unif(0.95, 1.05, u[mrow + 3])
        rrow = start + 4 * m_per
        rc_r = _unif(1e-15, 3e-15, u[rrow])
        rc_f = rc_r * _unif(0.95, 1.05, u[rrow + 1])
    else:
        mem_parent = np.empty(M, dtype=np.int64)
        res_r = np.empty(M); res_f = np.empty(M)
        cap_r = np.empty(M); cap_f = np.empty(M)
        rc_r = np.empty(nc); rc_f = np.empty(nc)
        integers, unif = rng_rc.integers, rng_rc.uniform
        for c in range(nc):
            s = int(net_mptr[c])
            sinks = net_sinks[c]
            m = len(sinks)
            if m <= 1:
                mem_parent[s:s + m] = c
            else:
                nodes = [c]
                for k in range(m):
                    mem_parent[s + k] = nodes[int(integers(0, len(nodes)))]
                    nodes.append(sinks[k])
            for k in range(m):
                r = unif(100.0, 2000.0)
                res_r[s + k] = r
                res_f[s + k] = r * unif(0.95, 1.05)
                cp = unif(0.5e-15, 5e-15)
                cap_r[s + k] = cp
                cap_f[s + k] = cp * unif(0.95, 1.05)
            rr = unif(1e-15, 3e-15)
            rc_r[c] = rr
            rc_f[c] = rr * unif(0.95, 1.05)
    mem_res = np.stack([res_r, res_f, res_r, res_f], axis=1)
    mem_cap = np.stack([cap_r, cap_f, cap_r, cap_f], axis=1)
    root_cap = np.stack([rc_r, rc_f, rc_r, rc_f], axis=1)

    ep_pin = np.asarray(ep_pins, dtype=np.int64)
    ep_required = np.tile(np.array([0.0, 0.0, clock_period, clock_period]), (len(ep_pin), 1))
    return RawDesign(
        n_pins=n_pins, clock_period=clock_period,
        net_root=np.arange(nc, dtype=np.int64), net_mptr=net_mptr,
        mem_pin=mem_pin, mem_parent_pin=mem_parent, mem_res=mem_res, mem_cap=mem_cap,
        root_cap=root_cap, arc_from=arc_from, arc_to=arc_to,
        arc_dlut=arc_dlut, arc_slut=arc_slut,
        lut_s_ptr=s_ptr, lut_l_ptr=l_ptr, lut_t_ptr=t_ptr,
        lut_s_flat=s_flat, lut_l_flat=l_flat, lut_t_flat=t_flat,
        pi_pin=pi_pin, pi_arrival=pi_arrival, pi_slew=pi_slew,
        ep_pin=ep_pin, ep_required=ep_required,
        meta={"generator": cfg.to_doc(), "layer_sizes": layer_sizes,
              "fanout_bumps": fanout_bumps},
    ).normalized()


def _pin_names(raw: RawDesign, n_cells: int) -> list:
    """The reference generator's pin names (generator.py:240-309): cell
    output ``c{cell}/o`` (pins 0..n_cells-1), the cell's k-th input
    ``c{cell}/i{k}`` (its k-th arc, in creation order), endpoint pins
    ``ep{j}`` in creation (= id) order."""
    names = [f"c{c}/o" for c in range(n_cells)] + [""] * (raw.n_pins - n_cells)
    to = np.asarray(raw.arc_to, dtype=np.int64)
    fr = np.asarray(raw.arc_from, dtype=np.int64)
    if len(to):
        first = np.concatenate([[0], np.flatnonzero(to[1:] != to[:-1]) + 1])
        k = np.arange(len(to)) - np.repeat(first, np.diff(np.concatenate([first, [len(to)]])))
        for p, c, kk in zip(fr.tolist(), to.tolist(), k.tolist()):
            names[p] = f"c{c}/i{kk}"
    j = 0
    for p in range(n_cells, raw.n_pins):
        if not names[p]:
            names[p] = f"ep{j}"
            j += 1
    return names


def generate_design(cfg: GeneratorConfig):
    """Object-model design (API convenience over :func:`generate_raw`), with
    the reference generator's pin names."""
    raw = generate_raw(cfg)
    d = raw_to_design(raw)
    d.pin_names = _pin_names(raw, cfg.num_cells)
    return d


# BASELINE.md §2 workloads
def config_c1(topology="star"):
    return GeneratorConfig(num_cells=2500, fanout=power_law(2.0, 64), depth_target=12,
                           seed=7, net_topology=topology)


def config_c2():
    return GeneratorConfig(num_cells=192500, fanout=power_law(2.0, 512), depth_target=40, seed=7)


def config_c3():
    return GeneratorConfig(num_cells=630000, fanout=power_law(2.0, 64), depth_target=60, seed=7)
