"""Netlist data model and the flat host-side ingest format.

Two representations of one design:

* ``Design`` and friends — the object model with the reference's field names
  (/root/reference/pkg/src/stasim/netlist.py:81-185).  Any object with these
  attributes (including the reference's own ``stasim.Design``) is accepted by
  :func:`design_to_raw`, so a user's existing designs drop in unchanged.
* ``RawDesign`` — plain numpy arrays, exactly what the C-ABI ``ws_create``
  (include/warpstar.h) uploads.  Topology is int32, values are float64.  The
  device derives every ``FlatDesign`` index array (levels, CSR, maps) from it
  (flatten.py:170-316 on the reference side).

Condition order is the reference's: 0 early-rise, 1 early-fall, 2 late-rise,
3 late-fall (netlist.py:41-45).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

N_COND = 4
EARLY_RISE, EARLY_FALL, LATE_RISE, LATE_FALL = range(N_COND)
COND_NAMES = ("early_rise", "early_fall", "late_rise", "late_fall")
EARLY_CONDS = (EARLY_RISE, EARLY_FALL)
LATE_CONDS = (LATE_RISE, LATE_FALL)


def corner(values) -> np.ndarray:
    """Scalar or length-4 sequence -> float64 corner vector (netlist.py:71-78)."""
    a = np.asarray(values, dtype=np.float64)
    if a.ndim == 0:
        a = np.full(N_COND, float(a))
    if a.shape != (N_COND,):
        raise ValueError(f"corner vector must have {N_COND} entries, got shape {a.shape}")
    return a


@dataclass(eq=False)
class Lut2D:
    """2-D table over (input slew, output load); 1x1 is a constant
    (netlist.py:81-113).  Identity (not content) is what flatten dedupes on."""

    slew_axis: np.ndarray
    load_axis: np.ndarray
    table: np.ndarray

    def __post_init__(self):
        self.slew_axis = np.asarray(self.slew_axis, dtype=np.float64)
        self.load_axis = np.asarray(self.load_axis, dtype=np.float64)
        self.table = np.asarray(self.table, dtype=np.float64)

    def check(self) -> list:
        """Problems of this table (empty when well formed): axes 1-D,
        non-empty, strictly increasing; table (nS, nL); finite entries."""
        from .design_io import lut_problems
        return lut_problems(self.slew_axis, self.load_axis, self.table)


@dataclass
class TimingArc:
    from_pin: int
    to_pin: int
    delay_luts: list
    slew_luts: list


@dataclass
class Cell:
    arcs: list


@dataclass
class Net:
    """Rooted RC tree; members in topological order (netlist.py:132-150)."""

    root: int
    member_pins: list
    member_parents: list
    member_res: np.ndarray
    member_caps: np.ndarray
    root_cap: np.ndarray

    def __post_init__(self):
        m = len(self.member_pins)
        self.member_res = np.asarray(self.member_res, dtype=np.float64).reshape(m, N_COND)
        self.member_caps = np.asarray(self.member_caps, dtype=np.float64).reshape(m, N_COND)
        self.root_cap = corner(self.root_cap)


@dataclass
class PrimaryInput:
    pin: int
    arrival: np.ndarray
    slew: np.ndarray

    def __post_init__(self):
        self.arrival = corner(self.arrival)
        self.slew = corner(self.slew)


@dataclass
class Endpoint:
    pin: int
    required: np.ndarray

    def __post_init__(self):
        self.required = corner(self.required)


@dataclass
class Design:
    pin_names: list
    cells: list
    nets: list
    primary_inputs: list
    endpoints: list
    clock_period: float
    meta: dict = field(default_factory=dict)

    @property
    def n_pins(self):
        return len(self.pin_names)


# ---------------------------------------------------------------------------
# flat ingest format

_I32 = np.int32


@dataclass
class RawDesign:
    """Flat arrays of one design, in the reference's own orders.

    nets: ``net_root[N]``, members concatenated net by net
    (``net_mptr[N+1]`` offsets, ``mem_pin``, ``mem_parent_pin`` = parent PIN id),
    ``mem_res``/``mem_cap`` (M,4), ``root_cap`` (N,4).
    arcs: cells in order, arcs in order (flatten.py:222): ``arc_from``,
    ``arc_to``, ``arc_dlut``/``arc_slut`` (A,4) ids into the LUT pool.
    LUT pool: deduplicated in first-appearance order exactly like
    flatten.py:211-244, packed as ``lut_{s,l,t}_ptr`` / ``lut_{s,l,t}_flat``.
    seeds: ``pi_pin``/``pi_arrival``/``pi_slew``, ``ep_pin``/``ep_required``.
    """

    n_pins: int
    clock_period: float
    net_root: np.ndarray
    net_mptr: np.ndarray
    mem_pin: np.ndarray
    mem_parent_pin: np.ndarray
    mem_res: np.ndarray
    mem_cap: np.ndarray
    root_cap: np.ndarray
    arc_from: np.ndarray
    arc_to: np.ndarray
    arc_dlut: np.ndarray
    arc_slut: np.ndarray
    lut_s_ptr: np.ndarray
    lut_l_ptr: np.ndarray
    lut_t_ptr: np.ndarray
    lut_s_flat: np.ndarray
    lut_l_flat: np.ndarray
    lut_t_flat: np.ndarray
    pi_pin: np.ndarray
    pi_arrival: np.ndarray
    pi_slew: np.ndarray
    ep_pin: np.ndarray
    ep_required: np.ndarray
    meta: dict = field(default_factory=dict)

    @property
    def n_nets(self):
        return int(len(self.net_root))

    @property
    def n_members(self):
        return int(len(self.mem_pin))

    @property
    def n_arcs(self):
        return int(len(self.arc_from))

    @property
    def n_luts(self):
        return int(len(self.lut_s_ptr) - 1)

    def normalized(self) -> "RawDesign":
        """Contiguous arrays with the dtypes the C-ABI expects."""
        def i32(a, shape=None):
            a = np.asarray(a)
            if a.dtype != _I32 and a.size:
                if not np.issubdtype(a.dtype, np.integer):
                    if not np.array_equal(a, np.trunc(a)):
                        raise ValueError("index arrays must hold integers")
                lo, hi = a.min(), a.max()
                if lo < np.iinfo(_I32).min or hi > np.iinfo(_I32).max:
                    raise ValueError(f"index {hi if hi > 0 else lo} does not fit the device's "
                                     f"int32 indices (ADVICE r1: no silent wrap-around)")
            a = np.ascontiguousarray(a, dtype=_I32)
            return a.reshape(shape) if shape is not None else a

        def f64(a, shape=None):
            a = np.ascontiguousarray(a, dtype=np.float64)
            return a.reshape(shape) if shape is not None else a

        n, m, a_ = len(self.net_root), len(self.mem_pin), len(self.arc_from)
        return RawDesign(
            n_pins=int(self.n_pins), clock_period=float(self.clock_period),
            net_root=i32(self.net_root), net_mptr=np.ascontiguousarray(self.net_mptr, dtype=np.int64),
            mem_pin=i32(self.mem_pin), mem_parent_pin=i32(self.mem_parent_pin),
            mem_res=f64(self.mem_res, (m, N_COND)), mem_cap=f64(self.mem_cap, (m, N_COND)),
            root_cap=f64(self.root_cap, (n, N_COND)),
            arc_from=i32(self.arc_from), arc_to=i32(self.arc_to),
            arc_dlut=i32(self.arc_dlut, (a_, N_COND)), arc_slut=i32(self.arc_slut, (a_, N_COND)),
            lut_s_ptr=i32(self.lut_s_ptr), lut_l_ptr=i32(self.lut_l_ptr), lut_t_ptr=i32(self.lut_t_ptr),
            lut_s_flat=f64(self.lut_s_flat), lut_l_flat=f64(self.lut_l_flat),
            lut_t_flat=f64(self.lut_t_flat),
            pi_pin=i32(self.pi_pin), pi_arrival=f64(self.pi_arrival, (len(self.pi_pin), N_COND)),
            pi_slew=f64(self.pi_slew, (len(self.pi_pin), N_COND)),
            ep_pin=i32(self.ep_pin), ep_required=f64(self.ep_required, (len(self.ep_pin), N_COND)),
            meta=dict(self.meta),
        )


def pack_luts(luts) -> tuple:
    """Pack a list of Lut2D-like objects into the reference's flat LUT pool
    (flatten.py:235-244)."""
    n = len(luts)
    s_ptr = np.zeros(n + 1, dtype=np.int64)
    l_ptr = np.zeros(n + 1, dtype=np.int64)
    t_ptr = np.zeros(n + 1, dtype=np.int64)
    for i, lut in enumerate(luts):
        s_ptr[i + 1] = s_ptr[i] + np.asarray(lut.slew_axis).size
        l_ptr[i + 1] = l_ptr[i] + np.asarray(lut.load_axis).size
        t_ptr[i + 1] = t_ptr[i] + np.asarray(lut.table).size
    s_flat = (np.concatenate([np.asarray(l.slew_axis, dtype=np.float64).ravel() for l in luts])
              if n else np.zeros(0))
    l_flat = (np.concatenate([np.asarray(l.load_axis, dtype=np.float64).ravel() for l in luts])
              if n else np.zeros(0))
    t_flat = (np.concatenate([np.asarray(l.table, dtype=np.float64).ravel() for l in luts])
              if n else np.zeros(0))
    return s_ptr, l_ptr, t_ptr, s_flat, l_flat, t_flat


def design_to_raw(design) -> RawDesign:
    """Object model -> flat arrays.  Host-side packing only (no timing math):
    member/parent lists are concatenated and LUTs are deduplicated by object
    identity in first-appearance order, cond by cond, delay before slew, as
    flatten.py:211-233 does."""
    nets = design.nets
    n_nets = len(nets)
    counts = np.fromiter((len(n.member_pins) for n in nets), dtype=np.int64, count=n_nets)
    net_mptr = np.zeros(n_nets + 1, dtype=np.int64)
    np.cumsum(counts, out=net_mptr[1:])
    m = int(net_mptr[-1])
    net_root = np.fromiter((n.root for n in nets), dtype=np.int64, count=n_nets)
    mem_pin = np.fromiter((p for n in nets for p in n.member_pins), dtype=np.int64, count=m)
    mem_parent = np.fromiter((p for n in nets for p in n.member_parents), dtype=np.int64, count=m)
    if m:
        mem_res = np.concatenate([np.asarray(n.member_res, dtype=np.float64).reshape(-1, N_COND)
                                  for n in nets])
        mem_cap = np.concatenate([np.asarray(n.member_caps, dtype=np.float64).reshape(-1, N_COND)
                                  for n in nets])
    else:
        mem_res = np.zeros((0, N_COND))
        mem_cap = np.zeros((0, N_COND))
    root_cap = (np.stack([corner(n.root_cap) for n in nets]) if n_nets
                else np.zeros((0, N_COND)))

    lut_ids = {}
    luts = []
    arcs = [arc for cell in design.cells for arc in cell.arcs]
    n_arcs = len(arcs)
    arc_from = np.fromiter((a.from_pin for a in arcs), dtype=np.int64, count=n_arcs)
    arc_to = np.fromiter((a.to_pin for a in arcs), dtype=np.int64, count=n_arcs)
    arc_dlut = np.zeros((n_arcs, N_COND), dtype=np.int64)
    arc_slut = np.zeros((n_arcs, N_COND), dtype=np.int64)
    for ai, arc in enumerate(arcs):
        for c in range(N_COND):
            for lst, out in ((arc.delay_luts, arc_dlut), (arc.slew_luts, arc_slut)):
                lut = lst[c]
                got = lut_ids.get(id(lut))
                if got is None:
                    got = lut_ids[id(lut)] = len(luts)
                    luts.append(lut)
                out[ai, c] = got
    s_ptr, l_ptr, t_ptr, s_flat, l_flat, t_flat = pack_luts(luts)

    pis = design.primary_inputs
    eps = design.endpoints
    pi_pin = np.fromiter((p.pin for p in pis), dtype=np.int64, count=len(pis))
    pi_arrival = np.stack([corner(p.arrival) for p in pis]) if pis else np.zeros((0, N_COND))
    pi_slew = np.stack([corner(p.slew) for p in pis]) if pis else np.zeros((0, N_COND))
    ep_pin = np.fromiter((e.pin for e in eps), dtype=np.int64, count=len(eps))
    ep_required = np.stack([corner(e.required) for e in eps]) if eps else np.zeros((0, N_COND))
    return RawDesign(
        n_pins=int(design.n_pins), clock_period=float(design.clock_period),
        net_root=net_root, net_mptr=net_mptr, mem_pin=mem_pin, mem_parent_pin=mem_parent,
        mem_res=mem_res, mem_cap=mem_cap, root_cap=root_cap,
        arc_from=arc_from, arc_to=arc_to, arc_dlut=arc_dlut, arc_slut=arc_slut,
        lut_s_ptr=s_ptr, lut_l_ptr=l_ptr, lut_t_ptr=t_ptr,
        lut_s_flat=s_flat, lut_l_flat=l_flat, lut_t_flat=t_flat,
        pi_pin=pi_pin, pi_arrival=pi_arrival, pi_slew=pi_slew,
        ep_pin=ep_pin, ep_required=ep_required,
        meta=dict(getattr(design, "meta", {}) or {}),
    ).normalized()


def raw_to_design(raw: RawDesign) -> Design:
    """Flat arrays -> object model (API convenience; slow at 10^6 pins)."""
    luts = []
    for i in range(raw.n_luts):
        s = raw.lut_s_flat[raw.lut_s_ptr[i]:raw.lut_s_ptr[i + 1]]
        l = raw.lut_l_flat[raw.lut_l_ptr[i]:raw.lut_l_ptr[i + 1]]
        t = raw.lut_t_flat[raw.lut_t_ptr[i]:raw.lut_t_ptr[i + 1]].reshape(len(s), len(l))
        luts.append(Lut2D(s.copy(), l.copy(), t.copy()))
    # one cell per run of arcs driving the same pin (the reference groups a
    # cell's arcs by output pin; any grouping gives the same flat arc order)
    cells = []
    cur, cur_to = [], None
    for a in range(raw.n_arcs):
        to = int(raw.arc_to[a])
        if cur and to != cur_to:
            cells.append(Cell(cur))
            cur = []
        cur_to = to
        cur.append(TimingArc(int(raw.arc_from[a]), to,
                             [luts[i] for i in raw.arc_dlut[a]],
                             [luts[i] for i in raw.arc_slut[a]]))
    if cur:
        cells.append(Cell(cur))
    nets = []
    for n in range(raw.n_nets):
        s, e = int(raw.net_mptr[n]), int(raw.net_mptr[n + 1])
        nets.append(Net(int(raw.net_root[n]), raw.mem_pin[s:e].tolist(),
                        raw.mem_parent_pin[s:e].tolist(), raw.mem_res[s:e].copy(),
                        raw.mem_cap[s:e].copy(), raw.root_cap[n].copy()))
    pis = [PrimaryInput(int(p), raw.pi_arrival[i], raw.pi_slew[i])
           for i, p in enumerate(raw.pi_pin)]
    eps = [Endpoint(int(p), raw.ep_required[i]) for i, p in enumerate(raw.ep_pin)]
    names = [f"p{i}" for i in range(raw.n_pins)]
    return Design(names, cells, nets, pis, eps, float(raw.clock_period), dict(raw.meta))

