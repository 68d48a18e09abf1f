"""Design validation and the JSON document format (host side, not on the
timed path).

Drop-in for the reference's model checks and interchange
(/root/reference/pkg/src/stasim/netlist.py:48-59 error types, 191-313
``validate``, 385-559 ``serialize_design`` / ``parse_design``):

* ``validate(design)`` returns the list of ``Violation``s of an object-model
  ``Design`` (or of a ``RawDesign``): dangling references, multiple drivers,
  self-loop arcs, malformed LUTs, non-topological RC trees, bad values,
  undriven roots / arc sources, dangling sinks, the clock period and
  combinational cycles.  The checks run vectorized over the flat arrays, so
  they stay fast on 10^6-pin designs;
* ``serialize_design`` / ``parse_design`` read and write the reference's
  document (same keys, same order, LUTs pooled by content, ``indent=1``), so
  documents written by either package load in the other and re-serialise
  byte for byte;
* ``engine_violations(raw)`` is the subset the device build relies on (tree
  order, one driver per pin, increasing LUT axes): ``flatten`` /
  ``DeviceDesign`` raise ``DesignSemanticsError`` for those before anything
  reaches the kernels.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .netlist import (N_COND, Cell, Design, Endpoint, Lut2D, Net, PrimaryInput, RawDesign,
                      TimingArc, corner, design_to_raw)


@dataclass
class Violation:
    kind: str
    message: str

    def __str__(self):
        return f"[{self.kind}] {self.message}"


class DesignFormatError(ValueError):
    """A design document that is not syntactically well formed."""


class DesignSemanticsError(ValueError):
    """A well-formed design that violates a model invariant; carries the list."""

    def __init__(self, violations):
        self.violations = list(violations)
        shown = "; ".join(str(v) for v in self.violations[:8])
        extra = len(self.violations) - 8
        super().__init__(f"invalid design: {shown}" + (f" (+{extra} more)" if extra > 0 else ""))


# ---------------------------------------------------------------------------
# LUT checks

def lut_problems(slew_axis, load_axis, table) -> list:
    """Problems of one table: 1-D non-empty axes, table shape (nS, nL),
    strictly increasing axes, finite entries (Lut2D.check in the reference)."""
    s, l, t = (np.asarray(x, dtype=np.float64) for x in (slew_axis, load_axis, table))
    if s.ndim != 1 or l.ndim != 1:
        return ["lut axes must be 1-D"]
    out = []
    if not s.size or not l.size:
        out.append("lut axes must be non-empty")
    if t.shape != (s.size, l.size):
        out.append(f"lut table shape {t.shape} does not match axes ({s.size}, {l.size})")
    for name, ax in (("slew", s), ("load", l)):
        if ax.size > 1 and not bool(np.all(ax[1:] > ax[:-1])):
            out.append(f"lut {name} axis is not strictly increasing")
    for name, a in (("slew_axis", s), ("load_axis", l), ("table", t)):
        if a.size and not bool(np.isfinite(a).all()):
            out.append(f"lut {name} has non-finite entries")
    return out


def _pool_axis_problems(raw: RawDesign, tables: bool = True) -> np.ndarray:
    """Per pooled LUT: True where an axis is not strictly increasing or an
    entry (of an axis, or of the table with ``tables``) is non-finite
    (vectorized over the packed pool)."""
    bad = np.zeros(raw.n_luts, dtype=bool)
    for ptr, flat in ((raw.lut_s_ptr, raw.lut_s_flat), (raw.lut_l_ptr, raw.lut_l_flat)):
        ptr = np.asarray(ptr, dtype=np.int64)
        flat = np.asarray(flat, dtype=np.float64)
        if flat.size > 1:
            # a step inside one LUT's axis that does not increase
            step_bad = ~(flat[1:] > flat[:-1])
            owner = np.searchsorted(ptr, np.arange(1, flat.size), side="right") - 1
            same = owner == (np.searchsorted(ptr, np.arange(flat.size - 1), side="right") - 1)
            np.logical_or.at(bad, owner[step_bad & same], True)
        if flat.size:
            nf = ~np.isfinite(flat)
            if nf.any():
                np.logical_or.at(bad, np.searchsorted(ptr, np.flatnonzero(nf), side="right") - 1, True)
    t_ptr = np.asarray(raw.lut_t_ptr, dtype=np.int64)
    t = np.asarray(raw.lut_t_flat, dtype=np.float64)
    if tables and t.size and not np.isfinite(t).all():
        np.logical_or.at(bad, np.searchsorted(t_ptr, np.flatnonzero(~np.isfinite(t)), side="right") - 1, True)
    return bad


# ---------------------------------------------------------------------------
# array-level checks

def _member_local(raw: RawDesign):
    mptr = np.asarray(raw.net_mptr, dtype=np.int64)
    counts = np.diff(mptr)
    mem_net = np.repeat(np.arange(len(counts), dtype=np.int64), counts)
    local = np.arange(len(raw.mem_pin), dtype=np.int64) - mptr[mem_net] if len(mem_net) else mem_net
    return mem_net, local


def _tree_order_bad(raw: RawDesign, mem_net, local) -> np.ndarray:
    """Members whose parent is neither their net's root nor an EARLIER member
    of the same net (or that list their own root as a member)."""
    P = raw.n_pins
    mem_pin = np.asarray(raw.mem_pin, dtype=np.int64)
    parent = np.asarray(raw.mem_parent_pin, dtype=np.int64)
    root = np.asarray(raw.net_root, dtype=np.int64)
    if not len(mem_pin):
        return np.zeros(0, dtype=bool)
    # (net, local index) of every member pin, first occurrence
    net_of = np.full(P, -1, dtype=np.int64)
    loc_of = np.full(P, -1, dtype=np.int64)
    order = np.arange(len(mem_pin))[::-1]            # first occurrence wins
    net_of[mem_pin[order]] = mem_net[order]
    loc_of[mem_pin[order]] = local[order]
    ok_root = parent == root[mem_net]
    ok_mem = (net_of[parent] == mem_net) & (loc_of[parent] < local) & (loc_of[parent] >= 0)
    self_root = mem_pin == root[mem_net]
    return ~(ok_root | ok_mem) | self_root


def engine_violations(raw: RawDesign) -> list:
    """The invariants the device build relies on: RC trees in topological
    order, one driver per pin (a pin is a member of at most one net, roots at
    most one net, is targeted by arcs of one cell run), LUT axes strictly
    increasing.  Index ranges are checked by ws_create itself."""
    v = []
    P = raw.n_pins
    mem_pin = np.asarray(raw.mem_pin, dtype=np.int64)
    root = np.asarray(raw.net_root, dtype=np.int64)
    for name, pins in (("member", mem_pin), ("root", root)):
        if len(pins) and (pins.min() < 0 or pins.max() >= P):
            return [Violation("dangling-ref", f"a net {name} references a pin outside 0..{P - 1}")]
    mem_net, local = _member_local(raw)
    bad = np.flatnonzero(_tree_order_bad(raw, mem_net, local))
    for k in bad[:16]:
        v.append(Violation("non-tree-net",
                           f"net {int(mem_net[k])} not in topological order: member pin {int(mem_pin[k])} "
                           f"has parent {int(raw.mem_parent_pin[k])} which is not the root or an earlier "
                           f"member"))
    for name, pins in (("a member of two nets", mem_pin), ("the root of two nets", root)):
        if len(pins):
            cnt = np.bincount(pins, minlength=P)
            for p in np.flatnonzero(cnt > 1)[:16]:
                v.append(Violation("multi-driver", f"pin {int(p)} is {name}"))
    if raw.n_luts:
        # the device's axis search assumes sorted, finite axes (table
        # entries go through the same arithmetic as the reference's)
        for i in np.flatnonzero(_pool_axis_problems(raw, tables=False))[:16]:
            v.append(Violation("bad-lut", f"lut {int(i)}: axis not strictly increasing or "
                                          f"non-finite"))
    return v


def _ranges(starts, lens) -> np.ndarray:
    """concatenate(arange(s, s + n) for s, n in zip(starts, lens)), vectorized."""
    lens = np.asarray(lens, dtype=np.int64)
    tot = int(lens.sum())
    if not tot:
        return np.zeros(0, dtype=np.int64)
    keep = lens > 0
    st, ln = np.asarray(starts, dtype=np.int64)[keep], lens[keep]
    step = np.ones(tot, dtype=np.int64)
    heads = np.concatenate([[0], np.cumsum(ln)[:-1]])
    step[heads] = st - np.concatenate([[0], st[:-1] + ln[:-1] - 1])
    return np.cumsum(step)


def _find_cycle_root(raw: RawDesign, member_net_of_pin, arc_ok) -> int | None:
    """A pin on a combinational cycle of the net graph, or None: Kahn over the
    net dependencies (vectorized rounds), then a walk through stuck
    predecessors until a net repeats."""
    N = raw.n_nets
    if not N:
        return None
    root = np.asarray(raw.net_root, dtype=np.int64)
    root_net = np.full(raw.n_pins, -1, dtype=np.int64)
    root_net[root] = np.arange(N)
    af = np.asarray(raw.arc_from, dtype=np.int64)[arc_ok]
    at = np.asarray(raw.arc_to, dtype=np.int64)[arc_ok]
    src = member_net_of_pin[af]
    dst = root_net[at]
    keep = (src >= 0) & (dst >= 0)
    es, ed = src[keep], dst[keep]
    feed = member_net_of_pin[root]                      # feedthrough: root is a member
    fk = feed >= 0
    es = np.concatenate([es, feed[fk]])
    ed = np.concatenate([ed, np.flatnonzero(fk)])
    if len(es):
        pairs = np.unique(es * N + ed)
        es, ed = pairs // N, pairs % N
    indeg = np.bincount(ed, minlength=N)
    order = np.argsort(es, kind="stable")
    es_s, ed_s = es[order], ed[order]
    ptr = np.searchsorted(es_s, np.arange(N + 1))
    done = np.zeros(N, dtype=bool)
    frontier = np.flatnonzero(indeg == 0)
    while len(frontier):
        done[frontier] = True
        idx = _ranges(ptr[frontier], ptr[frontier + 1] - ptr[frontier])
        if len(idx):
            np.subtract.at(indeg, ed_s[idx], 1)
            cand = np.unique(ed_s[idx])
            frontier = cand[(indeg[cand] == 0) & ~done[cand]]
        else:
            frontier = np.zeros(0, dtype=np.int64)
    stuck = np.flatnonzero(~done)
    if not len(stuck):
        return None
    # predecessors among stuck nets; walk back until a net repeats
    by_dst = np.argsort(ed, kind="stable")
    ed_d, es_d = ed[by_dst], es[by_dst]
    dptr = np.searchsorted(ed_d, np.arange(N + 1))
    seen = {}
    n = int(stuck[0])
    while n not in seen:
        seen[n] = len(seen)
        preds = es_d[dptr[n]:dptr[n + 1]]
        preds = preds[~done[preds]]
        n = int(preds.min())
    return int(root[n])


def validate_raw(raw: RawDesign, cell_of_arc=None) -> list:
    """validate() over flat arrays.  ``cell_of_arc`` (the cell index of every
    arc) enables the one-cell-per-target check, which the flat arrays alone
    cannot express."""
    v = []
    P = raw.n_pins
    as_i = lambda a: np.asarray(a, dtype=np.int64)
    mem_pin, parent, root = as_i(raw.mem_pin), as_i(raw.mem_parent_pin), as_i(raw.net_root)
    af, at = as_i(raw.arc_from), as_i(raw.arc_to)
    pi_pin, ep_pin = as_i(raw.pi_pin), as_i(raw.ep_pin)
    inr = lambda a: (a >= 0) & (a < P)

    def dangling(arr, what):
        for i in np.flatnonzero(~inr(arr))[:16]:
            v.append(Violation("dangling-ref", f"{what} {int(i)} references pin {int(arr[i])} "
                                               f"outside 0..{P - 1}"))
    dangling(pi_pin, "primary input")
    dangling(ep_pin, "endpoint")
    dangling(af, "arc (from)")
    dangling(at, "arc (to)")
    dangling(root, "net root")
    dangling(mem_pin, "net member")
    dangling(parent, "net member parent")
    structural = any(x.kind == "dangling-ref" for x in v)

    pia = np.asarray(raw.pi_arrival, dtype=np.float64).reshape(-1, N_COND)
    pis = np.asarray(raw.pi_slew, dtype=np.float64).reshape(-1, N_COND)
    for i in np.flatnonzero(~(np.isfinite(pia).all(1) & np.isfinite(pis).all(1)))[:16]:
        v.append(Violation("bad-value", f"primary input {int(pi_pin[i])} has non-finite arrival/slew"))
    epr = np.asarray(raw.ep_required, dtype=np.float64).reshape(-1, N_COND)
    for i in np.flatnonzero(~np.isfinite(epr).all(1))[:16]:
        v.append(Violation("bad-value", f"endpoint pin {int(ep_pin[i])} has non-finite required time"))
    for i in np.flatnonzero(af == at)[:16]:
        v.append(Violation("bad-arc", f"arc {int(i)} is a self loop on pin {int(af[i])}"))
    if structural:
        return v

    # drivers: primary inputs, arc targets (one cell each), net members
    pc = np.bincount(pi_pin, minlength=P)
    for p in np.flatnonzero(pc > 1)[:16]:
        v.append(Violation("multi-driver", f"pin {int(p)} listed as primary input twice"))
    is_pi = pc > 0
    tgt = np.zeros(P, dtype=bool)
    tgt[at] = True
    if cell_of_arc is not None and len(at):
        cells = np.asarray(cell_of_arc, dtype=np.int64)
        pairs = np.unique(at * (int(cells.max()) + 1) + cells)
        per_pin = np.bincount(pairs // (int(cells.max()) + 1), minlength=P)
        for p in np.flatnonzero(per_pin > 1)[:16]:
            v.append(Violation("multi-driver", f"pin {int(p)} is an arc target of more than one cell"))
    for p in np.flatnonzero(is_pi & tgt)[:16]:
        v.append(Violation("multi-driver", f"pin {int(p)} driven by both a primary input and a cell"))
    rc = np.bincount(root, minlength=P)
    for p in np.flatnonzero(rc > 1)[:16]:
        v.append(Violation("multi-driver", f"pin {int(p)} roots more than one net"))
    mc = np.bincount(mem_pin, minlength=P)
    for p in np.flatnonzero(mc > 1)[:16]:
        v.append(Violation("multi-driver", f"pin {int(p)} is a member of more than one net"))
    is_mem = mc > 0
    for p in np.flatnonzero(is_mem & (is_pi | tgt))[:16]:
        v.append(Violation("multi-driver", f"pin {int(p)} driven by both its net and a "
                                           f"{'primary input' if is_pi[p] else 'cell'}"))
    mem_net, local = _member_local(raw)
    tree_bad = _tree_order_bad(raw, mem_net, local)
    for k in np.flatnonzero(tree_bad)[:16]:
        if mem_pin[k] == root[mem_net[k]]:
            msg = f"net {int(mem_net[k])}: root pin {int(mem_pin[k])} listed as a member"
        else:
            msg = (f"net {int(mem_net[k])} not in topological order: member pin {int(mem_pin[k])} has "
                   f"parent {int(parent[k])} which is not the root or an earlier member")
        v.append(Violation("non-tree-net", msg))
    # RC values per net: finite, then non-negative
    mres = np.asarray(raw.mem_res, dtype=np.float64).reshape(-1, N_COND)
    mcap = np.asarray(raw.mem_cap, dtype=np.float64).reshape(-1, N_COND)
    rcap = np.asarray(raw.root_cap, dtype=np.float64).reshape(-1, N_COND)
    N = raw.n_nets
    nonfin = ~np.isfinite(rcap).all(1)
    neg = (rcap < 0).any(1)
    if len(mem_pin):
        np.logical_or.at(nonfin, mem_net, ~(np.isfinite(mres).all(1) & np.isfinite(mcap).all(1)))
        np.logical_or.at(neg, mem_net, (mres < 0).any(1) | (mcap < 0).any(1))
    for n in np.flatnonzero(nonfin)[:16]:
        v.append(Violation("bad-value", f"net {int(n)} has non-finite res/cap entries"))
    for n in np.flatnonzero(neg & ~nonfin)[:16]:
        v.append(Violation("bad-value", f"net {int(n)} has negative res/cap entries"))
    # LUT pool
    if raw.n_luts:
        used = np.zeros(raw.n_luts, dtype=bool)
        used[np.asarray(raw.arc_dlut, dtype=np.int64).ravel()] = True
        used[np.asarray(raw.arc_slut, dtype=np.int64).ravel()] = True
        for i in np.flatnonzero(_pool_axis_problems(raw) & used)[:16]:
            v.append(Violation("bad-lut", f"lut {int(i)}: axis not strictly increasing or non-finite "
                                          f"entries"))
    # every root driven; every arc source carries a value; every sink consumed
    for n in np.flatnonzero(~(tgt[root] | is_pi[root] | is_mem[root]))[:16]:
        v.append(Violation("undriven-root", f"net {int(n)} root pin {int(root[n])} has no arc, net, or "
                                            f"primary input driving it"))
    src = np.zeros(P, dtype=bool)
    src[af] = True
    for p in np.flatnonzero(src & ~is_mem & ~is_pi)[:16]:
        v.append(Violation("undriven-pin", f"arc source pin {int(p)} is neither a net member nor a "
                                           f"primary input"))
    is_root = rc > 0
    is_ep = np.zeros(P, dtype=bool)
    is_ep[ep_pin] = True
    for p in np.flatnonzero(is_mem & ~src & ~is_root & ~is_ep)[:16]:
        v.append(Violation("dangling-pin", f"net member pin {int(p)} feeds no arc and is not an endpoint"))
    cp = raw.clock_period
    if not (isinstance(cp, (int, float, np.floating)) and np.isfinite(cp) and cp > 0):
        v.append(Violation("bad-value", f"clock_period must be a positive finite number, got {cp!r}"))
    if not any(x.kind == "non-tree-net" for x in v):
        net_of_pin = np.full(P, -1, dtype=np.int64)
        net_of_pin[mem_pin[::-1]] = mem_net[::-1]
        pin = _find_cycle_root(raw, net_of_pin, np.ones(len(af), dtype=bool))
        if pin is not None:
            v.append(Violation("cyclic", f"combinational cycle through pin {pin}"))
    return v


def validate(design) -> list:
    """Model violations of a design (an object-model ``Design``, the
    reference's own ``stasim.Design``, or a ``RawDesign``); empty when valid
    (netlist.py:191-313)."""
    if isinstance(design, RawDesign):
        return validate_raw(design)
    v = []
    n = design.n_pins

    def ref_ok(p):
        return isinstance(p, (int, np.integer)) and 0 <= p < n

    # object-model structure the flat arrays cannot hold: reference types,
    # four tables per condition list, each table well formed
    checked = {}
    for ci, cell in enumerate(design.cells):
        for ai, arc in enumerate(cell.arcs):
            where = f"cell {ci} arc {ai}"
            for p in (arc.from_pin, arc.to_pin):
                if not ref_ok(p):
                    v.append(Violation("dangling-ref", f"{where} references pin {p!r} outside 0..{n - 1}"))
            for kind, luts in (("delay", arc.delay_luts), ("slew", arc.slew_luts)):
                if len(luts) != N_COND:
                    v.append(Violation("bad-lut", f"{where} needs {N_COND} {kind} luts"))
                    continue
                for lut in luts:
                    probs = checked.get(id(lut))
                    if probs is None:
                        probs = checked[id(lut)] = lut_problems(lut.slew_axis, lut.load_axis, lut.table)
                    v.extend(Violation("bad-lut", f"{where}: {p}") for p in probs)
    for ni, net in enumerate(design.nets):
        refs = [net.root] + list(net.member_pins) + list(net.member_parents)
        for p in refs:
            if not ref_ok(p):
                v.append(Violation("dangling-ref", f"net {ni} references pin {p!r} outside 0..{n - 1}"))
    for what, items in (("primary input", design.primary_inputs), ("endpoint", design.endpoints)):
        for it in items:
            if not ref_ok(it.pin):
                v.append(Violation("dangling-ref", f"{what} references pin {it.pin!r} outside 0..{n - 1}"))
    if any(x.kind in ("dangling-ref",) for x in v) or any("needs" in x.message for x in v):
        return v
    raw = design_to_raw(design)
    cell_of_arc = np.repeat(np.arange(len(design.cells)), [len(c.arcs) for c in design.cells])
    rest = validate_raw(raw, cell_of_arc=cell_of_arc)
    # the per-table problems were reported per arc above
    return v + [x for x in rest if x.kind != "bad-lut"]


def check_engine_invariants(raw: RawDesign) -> None:
    vs = engine_violations(raw)
    if vs:
        raise DesignSemanticsError(vs)


# ---------------------------------------------------------------------------
# JSON document (the reference's interchange format)

def _floats(a):
    return [float(x) for x in np.asarray(a, dtype=np.float64).ravel()]


def _lut_doc(lut) -> dict:
    t = np.asarray(lut.table, dtype=np.float64)
    return {"slew_axis": _floats(lut.slew_axis), "load_axis": _floats(lut.load_axis),
            "table": [_floats(row) for row in t]}


def serialize_design(design) -> str:
    """The canonical JSON document of a design: top-level clock_period, pins,
    luts (tables pooled by content, first use first), cells, nets; two
    structurally equal designs give byte-identical text."""
    pool_index = {}
    pool = []

    def ref(lut):
        doc = _lut_doc(lut)
        key = json.dumps(doc)
        got = pool_index.get(key)
        if got is None:
            got = pool_index[key] = len(pool)
            pool.append(doc)
        return got

    cells = [{"arcs": [{"from": int(a.from_pin), "to": int(a.to_pin),
                        "delay_lut": [ref(x) for x in a.delay_luts],
                        "slew_lut": [ref(x) for x in a.slew_luts]} for a in cell.arcs]}
             for cell in design.cells]
    req = {int(e.pin): e for e in design.endpoints}
    seed = {int(p.pin): p for p in design.primary_inputs}
    pins = []
    for i, name in enumerate(design.pin_names):
        d = {"name": name, "is_endpoint": i in req}
        if i in req:
            d["required"] = _floats(req[i].required)
        if i in seed:
            d["arrival"] = _floats(seed[i].arrival)
            d["slew"] = _floats(seed[i].slew)
        pins.append(d)
    nets = []
    for net in design.nets:
        res = np.asarray(net.member_res, dtype=np.float64).reshape(-1, N_COND)
        cap = np.asarray(net.member_caps, dtype=np.float64).reshape(-1, N_COND)
        nets.append({"root": int(net.root), "root_cap": _floats(net.root_cap),
                     "members": [{"pin": int(p), "parent": int(q), "res": _floats(res[k]),
                                  "cap": _floats(cap[k])}
                                 for k, (p, q) in enumerate(zip(net.member_pins, net.member_parents))]})
    return json.dumps({"clock_period": float(design.clock_period), "pins": pins, "luts": pool,
                       "cells": cells, "nets": nets}, indent=1)


def _lut_from(obj, pool):
    if isinstance(obj, bool) or not isinstance(obj, (int, dict)):
        raise DesignFormatError(f"lut reference must be an index or an object, got {type(obj).__name__}")
    if isinstance(obj, int):
        if not 0 <= obj < len(pool):
            raise DesignFormatError(f"lut index {obj} outside shared pool of {len(pool)}")
        return pool[obj]
    try:
        return Lut2D(obj["slew_axis"], obj["load_axis"], obj["table"])
    except (KeyError, TypeError, ValueError) as e:
        raise DesignFormatError(f"malformed lut object: {e}") from e


def _four(obj, pool, what):
    if not isinstance(obj, list) or len(obj) != N_COND:
        raise DesignFormatError(f"{what} must be a list of {N_COND} lut references")
    return [_lut_from(x, pool) for x in obj]


def parse_design(text: str) -> Design:
    """Read and validate a design document; DesignFormatError for syntax /
    shape problems, DesignSemanticsError listing every model violation."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise DesignFormatError(f"JSON syntax error at line {e.lineno} column {e.colno}: {e.msg}") from e
    if not isinstance(doc, dict):
        raise DesignFormatError("top level of a design document must be an object")
    missing = [k for k in ("clock_period", "pins", "cells", "nets") if k not in doc]
    if missing:
        raise DesignFormatError(f"missing required top-level key {missing[0]!r}")
    pool = []
    for i, obj in enumerate(doc.get("luts", [])):
        if isinstance(obj, int):
            raise DesignFormatError(f"shared lut {i} may not itself be an index")
        pool.append(_lut_from(obj, pool))
    if not isinstance(doc["pins"], list):
        raise DesignFormatError('"pins" must be a list')
    names, pis, eps = [], [], []
    try:
        for i, p in enumerate(doc["pins"]):
            names.append(str(p["name"]))
            if p.get("is_endpoint", False):
                eps.append(Endpoint(i, corner(p["required"])))
            if "arrival" in p:
                pis.append(PrimaryInput(i, corner(p["arrival"]), corner(p.get("slew", 0.0))))
    except (KeyError, TypeError, ValueError) as e:
        raise DesignFormatError(f"malformed pin entry: {e}") from e
    try:
        cells = [Cell([TimingArc(int(a["from"]), int(a["to"]), _four(a["delay_lut"], pool, "delay_lut"),
                                 _four(a["slew_lut"], pool, "slew_lut")) for a in c["arcs"]])
                 for c in doc["cells"]]
    except (KeyError, TypeError, ValueError) as e:
        raise DesignFormatError(f"malformed cell entry: {e}") from e
    try:
        nets = []
        for nd in doc["nets"]:
            ms = nd["members"]
            m = len(ms)
            nets.append(Net(int(nd["root"]), [int(x["pin"]) for x in ms], [int(x["parent"]) for x in ms],
                            np.asarray([x["res"] for x in ms], dtype=np.float64).reshape(m, N_COND),
                            np.asarray([x["cap"] for x in ms], dtype=np.float64).reshape(m, N_COND),
                            corner(nd.get("root_cap", 0.0))))
    except (KeyError, TypeError, ValueError) as e:
        raise DesignFormatError(f"malformed net entry: {e}") from e
    try:
        cp = float(doc["clock_period"])
    except (TypeError, ValueError) as e:
        raise DesignFormatError(f"clock_period must be a number: {e}") from e
    design = Design(names, cells, nets, pis, eps, cp)
    bad = validate(design)
    if bad:
        raise DesignSemanticsError(bad)
    return design


def design_equal(a, b) -> bool:
    """Structural equality of two designs (values compared exactly)."""
    if list(a.pin_names) != list(b.pin_names) or float(a.clock_period) != float(b.clock_period):
        return False
    ra, rb = design_to_raw(a), design_to_raw(b)
    for f in ("net_root", "net_mptr", "mem_pin", "mem_parent_pin", "mem_res", "mem_cap", "root_cap",
              "arc_from", "arc_to", "pi_pin", "pi_arrival", "pi_slew", "ep_pin", "ep_required"):
        if not np.array_equal(getattr(ra, f), getattr(rb, f)):
            return False
    # tables by value (pools may differ in sharing)
    for side in ("arc_dlut", "arc_slut"):
        for x, y in zip(getattr(ra, side).ravel(), getattr(rb, side).ravel()):
            if not _same_lut(ra, int(x), rb, int(y)):
                return False
    return True


def _same_lut(ra, i, rb, j) -> bool:
    for p, f in (("lut_s_ptr", "lut_s_flat"), ("lut_l_ptr", "lut_l_flat"), ("lut_t_ptr", "lut_t_flat")):
        pa, pb = getattr(ra, p), getattr(rb, p)
        if not np.array_equal(getattr(ra, f)[pa[i]:pa[i + 1]], getattr(rb, f)[pb[j]:pb[j + 1]]):
            return False
    return True
