"""Timing and gradient reports in the reference's text format
(/root/reference/pkg/src/stasim/reports.py:30-243).

A report is a ``#`` header (tool + version + report kind, the sha256 of the
design's canonical JSON document), ``key = value`` summary lines, a blank
line, a field-name line, then one row per (pin, condition) — timing — or per
arc and per net edge — gradients — with floats in Python's shortest
round-trip ``repr``.  The layout is the reference's, so reports written by
either package compare line by line; with ``run_reference`` semantics
(sequential reduce mode) the timing report of a design is byte-identical to
the reference's.  Reports hold no wall-clock times (those go to the run
manifest).
"""

from __future__ import annotations

import hashlib
import json

import numpy as np

from . import __version__
from .design_io import serialize_design
from .netlist import COND_NAMES

TIMING_FIELDS = ("pin", "condition", "load", "delay", "impulse", "slew", "arrival", "required",
                 "slack")
GRADIENT_FIELDS = ("id", "from", "to", "delay_late_rise", "delay_late_fall", "grad_late_rise",
                   "grad_late_fall")
LATE = ("late-rise", "late-fall")
TOOL = "stasim"          # the report format's tool tag (drop-in)


def design_hash(design) -> str:
    """sha256 of the canonical design document (or of the given text)."""
    doc = design if isinstance(design, str) else serialize_design(design)
    return hashlib.sha256(doc.encode("utf-8")).hexdigest()


def fmt(x) -> str:
    return repr(float(x))


def header(kind: str, dhash: str) -> list:
    return [f"# {TOOL} {__version__} {kind} report", f"# design sha256: {dhash}"]


def render_csv(columns, rows) -> str:
    return "\n".join([",".join(columns)] + [",".join(str(r[c]) for c in columns) for r in rows]) + "\n"


def _flat(design):
    from .flatten import FlatDesign, flatten
    return design if isinstance(design, FlatDesign) else flatten(design)


def _names(flat):
    d = getattr(flat, "design", None)
    return list(d.pin_names) if d is not None else [f"p{i}" for i in range(flat.n_pins)]


def timing_summary(flat, state, cost_report=None) -> dict:
    from .sta import tns_wns
    t, w = tns_wns(state, flat)
    return {"tns": t, "wns": w, "level_count": flat.n_levels, "pins": flat.n_pins,
            "nets": flat.n_nets}


def _hash_of(flat, dhash):
    if dhash is not None:
        return dhash
    if getattr(flat, "design", None) is None:
        from .flatten import flat_to_raw
        from .ingest import raw_hash
        return raw_hash(flat_to_raw(flat))         # no document: the flat arrays' content hash
    return design_hash(flat.design)


def timing_report(design, state, scheme: str = "reference", cost_report=None, dhash=None) -> str:
    """One row per (pin, condition) after the design summary."""
    flat = _flat(design)
    rows = header("timing", _hash_of(flat, dhash))
    rows.append(f"# scheme: {scheme}")
    for k, v in timing_summary(flat, state, cost_report).items():
        rows.append(f"{k} = {v if isinstance(v, (int, str)) else fmt(v)}")
    rows += ["", " ".join(TIMING_FIELDS)]
    cols = [np.asarray(getattr(state, f)) for f in
            ("load", "net_delay", "impulse", "slew", "arrival", "required", "slack")]
    for p, name in enumerate(_names(flat)):
        for c in range(4):
            rows.append(" ".join([name, COND_NAMES[c]] + [fmt(a[p, c]) for a in cols]))
    return "\n".join(rows) + "\n"


def max_grad_coordinate(gstate) -> tuple:
    """(kind, index, condition, value) of the largest-magnitude gradient."""
    best = ("none", -1, "", 0.0)
    for kind, arr in (("arc", gstate.d_arc), ("edge", gstate.d_edge)):
        a = np.asarray(arr)
        if a.size:
            i, j = divmod(int(np.abs(a).argmax()), 2)
            v = float(a[i, j])
            if kind == "arc" or abs(v) > abs(best[3]):      # arcs first, edges if larger
                best = (kind, i, LATE[j], v)
    return best


def gradient_report(design, state, gstate, fd_report=None, dhash=None) -> str:
    """Per arc and per net edge: its late delays and their loss gradients."""
    flat = _flat(design)
    names = _names(flat)
    rows = header("gradient", _hash_of(flat, dhash))
    rows += [f"loss = {fmt(gstate.loss)}", f"gamma = {fmt(gstate.gamma)}",
             f"loss_kind = {gstate.loss_kind}"]
    kind, idx, cond, val = max_grad_coordinate(gstate)
    rows.append(f"max_grad_coordinate = {kind}:{idx}:{cond} value {fmt(val)}")
    if fd_report is not None:
        rows += [f"finite_diff_max_rel_error = {fmt(fd_report.max_rel_error)}",
                 f"finite_diff_max_abs_error = {fmt(fd_report.max_abs_error)}",
                 f"finite_diff_epsilon_dominated = {fd_report.epsilon_dominated}"]
    rows += ["", " ".join(GRADIENT_FIELDS)]
    ad, nd = np.asarray(state.arc_delay), np.asarray(state.net_delay)
    da, de = np.asarray(gstate.d_arc), np.asarray(gstate.d_edge)
    for a, (f, t) in enumerate(zip(flat.arc_from, flat.arc_to)):
        rows.append(" ".join([f"arc:{a}", names[f], names[t], fmt(ad[a, 2]), fmt(ad[a, 3]),
                              fmt(da[a, 0]), fmt(da[a, 1])]))
    net_ptr, mem_net, pl = flat.net_ptr, flat.mem_net, flat.mem_parent_loc
    for k, pin in enumerate(flat.mem_pin):
        if pl[k] > 0:
            ppin = flat.mem_pin[net_ptr[mem_net[k]] + pl[k] - 1]
            d = (nd[pin, 2] - nd[ppin, 2], nd[pin, 3] - nd[ppin, 3])
        else:
            ppin = flat.net_root[mem_net[k]]
            d = (nd[pin, 2], nd[pin, 3])
        rows.append(" ".join([f"edge:{k}", names[ppin], names[pin], fmt(d[0]), fmt(d[1]),
                              fmt(de[k, 0]), fmt(de[k, 1])]))
    return "\n".join(rows) + "\n"


def fusion_summary(dhash: str, seq, fused) -> str:
    """Measured sequential vs fused pipeline passes (the reference's schedule
    report layout; makespans are CUDA-event milliseconds, not simulated
    cycles)."""
    rows = header("schedule", dhash)
    rows += [f"sequential_makespan = {fmt(seq.makespan_ms)}",
             f"fused_makespan = {fmt(fused.makespan_ms)}",
             f"fused_mode = {fused.mode}", f"fused_kernels = {fused.n_kernels}"]
    return "\n".join(rows) + "\n"


def run_manifest(command: str, config: dict, dhash, seed, outputs: list, wall_time_s) -> str:
    """JSON run manifest; wall_time_s is informational only."""
    return json.dumps({"tool": TOOL, "version": __version__, "command": command, "config": config,
                       "design_sha256": dhash, "seed": seed, "outputs": outputs,
                       "wall_time_s": wall_time_s}, indent=1) + "\n"
