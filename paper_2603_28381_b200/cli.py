"""Command-line surface (the reference's cli.py:65-147
``gen`` / ``sta`` / ``grad`` with ``--scheme cuda``, over this repo's design
files).

    python -m paper_2603_28381_b200 gen   --config cfg.json --out d.npz
    python -m paper_2603_28381_b200 sta   --design d.npz [--report r.txt] [--mode fused]
    python -m paper_2603_28381_b200 grad  --design d.npz [--gamma G] [--loss hinge] [--report r.txt]
    python -m paper_2603_28381_b200 place --design d.npz [--seed S] [--steps K]

Reports keep the reference's layout (reports.py:44-206): a ``#`` header with
the design hash, ``key = value`` summary lines, then one row per (pin,
condition) for timing, or per arc / net edge for gradients, with floats in
shortest round-trip form.  Pins are named ``p<id>`` (design files carry no
pin names) and the hash is the ingest file's content hash (ingest.raw_hash)
rather than the sha256 of the reference's JSON document.  Exit code 0 on
success, 2 on a bad design file or argument (cli.py:220-222).
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import __version__
from .netlist import COND_NAMES

TIMING_FIELDS = ("pin", "condition", "load", "delay", "impulse", "slew", "arrival", "required",
                 "slack")


def _f(x) -> str:
    return repr(float(x))


def _header(kind: str, dhash: str) -> list:
    return [f"# warpstar-b200 {__version__} {kind} report", f"# design sha256: {dhash}"]


def _config_from_doc(doc: dict):
    from .generator import FanoutDist, GeneratorConfig
    doc = dict(doc)
    fan = doc.pop("fanout", None)
    if fan is not None:
        fan = dict(fan)
        kind = fan.pop("kind")
        doc["fanout"] = FanoutDist(kind, **fan)
    return GeneratorConfig(**doc)


def timing_report(raw, dev, mode: str, corner: int = 0) -> str:
    from . import ingest
    tns, wns, _ = dev.summary(corner)
    st = {f: dev.get(f, corner) for f in ("load", "net_delay", "impulse", "slew", "arrival",
                                         "required", "slack")}
    lines = _header("timing", raw.meta.get("hash") or ingest.raw_hash(raw))
    lines.append(f"# scheme: cuda ({mode})")
    lines += [f"tns = {_f(tns)}", f"wns = {_f(wns)}", f"level_count = {dev.n_levels}",
              f"pins = {dev.n_pins}", f"nets = {dev.n_nets}", "", " ".join(TIMING_FIELDS)]
    cols = [st[f] for f in ("load", "net_delay", "impulse", "slew", "arrival", "required", "slack")]
    for p in range(dev.n_pins):
        for c in range(4):
            lines.append(" ".join([f"p{p}", COND_NAMES[c]] + [_f(a[p, c]) for a in cols]))
    return "\n".join(lines) + "\n"


def gradient_report(raw, dev, gamma: float, loss_kind: str, corner: int = 0) -> str:
    from . import ingest
    _, _, loss = dev.summary(corner)
    d_arc, d_edge = dev.get("d_arc", corner), dev.get("d_edge", corner)
    arc_delay, nd = dev.get("arc_delay", corner), dev.get("net_delay", corner)
    lines = _header("gradient", raw.meta.get("hash") or ingest.raw_hash(raw))
    lines += [f"loss = {_f(loss)}", f"gamma = {_f(gamma)}", f"loss_kind = {loss_kind}"]
    best = ("none", -1, "", 0.0)
    if d_arc.size:
        a, j = divmod(int(np.abs(d_arc).argmax()), 2)
        best = ("arc", a, ("late-rise", "late-fall")[j], float(d_arc[a, j]))
    if d_edge.size:
        k, j = divmod(int(np.abs(d_edge).argmax()), 2)
        if abs(d_edge[k, j]) > abs(best[3]):
            best = ("edge", k, ("late-rise", "late-fall")[j], float(d_edge[k, j]))
    lines.append(f"max_grad_coordinate = {best[0]}:{best[1]}:{best[2]} value {_f(best[3])}")
    lines += ["", "id from to delay_late_rise delay_late_fall grad_late_rise grad_late_fall"]
    for a in range(len(raw.arc_from)):
        lines.append(" ".join([f"arc:{a}", f"p{raw.arc_from[a]}", f"p{raw.arc_to[a]}",
                               _f(arc_delay[a, 2]), _f(arc_delay[a, 3]), _f(d_arc[a, 0]),
                               _f(d_arc[a, 1])]))
    par = np.asarray(raw.mem_parent_pin)
    root = np.repeat(np.asarray(raw.net_root), np.diff(np.asarray(raw.net_mptr)))
    for k in range(len(raw.mem_pin)):
        pin, pp = int(raw.mem_pin[k]), int(par[k])
        if pp == root[k]:
            dl = (nd[pin, 2], nd[pin, 3])
        else:
            dl = (nd[pin, 2] - nd[pp, 2], nd[pin, 3] - nd[pp, 3])
        lines.append(" ".join([f"edge:{k}", f"p{pp}", f"p{pin}", _f(dl[0]), _f(dl[1]),
                               _f(d_edge[k, 0]), _f(d_edge[k, 1])]))
    return "\n".join(lines) + "\n"


def _write_or_print(path, text):
    if path:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


def cmd_gen(args) -> int:
    from . import ingest
    from .generator import generate_raw
    with open(args.config, "r", encoding="utf-8") as fh:
        cfg = _config_from_doc(json.load(fh))
    raw = generate_raw(cfg)
    h = ingest.save_raw(args.out, raw)
    print(f"#Cells {cfg.num_cells}  #Nets {raw.n_nets}  #Pins {raw.n_pins}  sha256 {h}")
    return 0


_MODES = {"fused": "RUN_FUSED", "persistent": "RUN_PERSISTENT", "streams": "RUN_TWO_STREAM",
          "sequential": None}


def _run(args, grad: bool):
    from . import _lib, ingest
    from .engine import DeviceDesign
    raw = ingest.load_raw(args.design)
    dev = DeviceDesign(raw)
    flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
    if _MODES[args.mode]:
        flags |= getattr(_lib, _MODES[args.mode])
    t0 = time.perf_counter()
    gamma = dev.run(flags, gamma=getattr(args, "gamma", None), loss=getattr(args, "loss", "hinge"))
    dev.sync()
    print(f"# {args.mode} pass: {1e3 * (time.perf_counter() - t0):.3f} ms (host wall, first call)",
          file=sys.stderr)
    return raw, dev, gamma


def cmd_sta(args) -> int:
    raw, dev, _ = _run(args, False)
    _write_or_print(args.report, timing_report(raw, dev, args.mode))
    dev.close()
    return 0


def cmd_grad(args) -> int:
    raw, dev, gamma = _run(args, True)
    _write_or_print(args.report, gradient_report(raw, dev, gamma, args.loss))
    dev.close()
    return 0


def cmd_place(args) -> int:
    from . import ingest, placement
    from .engine import DeviceDesign
    raw = ingest.load_raw(args.design)
    pl = placement.synthetic_placement(raw, seed=args.seed)
    dev = DeviceDesign(raw)
    timer = placement.PlacementTimer(dev, pl, loss=args.loss)
    rng = np.random.default_rng(args.seed)
    for t in range(args.steps):
        xy = pl.xy + args.sigma * rng.standard_normal(pl.cell_xy.shape)[pl.cell_of_pin] * (t > 0)
        tns, wns, loss = timer.step(xy)
        g = timer.grad_xy()
        print(f"step {t}: loss {_f(loss)} tns {_f(tns)} wns {_f(wns)} max|dL/dxy| {_f(np.abs(g).max())}")
    dev.close()
    return 0


def build_parser():
    p = argparse.ArgumentParser(prog="python -m paper_2603_28381_b200",
                                description="B200 differentiable STA (Warp-STAR hot path)")
    p.add_argument("--version", action="version", version=__version__)
    sub = p.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen", help="generate a synthetic design file")
    g.add_argument("--config", required=True, help="GeneratorConfig JSON")
    g.add_argument("--out", required=True, help="design file (.npz)")
    g.set_defaults(func=cmd_gen)
    for name, func, help_ in (("sta", cmd_sta, "timing report"), ("grad", cmd_grad, "gradient report")):
        s = sub.add_parser(name, help=help_)
        s.add_argument("--design", required=True)
        s.add_argument("--report", default=None, help="output file (default stdout)")
        s.add_argument("--mode", default="fused", choices=tuple(_MODES))
        if name == "grad":
            s.add_argument("--gamma", type=float, default=None)
            s.add_argument("--loss", default="hinge", choices=("hinge", "softplus"))
        s.set_defaults(func=func)
    s = sub.add_parser("place", help="placement steps with position gradients")
    s.add_argument("--design", required=True)
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--steps", type=int, default=3)
    s.add_argument("--sigma", type=float, default=0.5, help="cell move std-dev (um) per step")
    s.add_argument("--loss", default="hinge", choices=("hinge", "softplus"))
    s.set_defaults(func=cmd_place)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except BrokenPipeError:
        return 0
    except (ValueError, OSError, KeyError) as exc:
        print(f"warpstar-b200: error: {exc}", file=sys.stderr)
        return 2
