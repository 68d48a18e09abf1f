"""Command-line surface (the reference's cli.py:43-258
``gen`` / ``sta`` / ``grad``).

    python -m paper_2603_28381_b200 gen   --config cfg.json --out d.json|d.npz
    python -m paper_2603_28381_b200 sta   --design d.json|d.npz [--scheme reference|cuda]
                                          [--report r.txt] [--mode fused]
    python -m paper_2603_28381_b200 grad  --design d.json|d.npz [--gamma G] [--loss hinge]
                                          [--check [--strict]] [--fuse] [--report r.txt]
    python -m paper_2603_28381_b200 place --design d.npz [--seed S] [--steps K]

Design files are the reference's JSON document (parse_design /
serialize_design) or this repo's hash-verified ``.npz`` ingest file.  Every
pass runs on the device.  ``--scheme reference`` (the default, as in the
reference) is run_reference's semantics — np.add.reduceat root loads — so the
timing report of a JSON design is byte-identical to ``stasim sta --scheme
reference``'s; ``--scheme cuda`` is run_engine's tree-8 pass (the reference's
engine).  Reports follow reports.py's layout; ``--report`` writes the report
and a run manifest and prints the summary.  Exit code 0 on success, 1 when a
requested check fails, 2 on a bad design file or argument (cli.py:220-222).
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import __version__

GRAD_CHECK_THRESHOLD = 1e-4
_MODES = {"fused": "RUN_FUSED", "persistent": "RUN_PERSISTENT", "streams": "RUN_TWO_STREAM",
          "sequential": None}


def _config_from_doc(doc: dict):
    from .generator import FanoutDist, GeneratorConfig
    doc = dict(doc)
    fan = doc.pop("fanout", None)
    if fan is not None:
        fan = dict(fan)
        kind = fan.pop("kind")
        doc["fanout"] = FanoutDist(kind, **fan)
    return GeneratorConfig(**doc)


def _write(path, text):
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(text)


def _load(path):
    """(design object or RawDesign, design hash) of a JSON document or an
    ingest file."""
    from . import ingest, reports
    from .design_io import parse_design
    if path.endswith(".npz"):
        raw = ingest.load_raw(path)
        return raw, raw.meta.get("hash") or ingest.raw_hash(raw)
    with open(path, "r", encoding="utf-8") as fh:
        text = fh.read()
    return parse_design(text), reports.design_hash(text)


def _flat(design):
    from .flatten import flatten
    return flatten(design)


def _state(flat, scheme, mode):
    """The timing state of the pass the scheme names."""
    from . import _lib
    from .sta import TimingState, run_reference
    if scheme == "reference":
        return run_reference(flat)
    dev = flat.dev
    flags = _lib.RUN_HARD | (getattr(_lib, _MODES[mode]) if _MODES[mode] else 0)
    if mode != "sequential":
        flags |= _lib.RUN_LSE | _lib.RUN_GRAD
    dev.run(flags)
    return TimingState.from_device(dev, 0, n_levels=flat.n_levels)


def cmd_gen(args) -> int:
    from . import ingest, reports
    from .generator import generate_design, generate_raw
    t0 = time.perf_counter()
    with open(args.config, "r", encoding="utf-8") as fh:
        cfg = _config_from_doc(json.load(fh))
    if args.out.endswith(".npz"):
        raw = generate_raw(cfg)
        dhash = ingest.save_raw(args.out, raw)
        n_nets, n_pins = raw.n_nets, raw.n_pins
    else:
        from .design_io import serialize_design
        d = generate_design(cfg)
        text = serialize_design(d)
        _write(args.out, text)
        dhash, n_nets, n_pins = reports.design_hash(text), len(d.nets), d.n_pins
    _write(args.out + ".manifest.json",
           reports.run_manifest("gen", cfg.to_doc(), dhash, cfg.seed, [args.out], time.perf_counter() - t0))
    print(f"#Cells {cfg.num_cells}  #Nets {n_nets}  #Pins {n_pins}")
    return 0


def cmd_sta(args) -> int:
    from . import reports
    t0 = time.perf_counter()
    design, dhash = _load(args.design)
    flat = _flat(design)
    state = _state(flat, args.scheme, args.mode)
    text = reports.timing_report(flat, state, args.scheme, dhash=dhash)
    if args.report:
        _write(args.report, text)
        _write(args.report + ".manifest.json",
               reports.run_manifest("sta", {"design": args.design, "scheme": args.scheme}, dhash,
                                    None, [args.report], time.perf_counter() - t0))
        for k, v in reports.timing_summary(flat, state).items():
            print(f"{k} = {v}")
    else:
        sys.stdout.write(text)
    return 0


def cmd_grad(args) -> int:
    from . import reports
    from .diff import LseConfig, default_gamma, finite_diff_check, timing_gradients
    if args.gamma is not None and not args.gamma > 0:
        print("warpstar-b200: error: --gamma must be > 0", file=sys.stderr)
        return 2
    if args.strict and not args.check:
        print("warpstar-b200: error: --strict requires --check", file=sys.stderr)
        return 2
    design, dhash = _load(args.design)
    flat = _flat(design)
    state = _state(flat, args.scheme, "fused")
    gamma = args.gamma if args.gamma is not None else default_gamma(flat.clock_period)
    cfg = LseConfig(gamma)
    gstate = timing_gradients(flat, cfg=cfg, loss=args.loss, state=state)
    fd = finite_diff_check(flat, cfg=cfg, loss=args.loss) if args.check else None
    text = reports.gradient_report(flat, state, gstate, fd, dhash=dhash)
    rc = 0
    if args.fuse:
        from .fusion import FusionConfig, execute_fused, execute_sequential
        fcfg = FusionConfig(granularity=args.granularity, gamma=gamma, loss=args.loss)
        st_s, gs_s, seq = execute_sequential(flat, cfg=fcfg)
        st_f, gs_f, fus = execute_fused(flat, cfg=FusionConfig(granularity=args.granularity, gamma=gamma,
                                                               loss=args.loss, mode="streams"))
        text += "\n" + reports.fusion_summary(dhash, seq, fus)
        same = (all(np.array_equal(getattr(st_s, f), getattr(st_f, f), equal_nan=True)
                    for f in ("load", "net_delay", "impulse", "slew", "arrival", "required", "slack",
                              "arc_delay")) and gs_s.values_equal(gs_f))
        if not same:
            print("warpstar-b200: fused pipeline values differ from sequential", file=sys.stderr)
            rc = 1
    if args.report:
        _write(args.report, text)
        _write(args.report + ".manifest.json",
               reports.run_manifest("grad", {"design": args.design, "gamma": gamma, "loss": args.loss},
                                    dhash, None, [args.report], None))
        print(f"loss = {gstate.loss!r}")
    else:
        sys.stdout.write(text)
    if args.check and args.strict and fd.max_rel_error > GRAD_CHECK_THRESHOLD:
        print(f"warpstar-b200: finite-difference max rel error {fd.max_rel_error:.3e} exceeds "
              f"{GRAD_CHECK_THRESHOLD:.0e}", file=sys.stderr)
        rc = 1
    return rc


def cmd_place(args) -> int:
    from . import ingest, placement
    from .engine import DeviceDesign
    raw = ingest.load_raw(args.design)
    pl = placement.synthetic_placement(raw, seed=args.seed)
    dev = DeviceDesign(raw)
    timer = placement.PlacementTimer(dev, pl, loss=args.loss)
    rng = np.random.default_rng(args.seed)
    f = lambda x: repr(float(x))
    for t in range(args.steps):
        xy = pl.xy + args.sigma * rng.standard_normal(pl.cell_xy.shape)[pl.cell_of_pin] * (t > 0)
        tns, wns, loss = timer.step(xy)
        g = timer.grad_xy()
        print(f"step {t}: loss {f(loss)} tns {f(tns)} wns {f(wns)} max|dL/dxy| {f(np.abs(g).max())}")
    dev.close()
    return 0


def build_parser():
    p = argparse.ArgumentParser(prog="python -m paper_2603_28381_b200",
                                description="B200 differentiable STA (Warp-STAR hot path)")
    p.add_argument("--version", action="version", version=f"stasim {__version__} (warpstar-b200)")
    sub = p.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen", help="generate a synthetic design (JSON document or .npz)")
    g.add_argument("--config", required=True, help="GeneratorConfig JSON")
    g.add_argument("--out", required=True, help="design file (.json or .npz)")
    g.set_defaults(func=cmd_gen)
    for name, func, help_ in (("sta", cmd_sta, "timing report"), ("grad", cmd_grad, "gradient report")):
        s = sub.add_parser(name, help=help_)
        s.add_argument("--design", required=True)
        s.add_argument("--scheme", default="reference", choices=("reference", "cuda"),
                       help="reference: run_reference semantics; cuda: the tree-8 engine pass")
        s.add_argument("--report", default=None, help="output file (stdout then carries the summary)")
        if name == "sta":
            s.add_argument("--mode", default="fused", choices=tuple(_MODES))
        else:
            s.add_argument("--gamma", type=float, default=None)
            s.add_argument("--loss", default="hinge", choices=("hinge", "softplus"))
            s.add_argument("--check", action="store_true", help="finite-difference gradient check")
            s.add_argument("--strict", action="store_true", help="with --check: exit 1 above 1e-4")
            s.add_argument("--fuse", action="store_true", help="sequential vs two-stream pipeline")
            s.add_argument("--granularity", type=int, default=10)
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
