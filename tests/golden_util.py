"""Loaders for the golden fixtures produced by tests/golden/make_golden.py
(outputs of the reference itself)."""

import glob
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

ST_FIELDS = ("load", "net_delay", "impulse", "slew", "arrival", "required", "slack", "arc_delay")
G_FIELDS = ("lse_arrival", "arc_weights", "d_arc", "d_edge", "adjoint")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def raw_of(g):
    from paper_2603_28381_b200.netlist import RawDesign
    kw = {k[4:]: v for k, v in g.items() if k.startswith("raw_")}
    return RawDesign(n_pins=int(g["n_pins"]), clock_period=float(g["clock_period"]), **kw).normalized()


def raw_ns(g):
    return SimpleNamespace(n_pins=int(g["n_pins"]), clock_period=float(g["clock_period"]),
                           **{k[4:]: v for k, v in g.items() if k.startswith("raw_")})


def max_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return float("inf")
    fa, fb = np.isfinite(a), np.isfinite(b)
    if not np.array_equal(fa, fb):
        return float("inf")
    if not np.array_equal(a[~fa], b[~fb]):
        return float("inf")
    if not fa.any():
        return 0.0
    d = np.abs(a[fa] - b[fa])
    return float((d / np.maximum(np.abs(b[fa]), 1e-30)).max())


def grad_close(a, b, rtol=1e-4):
    """north_star gradient tolerance: 1e-4 relative, elementwise, with a floor
    of 1e-9 x the array's largest magnitude for entries that are ~0."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    fa, fb = np.isfinite(a), np.isfinite(b)
    if not np.array_equal(fa, fb):
        return False
    if not fa.any():
        return True
    scale = float(np.abs(b[fb]).max())
    floor = 1e-9 * scale if scale > 0 else 1e-300
    d = np.abs(a[fa] - b[fb])
    return bool(np.all(d <= rtol * np.maximum(np.abs(b[fb]), floor)))
