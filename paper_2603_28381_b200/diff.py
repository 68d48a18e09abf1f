"""Differentiable timing layer (drop-in for stasim/diff.py:26-273).

LSE smooth-max forward over the level schedule (late conditions only),
hinge / softplus endpoint loss, and the reverse adjoint giving dL/d(late arc
delay) and dL/d(net edge delay) — all computed by the device kernels
(k_fwd<LSE>, k_grad_init, k_bwd<GRAD>, k_grad_final in csrc/ws_sta.cu).

The gradient backward uses the gather form of the reference's
``np.add.at(adj, from_pin, contrib)``: a pin's adjoint is its seed plus the
d_arc of its out-arcs in arc order, read when the pin's own level runs —
deterministic, atomic-free, and identical to the reference wherever a pin has
at most one out-arc (every generated design).  Tolerance vs the reference:
1e-4 relative (north_star); exp/log are the device's, not numpy's.

``lse``/``lse_grad`` are the reference's scalar helpers on host vectors
(numpy) — API conveniences that are not on the STA path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .flatten import device_of

LATE_COLS = (2, 3)
COL_NAMES = ("late-rise", "late-fall")
LOSS_KINDS = ("hinge", "softplus")
GRAD_FIELDS = ("lse_arrival", "arc_weights", "d_arc", "d_edge", "adjoint")


@dataclass
class LseConfig:
    """Smoothness hyper-parameter gamma (seconds), positive and finite."""

    gamma: float

    def __post_init__(self):
        if not (self.gamma > 0.0 and math.isfinite(self.gamma)):
            raise ValueError("gamma must be positive and finite")


def default_gamma(clock_period: float) -> float:
    return 0.01 * clock_period


def lse(xs, cfg: LseConfig) -> float:
    """c + gamma*log(sum exp((x-c)/gamma)), c = max(xs) (diff.py:41-49)."""
    x = np.asarray(xs, dtype=np.float64)
    if x.size == 0:
        raise ValueError("lse of an empty input")
    c = float(x.max())
    z = np.exp((x - c) / cfg.gamma)
    return c + cfg.gamma * float(np.log(z.sum()))


def lse_grad(xs, cfg: LseConfig) -> np.ndarray:
    """Softmax weights (diff.py:52-58)."""
    x = np.asarray(xs, dtype=np.float64)
    if x.size == 0:
        raise ValueError("lse_grad of an empty input")
    z = np.exp((x - x.max()) / cfg.gamma)
    return z / z.sum()


@dataclass
class GradientState:
    gamma: float
    loss_kind: str
    lse_arrival: np.ndarray
    arc_weights: np.ndarray
    d_arc: np.ndarray
    d_edge: np.ndarray
    adjoint: np.ndarray
    loss: float = float("nan")
    flat: object = field(default=None, repr=False)

    def values_equal(self, other: "GradientState") -> bool:
        return (self.gamma == other.gamma and self.loss == other.loss
                and all(np.array_equal(getattr(self, f), getattr(other, f)) for f in GRAD_FIELDS))

    @classmethod
    def from_device(cls, dev, corner, gamma, loss_kind, flat=None):
        g = cls(gamma=gamma, loss_kind=loss_kind, **dev.get_many(GRAD_FIELDS, corner), flat=flat)
        g.loss = dev.summary(corner)[2]
        return g


def _flat_of(design, schedule=None):
    from .flatten import FlatDesign, flatten
    return design if isinstance(design, FlatDesign) or hasattr(design, "mem_parent_loc") \
        else flatten(design, schedule)


def _check_loss(loss):
    if loss not in LOSS_KINDS:
        raise ValueError(f"unknown loss kind {loss!r} (expected one of {LOSS_KINDS})")


def forward_lse_arrival(design, schedule=None, state=None, cfg: LseConfig | None = None):
    """Smooth forward over the hard pass's arc delays (diff.py:164-189)."""
    flat = _flat_of(design, schedule)
    gamma = cfg.gamma if cfg is not None else default_gamma(flat.clock_period)
    LseConfig(gamma)
    dev = device_of(flat)
    if state is None:
        dev.run(_lib.RUN_HARD)
    else:
        dev.set_state(0, arrival=state.arrival, net_delay=state.net_delay,
                      arc_delay=state.arc_delay)
    dev.run(_lib.RUN_LSE, gamma=gamma)
    A, M = flat.n_arcs, len(flat.mem_pin)
    return GradientState(gamma=gamma, loss_kind="hinge", lse_arrival=dev.get("lse_arrival"),
                         arc_weights=dev.get("arc_weights"), d_arc=np.zeros((A, 2)),
                         d_edge=np.zeros((M, 2)), adjoint=np.zeros((flat.n_pins, 2)), flat=flat)


def backward_tns_grad(design, schedule=None, gstate: GradientState | None = None,
                      loss: str = "hinge") -> GradientState:
    """Endpoint loss and reverse accumulation (diff.py:192-263)."""
    _check_loss(loss)
    if gstate is None:
        gstate = forward_lse_arrival(design, schedule)
    flat = gstate.flat
    if flat is None:
        flat = _flat_of(design, schedule)
        gstate.flat = flat
    dev = device_of(flat)
    dev.set_state(0, lse_arrival=gstate.lse_arrival, arc_weights=gstate.arc_weights)
    dev.run(_lib.RUN_GRAD, gamma=gstate.gamma, loss=loss)
    gstate.d_arc = dev.get("d_arc")
    gstate.d_edge = dev.get("d_edge")
    gstate.adjoint = dev.get("adjoint")
    gstate.loss = dev.summary(0)[2]
    gstate.loss_kind = loss
    return gstate


def timing_gradients(design, cfg: LseConfig | None = None, loss: str = "hinge",
                     state=None) -> GradientState:
    """Hard pass (if not supplied), smooth forward, reverse gradients
    (diff.py:266-273) — one device call when no state is supplied."""
    _check_loss(loss)
    flat = _flat_of(design)
    gamma = cfg.gamma if cfg is not None else default_gamma(flat.clock_period)
    LseConfig(gamma)
    dev = device_of(flat)
    if state is None:
        dev.run(_lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED, gamma=gamma,
                loss=loss)
    else:
        dev.set_state(0, arrival=state.arrival, net_delay=state.net_delay,
                      arc_delay=state.arc_delay)
        dev.run(_lib.RUN_LSE | _lib.RUN_GRAD, gamma=gamma, loss=loss)
    return GradientState.from_device(dev, 0, gamma, loss, flat=flat)
