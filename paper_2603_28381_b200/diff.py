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


# ---------------------------------------------------------------------------
# finite-difference validation (diff.py:339-474)

@dataclass
class FiniteDiffReport:
    max_rel_error: float
    max_abs_error: float
    worst_coordinate: tuple | None   # (kind, index, condition name)
    n_coords: int
    n_significant: int
    epsilon: float
    gamma: float
    epsilon_dominated: bool
    loss_kind: str
    n_refined: int = 0

    def __str__(self):
        flag = " [epsilon-dominated]" if self.epsilon_dominated else ""
        return (f"finite-diff: max rel {self.max_rel_error:.3e} (abs {self.max_abs_error:.3e}) over "
                f"{self.n_significant}/{self.n_coords} coords at eps={self.epsilon:.3e}, "
                f"gamma={self.gamma:.3e}{flag}")


def _smooth_loss_ld(flat, gamma, seed, arc_d, edges, loss):
    """The smooth loss in extended precision (numpy long double) from seed
    arrivals (P,2), late arc delays (A,2) and member edge delays (M,2): LSE
    over every arc-driven root's in-arcs, level by level, root + path delay
    for the members, then the hinge / softplus endpoint loss (the
    definitions of diff.py:123-212).  Finite-difference quotients need the
    extra digits: a coordinate's loss change is ~eps * |grad| while the loss
    itself carries FP64 rounding of ~1e-16 * |loss|."""
    ld = np.longdouble
    g = ld(gamma)
    lse = np.asarray(seed, dtype=ld).copy()
    net_ptr = np.asarray(flat.net_ptr, dtype=np.int64)
    pl = np.asarray(flat.mem_parent_loc, dtype=np.int64)
    mem_net = np.asarray(flat.mem_net, dtype=np.int64)
    path = np.zeros_like(np.asarray(edges, dtype=ld))
    e = np.asarray(edges, dtype=ld)
    # cumulative path delay: members are topologically ordered within a net
    local = np.asarray(flat.mem_local, dtype=np.int64)
    for pos in range(int(local.max()) + 1 if len(local) else 0):
        idx = np.flatnonzero(local == pos)
        par = pl[idx]
        base = np.zeros((len(idx), 2), dtype=ld)
        inner = par > 0
        base[inner] = path[net_ptr[mem_net[idx[inner]]] + par[inner] - 1]
        path[idx] = e[idx] + base
    in_ptr = np.asarray(flat.net_in_ptr, dtype=np.int64)
    in_arc = np.asarray(flat.net_in_arc, dtype=np.int64)
    a_from = np.asarray(flat.arc_from, dtype=np.int64)
    roots = np.asarray(flat.net_root, dtype=np.int64)
    mem_pin = np.asarray(flat.mem_pin, dtype=np.int64)
    ad = np.asarray(arc_d, dtype=ld)
    for li in range(flat.n_levels):
        nets = np.asarray(flat.schedule.levels[li], dtype=np.int64)
        cnt = in_ptr[nets + 1] - in_ptr[nets]
        drv = nets[cnt > 0]
        if len(drv):
            c = cnt[cnt > 0]
            arcs = np.concatenate([in_arc[in_ptr[n]:in_ptr[n + 1]] for n in drv])
            seg = np.concatenate([[0], np.cumsum(c)[:-1]])
            x = lse[a_from[arcs]] + ad[arcs]
            cm = np.maximum.reduceat(x, seg, axis=0)
            z = np.exp((x - np.repeat(cm, c, axis=0)) / g)
            lse[roots[drv]] = cm + g * np.log(np.add.reduceat(z, seg, axis=0))
        mem = np.concatenate([np.arange(net_ptr[n], net_ptr[n + 1]) for n in nets]) if len(nets) else []
        if len(mem):
            lse[mem_pin[mem]] = lse[roots[mem_net[mem]]] + path[mem]
    v = lse[np.asarray(flat.ep_pin, dtype=np.int64)] - np.asarray(flat.ep_required, dtype=ld)[:, 2:4]
    if loss == "hinge":
        return np.maximum(v, 0).sum()
    return (np.maximum(v, 0) + g * np.log1p(np.exp(-np.abs(v) / g))).sum()


def finite_diff_check(design, cfg: LseConfig | None = None, epsilon: float | None = None,
                      loss: str = "hinge", grad_floor: float = 1e-8,
                      refine_threshold: float = 1e-5) -> FiniteDiffReport:
    """Central finite differences of the smooth loss against the device's
    analytic d_arc / d_edge, one late-column coordinate at a time
    (diff.py:339-474).  The device runs the hard pass (seed arrivals, arc and
    net delays) and the analytic gradients; the perturbed losses are
    evaluated on the host in long double, as the reference does, because an
    FP64 quotient of a coordinate with |grad| ~ 1e-7 is noise-limited at
    ~1e-3.  ``refine_threshold`` is accepted for API compatibility: the
    reference re-checks such coordinates with mpmath; the extended-precision
    quotients here are not refined (n_refined = 0)."""
    _check_loss(loss)
    flat = _flat_of(design)
    if epsilon is not None and epsilon <= 0:
        raise ValueError("epsilon must be positive")
    gamma = cfg.gamma if cfg is not None else default_gamma(flat.clock_period)
    LseConfig(gamma)
    eps = float(epsilon) if epsilon is not None else 1e-6 * flat.clock_period
    dev = device_of(flat)
    dev.run(_lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED, gamma=gamma, loss=loss)
    got = dev.get_many(("arrival", "arc_delay", "net_delay", "d_arc", "d_edge"))
    ld = np.longdouble
    seed = got["arrival"][:, 2:4].astype(ld)
    arc_d = got["arc_delay"][:, 2:4].astype(ld)
    mem_pin = np.asarray(flat.mem_pin, dtype=np.int64)
    nd = got["net_delay"][mem_pin][:, 2:4].astype(ld)
    pl = np.asarray(flat.mem_parent_loc, dtype=np.int64)
    net_ptr = np.asarray(flat.net_ptr, dtype=np.int64)
    pidx = np.where(pl > 0, net_ptr[np.asarray(flat.mem_net, dtype=np.int64)] + pl - 1, 0)
    edges = nd - np.where((pl > 0)[:, None], nd[pidx], ld(0))
    e = ld(eps)
    rows = []
    for a in range(flat.n_arcs):
        for j in range(2):
            up, dn = arc_d.copy(), arc_d.copy()
            up[a, j] += e
            dn[a, j] -= e
            fd = (_smooth_loss_ld(flat, gamma, seed, up, edges, loss)
                  - _smooth_loss_ld(flat, gamma, seed, dn, edges, loss)) / (2 * e)
            rows.append((float(got["d_arc"][a, j]), float(fd), ("arc", a, COL_NAMES[j])))
    for k in range(len(mem_pin)):
        for j in range(2):
            up, dn = edges.copy(), edges.copy()
            up[k, j] += e
            dn[k, j] -= e
            fd = (_smooth_loss_ld(flat, gamma, seed, arc_d, up, loss)
                  - _smooth_loss_ld(flat, gamma, seed, arc_d, dn, loss)) / (2 * e)
            rows.append((float(got["d_edge"][k, j]), float(fd), ("edge", k, COL_NAMES[j])))
    max_rel = max_abs = 0.0
    worst = None
    n_sig = 0
    for an, fd, coord in rows:
        err = abs(fd - an)
        max_abs = max(max_abs, err)
        if abs(an) > grad_floor:
            n_sig += 1
            if err / abs(an) > max_rel:
                max_rel, worst = err / abs(an), coord
    return FiniteDiffReport(max_rel_error=max_rel, max_abs_error=max_abs, worst_coordinate=worst,
                            n_coords=2 * (flat.n_arcs + len(mem_pin)), n_significant=n_sig,
                            epsilon=eps, gamma=gamma, epsilon_dominated=bool(eps >= 0.1 * gamma),
                            loss_kind=loss, n_refined=0)
