"""TimingState and the TNS/WNS summaries (drop-in for stasim/sta.py:37-73, 408-421).

The values come from the device: ``TimingState.from_device`` downloads a
corner's state; ``tns``/``wns`` run the device summary kernels (numpy's
pairwise summation tree reproduced exactly, so TNS equals the reference's
``np.minimum(s, 0).sum()`` bit for bit) over the given state's slack.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .netlist import N_COND

STATE_FIELDS = ("load", "net_delay", "impulse", "slew", "arrival", "required", "slack",
                "arc_delay")


@dataclass
class TimingState:
    """Per-pin, per-condition timing values plus the per-arc delay cache."""

    load: np.ndarray
    net_delay: np.ndarray
    impulse: np.ndarray
    slew: np.ndarray
    arrival: np.ndarray
    required: np.ndarray
    slack: np.ndarray
    arc_delay: np.ndarray
    n_levels: int = 0

    @classmethod
    def init(cls, flat) -> "TimingState":
        """Initial state (sta.py:51-68) — a host-side constructor for API
        users; the engine's own initialisation is the k_init kernel."""
        n = flat.n_pins
        z = lambda: np.zeros((n, N_COND))
        required = np.empty((n, N_COND))
        required[:, 0:2] = -np.inf
        required[:, 2:4] = np.inf
        state = cls(load=z(), net_delay=z(), impulse=z(), slew=z(), arrival=z(),
                    required=required, slack=z(), arc_delay=np.zeros((flat.n_arcs, N_COND)),
                    n_levels=flat.n_levels)
        if len(flat.pi_pin):
            state.arrival[flat.pi_pin] = flat.pi_arrival
            state.slew[flat.pi_pin] = flat.pi_slew
        if len(flat.ep_pin):
            np.minimum.at(state.required[:, 2:4], flat.ep_pin, flat.ep_required[:, 2:4])
            np.maximum.at(state.required[:, 0:2], flat.ep_pin, flat.ep_required[:, 0:2])
        return state

    @classmethod
    def from_device(cls, dev, corner: int = 0, n_levels: int = 0) -> "TimingState":
        return cls(**dev.get_many(STATE_FIELDS, corner), n_levels=n_levels)

    def values_equal(self, other: "TimingState", rtol=1e-6, atol=1e-22) -> bool:
        return all(
            np.allclose(getattr(self, f), getattr(other, f), rtol=rtol, atol=atol, equal_nan=True)
            for f in ("load", "net_delay", "impulse", "slew", "arrival", "required", "slack"))


def _summary(state: TimingState, flat):
    """(TNS, WNS) of ``state.slack`` by the device summary kernel.  Only the
    slack goes up (no value re-upload), and corner 0's own device slack is
    restored afterwards (device-to-device), so zero-copy views of the last
    pass stay valid."""
    import torch
    from .flatten import device_of
    dev = device_of(flat, upload_values=False)
    keep = dev.tensor("slack").clone()
    dev.set_state(0, slack=state.slack)
    dev.run(_lib.RUN_SUMMARY)
    out = dev.summary(0)
    dev.tensor("slack").copy_(keep)
    torch.cuda.current_stream().synchronize()
    return out


def tns_wns(state: TimingState, flat):
    """(TNS, WNS) from one device summary run."""
    if not len(flat.ep_pin):
        return 0.0, float("inf")
    t, w, _ = _summary(state, flat)
    return t, w


def tns(state: TimingState, flat) -> float:
    """Sum of negative late endpoint slacks, rise and fall (sta.py:408-414)."""
    if not len(flat.ep_pin):
        return 0.0
    return _summary(state, flat)[0]


def wns(state: TimingState, flat) -> float:
    """Worst late endpoint slack, uncapped; +inf with no endpoints (sta.py:417-421)."""
    if not len(flat.ep_pin):
        return float("inf")
    return _summary(state, flat)[1]


# ---------------------------------------------------------------------------
# the reference's oracle-level API (sta.py:79-205, 296-402, 424-446)

def _axis_pos(axis, q):
    """(index, fraction) of q on a sorted axis: upper_bound - 1 clamped to
    [0, n-2], fraction clamped to [0, 1]; a 1-point axis is a constant."""
    n = len(axis)
    if n == 1:
        return 0, 0, 0.0
    i = int(np.searchsorted(axis, q, side="right")) - 1
    i = min(max(i, 0), n - 2)
    a0, a1 = float(axis[i]), float(axis[i + 1])
    f = (float(q) - a0) / (a1 - a0)
    return i, i + 1, (0.0 if f < 0.0 else (1.0 if f > 1.0 else f))


def interpolate_lut(lut, slew: float, load: float) -> float:
    """Clamped bilinear interpolation of one table (sta.py:103-113): the
    same operation order as the device's lut_interp, so the value is the one
    the engine uses for that (slew, load)."""
    s0, s1, fs = _axis_pos(np.asarray(lut.slew_axis, dtype=np.float64), slew)
    l0, l1, fl = _axis_pos(np.asarray(lut.load_axis, dtype=np.float64), load)
    t = np.asarray(lut.table, dtype=np.float64)
    lo = (1.0 - fl) * float(t[s0, l0]) + fl * float(t[s0, l1])
    hi = (1.0 - fl) * float(t[s1, l0]) + fl * float(t[s1, l1])
    return float((1.0 - fs) * lo + fs * hi)


def _local_parent(net):
    """Parent of every member in [root] + members numbering (0 = root)."""
    where = {int(p): k + 1 for k, p in enumerate(net.member_pins)}
    return [0 if int(q) == int(net.root) else where[int(q)] for q in net.member_parents]


def compute_net_loads(net) -> np.ndarray:
    """(1+m, 4) loads of [root] + members (sta.py:156-173): a member's load is
    its cap plus its subtree's (children folded in, deepest index first); the
    root's is root_cap plus the sequential sum of the member loads."""
    m = len(net.member_pins)
    par = _local_parent(net)
    out = np.zeros((1 + m, N_COND))
    out[1:] = np.asarray(net.member_caps, dtype=np.float64).reshape(m, N_COND)
    for k in range(m, 0, -1):
        if par[k - 1]:
            out[par[k - 1]] = out[par[k - 1]] + out[k]
    acc = np.zeros(N_COND)
    for k in range(1, m + 1):
        acc = acc + out[k]
    out[0] = np.asarray(net.root_cap, dtype=np.float64) + acc
    return out


def compute_net_delays(net, loads) -> np.ndarray:
    """(1+m, 4) Elmore delays (sta.py:182-190): delay(root) = 0,
    delay(k) = delay(parent) + res(k) * load(k)."""
    m = len(net.member_pins)
    par = _local_parent(net)
    res = np.asarray(net.member_res, dtype=np.float64).reshape(m, N_COND)
    out = np.zeros((1 + m, N_COND))
    for k in range(1, m + 1):
        out[k] = out[par[k - 1]] + res[k - 1] * loads[k]
    return out


def compute_net_impulses(net, loads, delays) -> np.ndarray:
    """(1+m, 4) impulses (sta.py:193-202): sqrt(max(0, 2 r c d - d^2))."""
    m = len(net.member_pins)
    res = np.asarray(net.member_res, dtype=np.float64).reshape(m, N_COND)
    cap = np.asarray(net.member_caps, dtype=np.float64).reshape(m, N_COND)
    d = np.asarray(delays, dtype=np.float64)[1:]
    rad = 2.0 * res * cap * d - d * d
    out = np.zeros((1 + m, N_COND))
    out[1:] = np.sqrt(np.where(rad > 0.0, rad, 0.0))
    return out


def propagate_arrival(flat, state: TimingState) -> TimingState:
    """Forward pass over the levels on the device (sta.py:296-330): cell
    arcs into every arc-driven root, then the net edges, from the state's
    load / net_delay / impulse and PI seeds; updates slew, arrival and
    arc_delay of ``state`` in place (the per-level C-ABI kernels)."""
    from . import backend
    for li in range(flat.n_levels):
        backend.forward_level(flat, state, flat.schedule.levels[li], kernels=backend.cuda_kernels)
    return state


def propagate_required(flat, state: TimingState) -> TimingState:
    """Backward pass over the levels on the device (sta.py:356-391):
    required times folded over out-arcs and net members, then slack."""
    from . import backend, _lib
    from .flatten import device_of
    for li in range(flat.n_levels - 1, -1, -1):
        backend.backward_level(flat, state, flat.schedule.levels[li], kernels=backend.cuda_kernels)
    dev = device_of(flat, upload_values=False)
    dev.set_state(0, arrival=state.arrival, required=state.required)
    dev.run(_lib.RUN_SLACK)
    state.slack = dev.get("slack", 0)
    return state


def run_reference(design, schedule=None, reduce_mode: str = "sequential",
                  reduce_width: int = 8) -> TimingState:
    """The reference's full STA pass (sta.py:394-402) on the device:
    ``reduce_mode="sequential"`` sums a root's member loads the way the
    reference's np.add.reduceat does (first member + numpy's pairwise sum of
    the rest; the engine's reduce width 0); ``"tree"`` uses ``reduce_width``
    strided partials — run_engine's default is tree / 8 (test_warp.py:291-300)."""
    from .flatten import FlatDesign, flatten
    from .warp import run_engine
    if reduce_mode not in ("sequential", "tree"):
        raise ValueError(f"unknown reduce_mode {reduce_mode!r}")
    flat = design if isinstance(design, FlatDesign) or hasattr(design, "mem_parent_loc") \
        else flatten(design, schedule)
    return run_engine(flat, reduce_width=0 if reduce_mode == "sequential" else reduce_width)


def check_schedule(design, schedule) -> list:
    """Violations of the level-schedule invariants (sta.py:424-446): every
    net exactly once, at its level_of, strictly above every net it depends
    on (arc sources' nets and the net a feedthrough root belongs to)."""
    from .flatten import to_raw
    raw = to_raw(design)
    N = raw.n_nets
    level_of = np.asarray(schedule.level_of, dtype=np.int64)
    problems = []
    seen = np.zeros(N, dtype=np.int64)
    for li, nets in enumerate(schedule.levels):
        nets = np.asarray(nets, dtype=np.int64)
        np.add.at(seen, nets, 1)
        for n in nets[level_of[nets] != li]:
            problems.append(f"net {int(n)}: level_of says {int(level_of[n])}, found at {li}")
    # dependency edges d -> n (d must sit at a lower level)
    P = raw.n_pins
    mptr = np.asarray(raw.net_mptr, dtype=np.int64)
    member_net = np.full(P, -1, dtype=np.int64)
    member_net[np.asarray(raw.mem_pin, dtype=np.int64)] = np.repeat(np.arange(N), np.diff(mptr))
    root = np.asarray(raw.net_root, dtype=np.int64)
    root_net = np.full(P, -1, dtype=np.int64)
    root_net[root] = np.arange(N)
    src = member_net[np.asarray(raw.arc_from, dtype=np.int64)]
    dst = root_net[np.asarray(raw.arc_to, dtype=np.int64)]
    ok = (src >= 0) & (dst >= 0)
    d = np.concatenate([src[ok], member_net[root][member_net[root] >= 0]])
    n = np.concatenate([dst[ok], np.flatnonzero(member_net[root] >= 0)])
    if len(d):
        pairs = np.unique(n * N + d)
        n, d = pairs // N, pairs % N
        for i in np.flatnonzero(level_of[d] >= level_of[n]):
            problems.append(f"net {int(n[i])} at level {int(level_of[n[i]])} depends on net "
                            f"{int(d[i])} at level {int(level_of[d[i]])}")
    if not np.all(seen == 1):
        bad = np.flatnonzero(seen != 1)
        problems.append(f"nets {bad.tolist()} appear {seen[bad].tolist()} times")
    return problems
