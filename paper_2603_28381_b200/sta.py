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
