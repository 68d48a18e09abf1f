"""Engine driver (drop-in for stasim/warp.py:462-476 run_engine).

``run_engine(flat)`` runs the whole hard pass on the device in one call
(init, RC, forward per level, backward in reverse, slack, TNS/WNS) and
returns the TimingState.  With ``kernels=`` a kernel module (for instance
``get_backend("cuda")``, or any module with the reference's raw level-kernel
ABI) it instead drives that module level by level like the reference's
driver.  The warp cost simulator is out of scope: real warp
efficiency is measured with ncu.
"""

from __future__ import annotations

from . import _lib, backend
from .flatten import device_of
from .sta import TimingState


def run_engine(flat, reduce_width: int | None = None, kernels=None) -> TimingState:
    w = reduce_width if reduce_width is not None else 8
    if kernels is None:
        dev = device_of(flat)
        dev.run(_lib.RUN_HARD, reduce_width=w)
        st = TimingState.from_device(dev, 0, n_levels=flat.n_levels)
        return st
    state = TimingState.init(flat)
    for li in range(flat.n_levels):
        nets = flat.schedule.levels[li]
        backend.rc_level(flat, state, nets, reduce_width=w, kernels=kernels)
        backend.forward_level(flat, state, nets, kernels=kernels)
    for li in range(flat.n_levels - 1, -1, -1):
        backend.backward_level(flat, state, flat.schedule.levels[li], kernels=kernels)
    # slack: one device elementwise pass over the state
    dev = device_of(flat)
    dev.set_state(0, arrival=state.arrival, required=state.required)
    dev.run(_lib.RUN_SLACK)
    state.slack = dev.get("slack", 0)
    return state

