"""Position model and position gradients (north_star: "run backward for
gradients w.r.t. pin/cell positions").

The reference's gradients stop at delay space — ``d_arc`` and ``d_edge``
(diff.py:5-7; SPEC.md lists pin-location gradients as a non-goal) — so this
module adds the missing link on the device:

* a Manhattan wire model, evaluated by ``k_wire`` at the start of a pass
  (``RUN_WIRE``): member edge k between member pin p and its parent pin q
  (the net root at depth 0) has length ``len = |x_p - x_q| + |y_p - y_q|`` and
  ``mem_res = res0 + r_unit * len``, ``mem_cap = cap0 + c_unit * len``
  (per condition);
* the reverse-mode derivative of the reference's forward functions
  (rc_level, _interp, forward_level, _lse_forward_level) after the pass
  (``RUN_POSGRAD``): slew / load adjoints level by level, the Elmore adjoint
  of every net, then dL/dx, dL/dy per pin.

The CPU restatement is oracle/sta_oracle.c (orc_wire, orc_posgrad_level,
orc_pos_reduce); it is pinned by central finite differences of the
reference-restated loss (tests/test_place_oracle.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import DeviceDesign
from .netlist import RawDesign


@dataclass
class WireModel:
    """Per-unit-length wire resistance (ohm/um) and capacitance (F/um) per
    condition (ER, EF, LR, LF)."""

    r_unit: np.ndarray
    c_unit: np.ndarray

    def packed(self) -> np.ndarray:
        r = np.broadcast_to(np.asarray(self.r_unit, np.float64), (4,))
        c = np.broadcast_to(np.asarray(self.c_unit, np.float64), (4,))
        if not (np.all(np.isfinite(r)) and np.all(np.isfinite(c))):
            raise ValueError("wire coefficients must be finite")
        return np.concatenate([r, c]).astype(np.float64)


@dataclass
class Placement:
    """Pin coordinates (um), base RC per member edge, the wire model and the
    cell of every pin (for cell-level gradients)."""

    xy: np.ndarray          # (P,2)
    res0: np.ndarray        # (M,4)
    cap0: np.ndarray        # (M,4)
    wire: WireModel
    cell_of_pin: np.ndarray  # (P,) int64, cell (anchor) id of every pin
    cell_xy: np.ndarray      # (n_cells,2)
    pin_offset: np.ndarray   # (P,2) xy = cell_xy[cell_of_pin] + pin_offset


def parent_pins(raw: RawDesign) -> np.ndarray:
    """Parent pin of every member edge (the root for depth-0 members)."""
    return np.ascontiguousarray(raw.mem_parent_pin, dtype=np.int64)


def member_lengths(raw: RawDesign, xy: np.ndarray) -> np.ndarray:
    p, q = raw.mem_pin, parent_pins(raw)
    return np.abs(xy[p, 0] - xy[q, 0]) + np.abs(xy[p, 1] - xy[q, 1])


def synthetic_placement(raw: RawDesign, seed: int = 0, die_um: float = 1000.0,
                        wire_res_share: float = 0.9) -> Placement:
    """A deterministic placement of a generated design (this repo's synthetic
    input; the reference has no placement).

    Cells: every arc target (cell output) anchors its cell; a pin that
    sources an arc belongs to the cell of that arc's target; other pins are
    their own cell.  Cells are spread along x in pin-id order (generator
    layers are contiguous in id, so x follows logic depth) and uniformly in
    y; pins sit within +-1 um of their cell.  The wire coefficients are
    calibrated so that the mean member edge keeps the design's mean RC:
    ``wire_res_share`` of the resistance and all but the pin capacitance
    (res0 = (1 - share) * mem_res, cap0 = mem_cap / 2) come from length.
    """
    P = raw.n_pins
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))
    anchor = np.arange(P, dtype=np.int64)
    if len(raw.arc_from):
        anchor[raw.arc_from] = raw.arc_to      # input pin -> its cell's output pin
    anchors, cell_of_pin = np.unique(anchor, return_inverse=True)
    nc = len(anchors)
    rank = np.argsort(np.argsort(anchors, kind="stable"), kind="stable")
    cx = (rank + 0.5) / max(nc, 1) * die_um + rng.uniform(-2.0, 2.0, nc)
    cy = rng.uniform(0.0, die_um, nc)
    cell_xy = np.stack([cx, cy], axis=1)
    off = rng.uniform(-1.0, 1.0, (P, 2))
    xy = cell_xy[cell_of_pin] + off
    res = np.asarray(raw.mem_res, np.float64)
    cap = np.asarray(raw.mem_cap, np.float64)
    M = len(raw.mem_pin)
    if M:
        ln = member_lengths(raw, xy)
        mean_len = float(ln.mean()) if float(ln.mean()) > 0 else 1.0
        r_unit = wire_res_share * res.mean(axis=0) / mean_len
        c_unit = 0.5 * cap.mean(axis=0) / mean_len
    else:
        r_unit = c_unit = np.zeros(4)
    return Placement(xy=np.ascontiguousarray(xy), res0=(1.0 - wire_res_share) * res,
                     cap0=0.5 * cap, wire=WireModel(r_unit, c_unit),
                     cell_of_pin=cell_of_pin.astype(np.int64), cell_xy=cell_xy,
                     pin_offset=off)


def cell_gradients(d_xy, cell_of_pin, n_cells):
    """dL/d(cell x, y) = sum of its pins' dL/dxy (pins move with their cell).
    Works on numpy arrays or torch CUDA tensors."""
    if hasattr(d_xy, "is_cuda"):
        import torch
        out = torch.zeros((n_cells, 2), dtype=d_xy.dtype, device=d_xy.device)
        idx = cell_of_pin if hasattr(cell_of_pin, "is_cuda") else torch.as_tensor(
            cell_of_pin, device=d_xy.device)
        return out.index_add_(0, idx, d_xy)
    out = np.zeros((n_cells, 2))
    np.add.at(out, cell_of_pin, d_xy)
    return out


class PlacementTimer:
    """Timing-driven placement step on one B200: positions in, loss / TNS /
    WNS and dL/dxy out.

    ``step(xy)`` uploads positions (numpy host array or torch tensor; device
    tensors are copied D2D), then one ``ws_run`` does wire RC -> RC ->
    forward + LSE -> backward + adjoint -> position gradients on the
    device."""

    FLAGS = (_lib.RUN_WIRE | _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED
             | _lib.RUN_POSGRAD)

    def __init__(self, dev: DeviceDesign, placement: Placement, corner: int = 0,
                 gamma: float | None = None, loss: str = "hinge", graph: bool = True):
        self.dev, self.corner, self.loss_kind = dev, corner, loss
        self.gamma = 0.01 * dev.clock_period if gamma is None else float(gamma)
        self.flags = self.FLAGS | (_lib.RUN_GRAPH if graph else 0)
        dev.set_values(corner, res0=placement.res0, cap0=placement.cap0,
                       wire=placement.wire.packed(), xy=placement.xy)

    def set_positions(self, xy, stream=None):
        self.dev.set_values(self.corner, stream=stream, xy=xy)

    def step(self, xy=None, stream=None):
        if xy is not None:
            self.set_positions(xy, stream)
        self.dev.run(self.flags, corner=self.corner, gamma=self.gamma, loss=self.loss_kind,
                     stream=stream)
        return self.dev.summary(self.corner, stream)

    def grad_xy(self):
        return self.dev.get("d_xy", self.corner)

    def grad_xy_tensor(self):
        return self.dev.tensor("d_xy", self.corner)

    def gradients(self):
        """Host copies of every position-gradient array of the last step."""
        return {k: self.dev.get(k, self.corner)
                for k in ("d_res", "d_cap", "d_root_cap", "d_slew", "d_len", "d_xy")}


def descend(timer: PlacementTimer, placement: Placement, steps: int = 20, step_um: float = 1.0,
            stream=None):
    """A timing-driven placement loop on the device: every iteration runs one
    PlacementTimer step (wire RC -> pass -> dL/dxy), reduces the pin
    gradients to their cells and moves every cell against its gradient by at
    most ``step_um`` (the gradient is normalised by its largest cell
    component, so the step is scale-free).  Returns the (loss, tns, wns)
    history; the final coordinates stay in the timer's corner.

    This is the C4 workload with real gradient steps instead of random
    perturbations."""
    import torch
    dev = timer.dev
    xy = torch.as_tensor(placement.xy, device="cuda").clone()
    cell_xy = torch.as_tensor(placement.cell_xy, device="cuda").clone()
    cop = torch.as_tensor(placement.cell_of_pin, device="cuda")
    off = torch.as_tensor(placement.pin_offset, device="cuda")
    n_cells = cell_xy.shape[0]
    hist = []
    for _ in range(steps):
        torch.add(cell_xy.index_select(0, cop), off, out=xy)
        tns, wns, loss = timer.step(xy, stream=stream)
        hist.append((loss, tns, wns))
        g = cell_gradients(timer.grad_xy_tensor(), cop, n_cells)
        scale = g.abs().max()
        if float(scale) == 0.0:
            break
        cell_xy -= (step_um / scale) * g
    dev.sync(stream)
    return hist
