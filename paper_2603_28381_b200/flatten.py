"""Levelization and the flat array form of a design — built on the device.

Drop-in for /root/reference/pkg/src/stasim/flatten.py: ``levelize``,
``flatten``, ``FlatDesign``, ``LevelSchedule``, ``CycleError`` and
netlist.py's ``build_csr``/``CsrNetlist``.  The host only packs the design
into flat arrays (``netlist.design_to_raw``); every index array — member maps,
parent locations, arcs grouped by driven net and by source member, root
kinds, per-net counts, the longest-path level schedule and the Alg.1 CSR — is
computed by the ws_create kernels (csrc/ws_build.cu) and downloaded here as
int64 arrays identical to the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._lib import CycleError
from .engine import DeviceDesign
from .netlist import RawDesign, design_to_raw

ROOT_ARC_DRIVEN = 0
ROOT_PI = 1
ROOT_FEEDTHROUGH = 2

__all__ = ["CycleError", "LevelSchedule", "FlatDesign", "CsrNetlist", "levelize", "flatten",
           "build_csr", "to_raw", "device_of"]


@dataclass
class LevelSchedule:
    """Nets grouped into dependency levels (flatten.py:31-41)."""

    levels: list
    level_of: np.ndarray

    @property
    def n_levels(self):
        return len(self.levels)


@dataclass
class CsrNetlist:
    """Root-first pin CSR (netlist.py:360-367)."""

    pin_list: np.ndarray
    net_index: np.ndarray


def to_raw(design) -> RawDesign:
    if isinstance(design, RawDesign):
        return design.normalized()
    if isinstance(design, FlatDesign) or hasattr(design, "mem_parent_loc"):
        return flat_to_raw(design)
    return design_to_raw(design)


def _device_for(design, n_corners=1) -> DeviceDesign:
    return DeviceDesign(to_raw(design), n_corners=n_corners)


def levelize(design) -> LevelSchedule:
    """Longest-chain levels, computed on the device (flatten.py:44-80).
    Raises CycleError naming the root pin of the lowest-index stuck net."""
    dev = _device_for(design)
    try:
        return LevelSchedule(levels=dev.levels(), level_of=dev.topology("level_of"))
    finally:
        dev.close()


def build_csr(design) -> CsrNetlist:
    """Alg.1 layout with the root stored first (netlist.py:370-380), on device."""
    dev = _device_for(design)
    try:
        return CsrNetlist(pin_list=dev.topology("csr_pin_list"),
                          net_index=dev.topology("csr_net_index"))
    finally:
        dev.close()


@dataclass
class FlatDesign:
    """Field-for-field the reference's FlatDesign (flatten.py:83-136), plus the
    device context ``dev`` that holds the same arrays in HBM."""

    design: object
    schedule: LevelSchedule
    n_pins: int
    n_nets: int
    n_arcs: int
    clock_period: float
    net_ptr: np.ndarray
    net_root: np.ndarray
    root_cap: np.ndarray
    root_kind: np.ndarray
    mem_pin: np.ndarray
    mem_parent_loc: np.ndarray
    mem_res: np.ndarray
    mem_cap: np.ndarray
    mem_net: np.ndarray
    mem_local: np.ndarray
    lut_s_ptr: np.ndarray
    lut_l_ptr: np.ndarray
    lut_t_ptr: np.ndarray
    lut_s_flat: np.ndarray
    lut_l_flat: np.ndarray
    lut_t_flat: np.ndarray
    arc_from: np.ndarray
    arc_to: np.ndarray
    arc_dlut: np.ndarray
    arc_slut: np.ndarray
    net_in_ptr: np.ndarray
    net_in_arc: np.ndarray
    mem_out_ptr: np.ndarray
    mem_out_arc: np.ndarray
    net_m: np.ndarray
    net_a: np.ndarray
    net_o: np.ndarray
    member_of_pin: np.ndarray
    root_net_of_pin: np.ndarray
    pi_pin: np.ndarray
    pi_arrival: np.ndarray
    pi_slew: np.ndarray
    ep_pin: np.ndarray
    ep_required: np.ndarray
    is_endpoint: np.ndarray
    dev: DeviceDesign | None = field(default=None, repr=False, compare=False)
    _level_cache: dict = field(default_factory=dict, repr=False)

    @property
    def n_levels(self):
        return self.schedule.n_levels

    def level_nets(self, li):
        return self.schedule.levels[li]

    def level_view(self, li):
        """Per-level gathered indices (flatten.py:147-167), host-side
        convenience for callers that iterate levels."""
        hit = self._level_cache.get(li)
        if hit is not None:
            return hit
        nets = self.schedule.levels[li]
        mem_idx = (np.concatenate([np.arange(self.net_ptr[n], self.net_ptr[n + 1]) for n in nets])
                   .astype(np.int64) if len(nets) else np.zeros(0, dtype=np.int64))
        mem_seg = np.zeros(len(nets) + 1, dtype=np.int64)
        np.cumsum(self.net_m[nets], out=mem_seg[1:])
        arc_nets = nets[self.root_kind[nets] == ROOT_ARC_DRIVEN]
        arc_idx = (np.concatenate([self.net_in_arc[self.net_in_ptr[n]:self.net_in_ptr[n + 1]]
                                   for n in arc_nets]).astype(np.int64)
                   if len(arc_nets) else np.zeros(0, dtype=np.int64))
        arc_seg = np.zeros(len(arc_nets) + 1, dtype=np.int64)
        np.cumsum(self.net_a[arc_nets], out=arc_seg[1:])
        view = (nets, mem_idx, mem_seg, arc_nets, arc_idx, arc_seg)
        self._level_cache[li] = view
        return view


def flatten(design, schedule: LevelSchedule | None = None, n_corners: int = 1) -> FlatDesign:
    """Upload ``design`` and build its FlatDesign on the device.

    ``design`` may be a reference ``stasim.Design``, this package's
    ``Design`` or a ``RawDesign``.  A caller-supplied ``schedule`` is kept as
    the FlatDesign's schedule (results are schedule-invariant for any valid
    schedule; the device runs its own)."""
    raw = to_raw(design)
    dev = DeviceDesign(raw, n_corners=n_corners)
    flat = _make_flat(design, raw, dev, schedule)
    return flat


def _make_flat(design, raw, dev, schedule):
    if schedule is None:
        schedule = LevelSchedule(levels=dev.levels(), level_of=dev.topology("level_of"))
    t = dev.topology
    n, m, a = raw.n_nets, raw.n_members, raw.n_arcs
    i64 = lambda x: np.asarray(x, dtype=np.int64)
    flat = FlatDesign(
        design=design if not isinstance(design, RawDesign) else None, schedule=schedule,
        n_pins=int(raw.n_pins), n_nets=n, n_arcs=a, clock_period=float(raw.clock_period),
        net_ptr=t("net_ptr"), net_root=t("net_root"), root_cap=raw.root_cap.reshape(n, 4).copy(),
        root_kind=t("root_kind"), mem_pin=t("mem_pin"), mem_parent_loc=t("mem_parent_loc"),
        mem_res=raw.mem_res.reshape(m, 4).copy(), mem_cap=raw.mem_cap.reshape(m, 4).copy(),
        mem_net=t("mem_net"), mem_local=t("mem_local"),
        lut_s_ptr=i64(raw.lut_s_ptr), lut_l_ptr=i64(raw.lut_l_ptr), lut_t_ptr=i64(raw.lut_t_ptr),
        lut_s_flat=raw.lut_s_flat.copy(), lut_l_flat=raw.lut_l_flat.copy(),
        lut_t_flat=raw.lut_t_flat.copy(),
        arc_from=t("arc_from"), arc_to=t("arc_to"), arc_dlut=t("arc_dlut"), arc_slut=t("arc_slut"),
        net_in_ptr=t("net_in_ptr"), net_in_arc=t("net_in_arc"),
        mem_out_ptr=t("mem_out_ptr"), mem_out_arc=t("mem_out_arc"),
        net_m=t("net_m"), net_a=t("net_a"), net_o=t("net_o"),
        member_of_pin=t("member_of_pin"), root_net_of_pin=t("root_net_of_pin"),
        pi_pin=i64(raw.pi_pin), pi_arrival=raw.pi_arrival.reshape(-1, 4).copy(),
        pi_slew=raw.pi_slew.reshape(-1, 4).copy(),
        ep_pin=i64(raw.ep_pin), ep_required=raw.ep_required.reshape(-1, 4).copy(),
        is_endpoint=t("is_endpoint"), dev=dev,
    )
    flat._dev_key = _topo_key(flat)
    return flat


def flat_to_raw(flat) -> RawDesign:
    """A FlatDesign (ours or the reference's) back to ingest arrays: member
    parents as pins (mem_parent_loc 0 -> the root, k -> member k-1)."""
    net_ptr = np.asarray(flat.net_ptr, dtype=np.int64)
    mem_pin = np.asarray(flat.mem_pin, dtype=np.int64)
    pl = np.asarray(flat.mem_parent_loc, dtype=np.int64)
    n = len(net_ptr) - 1
    m = len(mem_pin)
    mem_net = np.repeat(np.arange(n, dtype=np.int64), np.diff(net_ptr))
    parent = np.asarray(flat.net_root, dtype=np.int64)[mem_net].copy() if m else np.zeros(0, np.int64)
    inner = pl > 0
    parent[inner] = mem_pin[net_ptr[mem_net[inner]] + pl[inner] - 1]
    return RawDesign(
        n_pins=int(flat.n_pins), clock_period=float(flat.clock_period),
        net_root=flat.net_root, net_mptr=net_ptr, mem_pin=mem_pin, mem_parent_pin=parent,
        mem_res=flat.mem_res, mem_cap=flat.mem_cap, root_cap=flat.root_cap,
        arc_from=flat.arc_from, arc_to=flat.arc_to, arc_dlut=flat.arc_dlut, arc_slut=flat.arc_slut,
        lut_s_ptr=flat.lut_s_ptr, lut_l_ptr=flat.lut_l_ptr, lut_t_ptr=flat.lut_t_ptr,
        lut_s_flat=flat.lut_s_flat, lut_l_flat=flat.lut_l_flat, lut_t_flat=flat.lut_t_flat,
        pi_pin=flat.pi_pin, pi_arrival=flat.pi_arrival, pi_slew=flat.pi_slew,
        ep_pin=flat.ep_pin, ep_required=flat.ep_required,
    ).normalized()


_TOPO_KEYS = ("net_ptr", "net_root", "mem_pin", "mem_parent_loc", "arc_from", "arc_to",
              "arc_dlut", "arc_slut", "lut_s_ptr", "lut_l_ptr", "lut_t_ptr", "lut_s_flat",
              "lut_l_flat", "pi_pin", "ep_pin")


def _topo_key(flat):
    return tuple(id(getattr(flat, k)) for k in _TOPO_KEYS)


def device_of(flat, upload_values: bool = True) -> DeviceDesign:
    """The device context of a FlatDesign with the flat's CURRENT value arrays
    uploaded (callers may substitute mem_res/mem_cap/... as the reference's
    copy.copy(flat) workflow does).  Rebinding an index array
    (e.g. ``flat2.ep_pin = ...``) gets a freshly built device context;
    mutating index arrays in place is not supported."""
    dev = getattr(flat, "dev", None)
    key = _topo_key(flat)
    if dev is None or getattr(flat, "_dev_key", None) != key:
        dev = DeviceDesign(flat_to_raw(flat))
        try:
            flat.dev = dev
            flat._dev_key = key
        except AttributeError:
            pass
    elif upload_values:
        dev.set_values(0, mem_res=flat.mem_res, mem_cap=flat.mem_cap, root_cap=flat.root_cap,
                       lut_t_flat=flat.lut_t_flat, pi_arrival=flat.pi_arrival,
                       pi_slew=flat.pi_slew, ep_required=flat.ep_required)
    return dev
