"""CPU ORACLE (test infrastructure only) — Python driver over sta_oracle.c.

Restates the reference's driver-level routines over the C restatement of its
kernels:

* ``flatten_raw``   — flatten.py:170-316 + levelize flatten.py:44-80 + build_csr
                      netlist.py:370-380, from the flat ingest arrays;
* ``run_engine``    — warp.py:462-476 (per-level rc/forward, reverse backward,
                      slack);
* ``timing_gradients`` — diff.py:164-273 (LSE forward, endpoint loss, reverse
                      adjoint), seeded from the hard pass like
                      forward_lse_arrival (diff.py:176).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module.  The product package never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "sta_oracle.c")

ROOT_ARC_DRIVEN, ROOT_PI, ROOT_FEEDTHROUGH = 0, 1, 2


def build(force=False):
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", SRC,
                               "-o", LIB_PATH, "-lm"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.orc_levelize.restype = ctypes.c_int64
        _lib.orc_rc_level.restype = ctypes.c_int
        _lib.orc_endpoint_loss.restype = ctypes.c_double
        _lib.orc_interp.restype = ctypes.c_double
        _lib.orc_pairwise.restype = ctypes.c_double
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleCycleError(ValueError):
    def __init__(self, pin):
        self.pin = pin
        super().__init__(f"combinational cycle through pin {pin}")


def flatten_raw(raw):
    """FlatDesign-equivalent namespace (int64 indices, reference dtypes)."""
    L = lib()
    P = int(raw.n_pins)
    net_ptr = _i64(raw.net_mptr)
    net_root = _i64(raw.net_root)
    mem_pin = _i64(raw.mem_pin)
    mem_parent_pin = _i64(raw.mem_parent_pin)
    N, M = len(net_root), len(mem_pin)
    arc_from, arc_to = _i64(raw.arc_from), _i64(raw.arc_to)
    A = len(arc_from)
    member_of_pin = np.empty(P, np.int64)
    root_net_of_pin = np.empty(P, np.int64)
    mem_parent_loc = np.empty(M, np.int64)
    mem_net = np.empty(M, np.int64)
    mem_local = np.empty(M, np.int64)
    L.orc_maps(ctypes.c_int64(P), ctypes.c_int64(N), _p(net_ptr), _p(net_root), _p(mem_pin),
               _p(mem_parent_pin), _p(member_of_pin), _p(root_net_of_pin), _p(mem_parent_loc),
               _p(mem_net), _p(mem_local))
    level = np.empty(N, np.int64)
    nl = L.orc_levelize(ctypes.c_int64(P), ctypes.c_int64(N), _p(net_ptr), _p(net_root),
                        _p(mem_pin), ctypes.c_int64(A), _p(arc_from), _p(arc_to), _p(level))
    if nl < 0:
        raise OracleCycleError(int(net_root[-nl - 1]))
    levels = [np.flatnonzero(level == li).astype(np.int64) for li in range(nl)]

    def group(keys, nk):
        ptr = np.empty(nk + 1, np.int64)
        idx = np.empty(int((keys >= 0).sum()), np.int64)
        L.orc_group(ctypes.c_int64(len(keys)), _p(keys), ctypes.c_int64(nk), _p(ptr), _p(idx))
        return ptr, idx

    net_in_ptr, net_in_arc = group(_i64(root_net_of_pin[arc_to]) if A else np.zeros(0, np.int64), N)
    mem_out_ptr, mem_out_arc = group(_i64(member_of_pin[arc_from]) if A else np.zeros(0, np.int64), M)
    pi_pin = _i64(raw.pi_pin)
    ep_pin = _i64(raw.ep_pin)
    is_endpoint = np.zeros(P, dtype=bool)
    is_endpoint[ep_pin] = True
    pi_set = np.zeros(P, dtype=bool)
    pi_set[pi_pin] = True
    root_kind = np.full(N, ROOT_PI, np.int64)
    has_in = np.diff(net_in_ptr) > 0
    feed = member_of_pin[net_root] >= 0 if N else np.zeros(0, bool)
    root_kind[~has_in & feed] = ROOT_FEEDTHROUGH
    root_kind[has_in] = ROOT_ARC_DRIVEN
    net_m = np.diff(net_ptr)
    net_a = np.diff(net_in_ptr)
    net_o = mem_out_ptr[net_ptr[1:]] - mem_out_ptr[net_ptr[:-1]]
    # build_csr (netlist.py:370-380): root first, then members
    net_index = net_ptr + np.arange(N + 1, dtype=np.int64)
    pin_list = np.empty(N + M, np.int64)
    if N:
        pin_list[net_index[:-1]] = net_root
        pos = np.arange(M, dtype=np.int64) + mem_net + 1
        pin_list[pos] = mem_pin
    return SimpleNamespace(
        n_pins=P, n_nets=N, n_arcs=A, clock_period=float(raw.clock_period),
        levels=levels, level_of=level, n_levels=nl,
        net_ptr=net_ptr, net_root=net_root, root_cap=_f64(raw.root_cap).reshape(N, 4),
        root_kind=root_kind, mem_pin=mem_pin, mem_parent_loc=mem_parent_loc,
        mem_res=_f64(raw.mem_res).reshape(M, 4), mem_cap=_f64(raw.mem_cap).reshape(M, 4),
        mem_net=mem_net, mem_local=mem_local,
        lut_s_ptr=_i64(raw.lut_s_ptr), lut_l_ptr=_i64(raw.lut_l_ptr), lut_t_ptr=_i64(raw.lut_t_ptr),
        lut_s_flat=_f64(raw.lut_s_flat), lut_l_flat=_f64(raw.lut_l_flat),
        lut_t_flat=_f64(raw.lut_t_flat),
        arc_from=arc_from, arc_to=arc_to, arc_dlut=_i64(raw.arc_dlut).reshape(A, 4),
        arc_slut=_i64(raw.arc_slut).reshape(A, 4),
        net_in_ptr=net_in_ptr, net_in_arc=net_in_arc,
        mem_out_ptr=mem_out_ptr, mem_out_arc=mem_out_arc,
        net_m=net_m, net_a=net_a, net_o=net_o,
        member_of_pin=member_of_pin, root_net_of_pin=root_net_of_pin,
        pi_pin=pi_pin, pi_arrival=_f64(raw.pi_arrival).reshape(-1, 4),
        pi_slew=_f64(raw.pi_slew).reshape(-1, 4),
        ep_pin=ep_pin, ep_required=_f64(raw.ep_required).reshape(-1, 4),
        is_endpoint=is_endpoint, pin_list=pin_list, net_index=net_index,
    )


def init_state(flat):
    """TimingState.init (sta.py:51-68)."""
    P = flat.n_pins
    z = lambda: np.zeros((P, 4))
    req = np.empty((P, 4))
    req[:, 0:2] = -np.inf
    req[:, 2:4] = np.inf
    st = SimpleNamespace(load=z(), net_delay=z(), impulse=z(), slew=z(), arrival=z(),
                         required=req, slack=z(), arc_delay=np.zeros((flat.n_arcs, 4)))
    if len(flat.pi_pin):
        st.arrival[flat.pi_pin] = flat.pi_arrival
        st.slew[flat.pi_pin] = flat.pi_slew
    if len(flat.ep_pin):
        np.minimum.at(st.required[:, 2:4], flat.ep_pin, flat.ep_required[:, 2:4])
        np.maximum.at(st.required[:, 0:2], flat.ep_pin, flat.ep_required[:, 0:2])
    return st


def rc_level(flat, st, nets, w=8):
    nets = _i64(nets)
    rc = lib().orc_rc_level(ctypes.c_int64(len(nets)), _p(nets), _p(flat.net_ptr),
                            _p(flat.net_root), _p(flat.root_cap), _p(flat.mem_pin),
                            _p(flat.mem_parent_loc), _p(flat.mem_res), _p(flat.mem_cap),
                            _p(flat.root_net_of_pin), _p(st.load), _p(st.net_delay),
                            _p(st.impulse), ctypes.c_int(w))
    if rc != 0:
        raise MemoryError()


def forward_level(flat, st, nets):
    nets = _i64(nets)
    lib().orc_forward_level(ctypes.c_int64(len(nets)), _p(nets), _p(flat.net_ptr),
                            _p(flat.net_root), _p(flat.root_kind), _p(flat.mem_pin),
                            _p(flat.net_in_ptr), _p(flat.net_in_arc), _p(flat.arc_from),
                            _p(flat.arc_dlut), _p(flat.arc_slut), _p(flat.lut_s_ptr),
                            _p(flat.lut_l_ptr), _p(flat.lut_t_ptr), _p(flat.lut_s_flat),
                            _p(flat.lut_l_flat), _p(flat.lut_t_flat), _p(st.load),
                            _p(st.net_delay), _p(st.impulse), _p(st.slew), _p(st.arrival),
                            _p(st.arc_delay))


def backward_level(flat, st, nets):
    nets = _i64(nets)
    lib().orc_backward_level(ctypes.c_int64(len(nets)), _p(nets), _p(flat.net_ptr),
                             _p(flat.net_root), _p(flat.mem_pin), _p(flat.mem_out_ptr),
                             _p(flat.mem_out_arc), _p(flat.arc_to), _p(st.net_delay),
                             _p(st.required), _p(st.arc_delay))


def run_engine(flat, reduce_width=8):
    """warp.run_engine (warp.py:462-476)."""
    st = init_state(flat)
    for li in range(flat.n_levels):
        rc_level(flat, st, flat.levels[li], reduce_width)
        forward_level(flat, st, flat.levels[li])
    for li in range(flat.n_levels - 1, -1, -1):
        backward_level(flat, st, flat.levels[li])
    st.slack[:, 0:2] = st.arrival[:, 0:2] - st.required[:, 0:2]
    st.slack[:, 2:4] = st.required[:, 2:4] - st.arrival[:, 2:4]
    return st


def timing_gradients(flat, st, gamma=None, loss="hinge"):
    """diff.timing_gradients with state supplied (diff.py:266-273)."""
    L = lib()
    g = 0.01 * flat.clock_period if gamma is None else float(gamma)
    kind = {"hinge": 0, "softplus": 1}[loss]
    P, A, M = flat.n_pins, flat.n_arcs, len(flat.mem_pin)
    lse_at = np.ascontiguousarray(st.arrival[:, 2:4])
    arc_d = np.ascontiguousarray(st.arc_delay[:, 2:4])
    path = np.ascontiguousarray(st.net_delay[flat.mem_pin][:, 2:4]) if M else np.zeros((0, 2))
    weights = np.zeros((A, 2))
    scratch = np.zeros(2 * max(1, int(flat.net_a.max()) if len(flat.net_a) else 1))
    for li in range(flat.n_levels):
        nets = _i64(flat.levels[li])
        L.orc_lse_level(ctypes.c_int64(len(nets)), _p(nets), _p(flat.net_ptr), _p(flat.net_root),
                        _p(flat.root_kind), _p(flat.mem_pin), _p(flat.net_in_ptr),
                        _p(flat.net_in_arc), _p(flat.arc_from), ctypes.c_double(g), _p(lse_at),
                        _p(arc_d), _p(path), _p(weights), _p(scratch))
    adj = np.zeros((P, 2))
    E = len(flat.ep_pin)
    sc = np.zeros(max(1, 2 * E))
    lossv = L.orc_endpoint_loss(ctypes.c_int64(E), _p(flat.ep_pin), _p(flat.ep_required),
                                _p(lse_at), ctypes.c_double(g), ctypes.c_int(kind), _p(adj),
                                _p(sc))
    d_arc = np.zeros((A, 2))
    d_edge = np.zeros((M, 2))
    for li in range(flat.n_levels - 1, -1, -1):
        nets = _i64(flat.levels[li])
        L.orc_grad_level(ctypes.c_int64(len(nets)), _p(nets), _p(flat.net_ptr), _p(flat.net_root),
                         _p(flat.root_kind), _p(flat.mem_pin), _p(flat.mem_parent_loc),
                         _p(flat.net_in_ptr), _p(flat.net_in_arc), _p(flat.arc_from), _p(adj),
                         _p(d_arc), _p(d_edge), _p(weights))
    return SimpleNamespace(gamma=g, loss_kind=loss, lse_arrival=lse_at, arc_weights=weights,
                           d_arc=d_arc, d_edge=d_edge, adjoint=adj, loss=float(lossv))


def tns(st, flat):
    if not len(flat.ep_pin):
        return 0.0
    s = st.slack[flat.ep_pin][:, 2:4]
    return float(np.minimum(s, 0.0).sum())


def wns(st, flat):
    if not len(flat.ep_pin):
        return float("inf")
    return float(st.slack[flat.ep_pin][:, 2:4].min())


def interpolate(flat, lut, qs, ql):
    return lib().orc_interp(ctypes.c_int64(lut), _p(flat.lut_s_ptr), _p(flat.lut_l_ptr),
                            _p(flat.lut_t_ptr), _p(flat.lut_s_flat), _p(flat.lut_l_flat),
                            _p(flat.lut_t_flat), ctypes.c_double(qs), ctypes.c_double(ql))


# ---------------------------------------------------------------------------
# Position model + position gradients.  The reference
# has no position model (SPEC.md: pin-location gradients are a non-goal), so
# these are this repo's definitions, pinned by central finite differences of
# the reference-restated loss (tests/test_place_oracle.py).

def parent_pins(flat):
    """Parent pin of every member: the net root for depth 0, else the parent
    member's pin (mem_parent_loc, flatten.py:198-203)."""
    M = len(flat.mem_pin)
    if M == 0:
        return np.zeros(0, np.int64)
    pl = flat.mem_parent_loc
    root = flat.net_root[flat.mem_net]
    s = flat.net_ptr[flat.mem_net]
    par = np.where(pl > 0, flat.mem_pin[np.maximum(s + pl - 1, 0)], root)
    return np.ascontiguousarray(par, dtype=np.int64)


def pin_out(flat):
    """Arcs grouped by source pin, ascending arc id (CSR over all pins)."""
    P = flat.n_pins
    order = np.argsort(flat.arc_from, kind="stable").astype(np.int64)
    ptr = np.zeros(P + 1, np.int64)
    np.add.at(ptr, flat.arc_from + 1, 1)
    return np.cumsum(ptr), order


def wire(flat, xy, res0, cap0, r_unit, c_unit):
    """mem_res / mem_cap of the Manhattan wire model (orc_wire)."""
    M = len(flat.mem_pin)
    res, cap = np.zeros((M, 4)), np.zeros((M, 4))
    lib().orc_wire(ctypes.c_int64(M), _p(_i64(flat.mem_pin)), _p(parent_pins(flat)), _p(_f64(xy)),
                   _p(_f64(res0)), _p(_f64(cap0)), _p(_f64(r_unit)), _p(_f64(c_unit)), _p(res),
                   _p(cap))
    return res, cap


def with_values(flat, **arrays):
    """copy.copy(flat) with value arrays substituted."""
    import copy
    f = copy.copy(flat)
    for k, v in arrays.items():
        setattr(f, k, np.ascontiguousarray(v, dtype=np.float64))
    return f


def placed_loss(flat, xy, res0, cap0, r_unit, c_unit, gamma, loss="hinge"):
    """positions -> wire RC -> run_engine -> timing_gradients loss."""
    res, cap = wire(flat, xy, res0, cap0, r_unit, c_unit)
    f = with_values(flat, mem_res=res, mem_cap=cap)
    st = run_engine(f)
    return timing_gradients(f, st, gamma=gamma, loss=loss).loss


def interp_grad(flat, lut, qs, ql):
    out = np.zeros(2)
    lib().orc_interp_grad(ctypes.c_int64(lut), _p(flat.lut_s_ptr), _p(flat.lut_l_ptr),
                          _p(flat.lut_t_ptr), _p(flat.lut_s_flat), _p(flat.lut_l_flat),
                          _p(flat.lut_t_flat), ctypes.c_double(qs), ctypes.c_double(ql), _p(out))
    return out


def position_gradients(flat, st, gr, xy=None, r_unit=None, c_unit=None):
    """Reverse sweep of orc_posgrad_level over the levels (descending), then
    orc_pos_reduce when positions are given.  flat must hold the RC values the
    state was computed with."""
    L = lib()
    P, A, M, N = flat.n_pins, flat.n_arcs, len(flat.mem_pin), len(flat.net_root)
    po_ptr, po_arc = pin_out(flat)
    gs, gsr, gsa = np.zeros((P, 2)), np.zeros((P, 2)), np.zeros((A, 2))
    gl = np.zeros((N, 2))
    d_res, d_cap, d_root_cap = np.zeros((M, 2)), np.zeros((M, 2)), np.zeros((N, 2))
    mx = int(flat.net_m.max()) if N else 1
    scratch = np.zeros(3 * max(1, mx))
    adj = np.ascontiguousarray(gr.adjoint)
    d_arc = np.ascontiguousarray(gr.d_arc)
    for li in range(flat.n_levels - 1, -1, -1):
        nets = _i64(flat.levels[li])
        L.orc_posgrad_level(
            ctypes.c_int64(len(nets)), _p(nets), _p(flat.net_ptr), _p(flat.net_root),
            _p(flat.root_kind), _p(flat.mem_pin), _p(flat.mem_parent_loc), _p(flat.net_in_ptr),
            _p(flat.net_in_arc), _p(flat.arc_from), _p(flat.arc_dlut), _p(flat.arc_slut),
            _p(po_ptr), _p(po_arc), _p(flat.root_net_of_pin), _p(flat.lut_s_ptr),
            _p(flat.lut_l_ptr), _p(flat.lut_t_ptr), _p(flat.lut_s_flat), _p(flat.lut_l_flat),
            _p(flat.lut_t_flat), _p(flat.mem_res), _p(flat.mem_cap), _p(st.load),
            _p(st.net_delay), _p(st.impulse), _p(st.slew), _p(st.arrival), _p(st.arc_delay),
            _p(adj), _p(d_arc), _p(gs), _p(gsr), _p(gsa), _p(gl), _p(d_res), _p(d_cap),
            _p(d_root_cap), _p(scratch))
    out = SimpleNamespace(d_slew=gs, d_load=gl, d_res=d_res, d_cap=d_cap, d_root_cap=d_root_cap)
    if xy is not None:
        g_len, dxy = np.zeros(M), np.zeros((P, 2))
        L.orc_pos_reduce(ctypes.c_int64(M), _p(_i64(flat.mem_pin)), _p(parent_pins(flat)),
                         _p(_f64(xy)), _p(_f64(r_unit)), _p(_f64(c_unit)), _p(d_res), _p(d_cap),
                         _p(g_len), _p(dxy))
        out.g_len, out.d_xy = g_len, dxy
    return out
