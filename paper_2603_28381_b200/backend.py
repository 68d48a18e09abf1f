"""Backend plugin (drop-in for stasim/backend.py:13-66).

One backend exists: ``"cuda"`` — the sm_100a kernels of libwarpstar_b200.so.
There is no CPU fallback and no multi-backend dispatch; ``get_backend`` of any
other name raises ``ValueError`` (the reference's test_backends.py:23-25
requires ``get_backend("gpu")`` to raise).  ``STASIM_NO_EXT`` is not honoured:
without the library the package fails loudly at first use.

The ``cuda`` backend module exposes the reference's raw per-level kernel
ABI (_kernels.pyx:84-91, 159-172, 213-219): numpy arrays in, output arrays
updated in place, through the C-ABI shims ws_rc_level / ws_forward_level /
ws_backward_level.  ``run_engine(flat, kernels=get_backend("cuda"))`` drives
them level by level exactly as the reference's driver does.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np

from ._lib import check, lib, ptr


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64_in(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _out(a):
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
        raise ValueError("output arrays must be C-contiguous float64")
    return a


def rc_level_raw(nets, net_ptr, net_root, root_cap, mem_pin, mem_parent_loc, mem_res, mem_cap,
                 root_net_of_pin, load, net_delay, impulse, reduce_width):
    nets, net_ptr, net_root = _i64(nets), _i64(net_ptr), _i64(net_root)
    mem_pin, mem_parent_loc, root_net_of_pin = _i64(mem_pin), _i64(mem_parent_loc), _i64(root_net_of_pin)
    root_cap, mem_res, mem_cap = _f64_in(root_cap), _f64_in(mem_res), _f64_in(mem_cap)
    check(lib().ws_rc_level(len(nets), ptr(nets), len(net_root), ptr(net_ptr), ptr(net_root),
                            ptr(root_cap), len(mem_pin), ptr(mem_pin), ptr(mem_parent_loc),
                            ptr(mem_res), ptr(mem_cap), len(root_net_of_pin), ptr(root_net_of_pin),
                            ptr(_out(load)), ptr(_out(net_delay)), ptr(_out(impulse)),
                            int(reduce_width)))


def forward_level_raw(nets, net_ptr, net_root, root_kind, mem_pin, net_in_ptr, net_in_arc,
                      arc_from, arc_dlut, arc_slut, lut_s_ptr, lut_l_ptr, lut_t_ptr, lut_s_flat,
                      lut_l_flat, lut_t_flat, load, net_delay, impulse, slew, arrival, arc_delay):
    a = [_i64(x) for x in (nets, net_ptr, net_root, root_kind, mem_pin, net_in_ptr, net_in_arc,
                           arc_from, arc_dlut, arc_slut, lut_s_ptr, lut_l_ptr, lut_t_ptr)]
    (nets, net_ptr, net_root, root_kind, mem_pin, net_in_ptr, net_in_arc, arc_from, arc_dlut,
     arc_slut, lut_s_ptr, lut_l_ptr, lut_t_ptr) = a
    f = [_f64_in(x) for x in (lut_s_flat, lut_l_flat, lut_t_flat, load, net_delay, impulse)]
    lut_s_flat, lut_l_flat, lut_t_flat, load, net_delay, impulse = f
    check(lib().ws_forward_level(len(nets), ptr(nets), len(net_root), ptr(net_ptr), ptr(net_root),
                                 ptr(root_kind), len(mem_pin), ptr(mem_pin), ptr(net_in_ptr),
                                 ptr(net_in_arc), len(arc_from), ptr(arc_from), ptr(arc_dlut),
                                 ptr(arc_slut), len(lut_s_ptr) - 1, ptr(lut_s_ptr), ptr(lut_l_ptr),
                                 ptr(lut_t_ptr), ptr(lut_s_flat), ptr(lut_l_flat), ptr(lut_t_flat),
                                 load.shape[0], ptr(load), ptr(net_delay), ptr(impulse),
                                 ptr(_out(slew)), ptr(_out(arrival)), ptr(_out(arc_delay))))


def backward_level_raw(nets, net_ptr, net_root, mem_pin, mem_out_ptr, mem_out_arc, arc_to,
                       net_delay, required, arc_delay):
    nets, net_ptr, net_root, mem_pin = _i64(nets), _i64(net_ptr), _i64(net_root), _i64(mem_pin)
    mem_out_ptr, mem_out_arc, arc_to = _i64(mem_out_ptr), _i64(mem_out_arc), _i64(arc_to)
    net_delay, arc_delay = _f64_in(net_delay), _f64_in(arc_delay)
    check(lib().ws_backward_level(len(nets), ptr(nets), len(net_root), ptr(net_ptr), ptr(net_root),
                                  len(mem_pin), ptr(mem_pin), ptr(mem_out_ptr), ptr(mem_out_arc),
                                  len(arc_to), ptr(arc_to), net_delay.shape[0], ptr(net_delay),
                                  ptr(_out(required)), ptr(arc_delay)))


cuda_kernels = SimpleNamespace(__name__="paper_2603_28381_b200.cuda_kernels",
                               rc_level=rc_level_raw, forward_level=forward_level_raw,
                               backward_level=backward_level_raw)
_ACTIVE = cuda_kernels


def backend_name() -> str:
    return "cuda"


def available_backends() -> dict:
    return {"cuda": cuda_kernels}


def get_backend(name: str):
    try:
        return available_backends()[name]
    except KeyError:
        raise ValueError(f"backend {name!r} not available (have {sorted(available_backends())})")


def rc_level(flat, state, nets, reduce_width=8, kernels=None):
    k = kernels if kernels is not None else _ACTIVE
    k.rc_level(nets, flat.net_ptr, flat.net_root, flat.root_cap, flat.mem_pin,
               flat.mem_parent_loc, flat.mem_res, flat.mem_cap, flat.root_net_of_pin,
               state.load, state.net_delay, state.impulse, reduce_width)


def forward_level(flat, state, nets, kernels=None):
    k = kernels if kernels is not None else _ACTIVE
    k.forward_level(nets, flat.net_ptr, flat.net_root, flat.root_kind, flat.mem_pin,
                    flat.net_in_ptr, flat.net_in_arc, flat.arc_from, flat.arc_dlut, flat.arc_slut,
                    flat.lut_s_ptr, flat.lut_l_ptr, flat.lut_t_ptr, flat.lut_s_flat,
                    flat.lut_l_flat, flat.lut_t_flat, state.load, state.net_delay, state.impulse,
                    state.slew, state.arrival, state.arc_delay)


def backward_level(flat, state, nets, kernels=None):
    k = kernels if kernels is not None else _ACTIVE
    k.backward_level(nets, flat.net_ptr, flat.net_root, flat.mem_pin, flat.mem_out_ptr,
                     flat.mem_out_arc, flat.arc_to, state.net_delay, state.required,
                     state.arc_delay)
