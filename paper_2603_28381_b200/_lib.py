"""ctypes binding of libwarpstar_b200.so (include/warpstar.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2603_28381_b200/csrc``).  There is no fallback: if the library
is missing, importing the engine raises ``ImportError`` — the product path
never silently degrades to a CPU implementation.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WS_LIB") or os.path.join(HERE, "libwarpstar_b200.so")

WS_OK, WS_ERR_VALUE, WS_ERR_CYCLE, WS_ERR_NOMEM, WS_ERR_CUDA, WS_ERR_STATE = range(6)

# value fields
V_MEM_RES, V_MEM_CAP, V_ROOT_CAP, V_LUT_T, V_PI_ARRIVAL, V_PI_SLEW, V_EP_REQUIRED = range(7)
V_XY, V_RES0, V_CAP0, V_WIRE = range(7, 11)
# state fields
(F_LOAD, F_NET_DELAY, F_IMPULSE, F_SLEW, F_ARRIVAL, F_REQUIRED, F_SLACK, F_ARC_DELAY,
 F_LSE_ARRIVAL, F_ARC_WEIGHTS, F_D_ARC, F_D_EDGE, F_ADJOINT, F_SUMMARY) = range(14)
F_D_RES, F_D_CAP, F_D_ROOT_CAP, F_D_SLEW, F_D_LEN, F_D_XY = range(14, 20)
F_D_ARC_SUM, F_D_EDGE_SUM = 20, 21
STATE_FIELDS = {"load": F_LOAD, "net_delay": F_NET_DELAY, "impulse": F_IMPULSE, "slew": F_SLEW,
                "arrival": F_ARRIVAL, "required": F_REQUIRED, "slack": F_SLACK,
                "arc_delay": F_ARC_DELAY, "lse_arrival": F_LSE_ARRIVAL,
                "arc_weights": F_ARC_WEIGHTS, "d_arc": F_D_ARC, "d_edge": F_D_EDGE,
                "adjoint": F_ADJOINT, "summary": F_SUMMARY,
                "d_res": F_D_RES, "d_cap": F_D_CAP, "d_root_cap": F_D_ROOT_CAP,
                "d_slew": F_D_SLEW, "d_len": F_D_LEN, "d_xy": F_D_XY,
                "d_arc_sum": F_D_ARC_SUM, "d_edge_sum": F_D_EDGE_SUM}
VALUE_FIELDS = {"mem_res": V_MEM_RES, "mem_cap": V_MEM_CAP, "root_cap": V_ROOT_CAP,
                "lut_t_flat": V_LUT_T, "pi_arrival": V_PI_ARRIVAL, "pi_slew": V_PI_SLEW,
                "ep_required": V_EP_REQUIRED, "xy": V_XY, "res0": V_RES0, "cap0": V_CAP0,
                "wire": V_WIRE}
TOPO_FIELDS = ("net_ptr", "net_root", "root_kind", "mem_pin", "mem_parent_loc", "mem_net",
               "mem_local", "arc_from", "arc_to", "arc_dlut", "arc_slut", "net_in_ptr",
               "net_in_arc", "mem_out_ptr", "mem_out_arc", "net_m", "net_a", "net_o",
               "member_of_pin", "root_net_of_pin", "is_endpoint", "level_of", "level_ptr",
               "level_nets", "csr_pin_list", "csr_net_index")
TOPO = {name: i for i, name in enumerate(TOPO_FIELDS)}

RUN_HARD, RUN_LSE, RUN_GRAD, RUN_TWO_STREAM, RUN_FUSED, RUN_GRAPH, RUN_SUMMARY, RUN_SLACK = (
    1, 2, 4, 8, 16, 32, 64, 128)
RUN_PERSISTENT = 256
RUN_WIRE, RUN_POSGRAD, RUN_TIMED = 512, 1024, 2048
RUN_CORNER_SUM = 4096
LOSS_KINDS = {"hinge": 0, "softplus": 1}
DIMS_LEN = 11

# every symbol include/warpstar.h declares (checked by tests/test_lib_symbols.py)
EXPORTS = ("ws_abi_version", "ws_last_error", "ws_last_error_pin", "ws_create", "ws_destroy",
           "ws_dims", "ws_topology_len", "ws_get_topology", "ws_set_values",
           "ws_perturb_values", "ws_run", "ws_get", "ws_device_ptr", "ws_value_ptr",
           "ws_summary", "ws_last_launch_count", "ws_set_state", "ws_set_probe", "ws_rc_level", "ws_forward_level",
           "ws_backward_level", "ws_kernel_times", "ws_run_kernel")

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_i32p = ctypes.POINTER(ctypes.c_int32)
_c_f64p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


class DesignDesc(ctypes.Structure):
    _fields_ = [
        ("n_pins", ctypes.c_int64), ("n_nets", ctypes.c_int64), ("n_members", ctypes.c_int64),
        ("n_arcs", ctypes.c_int64), ("n_luts", ctypes.c_int64), ("n_pi", ctypes.c_int64),
        ("n_ep", ctypes.c_int64), ("lut_s_len", ctypes.c_int64), ("lut_l_len", ctypes.c_int64),
        ("lut_t_len", ctypes.c_int64), ("clock_period", ctypes.c_double),
        ("net_root", _vp), ("net_mptr", _vp), ("mem_pin", _vp), ("mem_parent_pin", _vp),
        ("mem_res", _vp), ("mem_cap", _vp), ("root_cap", _vp),
        ("arc_from", _vp), ("arc_to", _vp), ("arc_dlut", _vp), ("arc_slut", _vp),
        ("lut_s_ptr", _vp), ("lut_l_ptr", _vp), ("lut_t_ptr", _vp),
        ("lut_s_flat", _vp), ("lut_l_flat", _vp), ("lut_t_flat", _vp),
        ("pi_pin", _vp), ("pi_arrival", _vp), ("pi_slew", _vp),
        ("ep_pin", _vp), ("ep_required", _vp),
    ]


class CycleError(ValueError):
    """Combinational cycle; carries a pin on the cycle (flatten.py:22-28)."""

    def __init__(self, pin, name=None):
        self.pin = pin
        label = f"pin {pin}" if name is None else f"pin {pin} ({name})"
        super().__init__(f"combinational cycle through {label}")


_lib = None


def lib():
    """The loaded library; raises ImportError when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` or `make -C paper_2603_28381_b200/csrc` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    L.ws_abi_version.restype = ctypes.c_int
    L.ws_last_error.restype = ctypes.c_char_p
    L.ws_last_error_pin.restype = ctypes.c_int64
    L.ws_create.argtypes = [ctypes.POINTER(DesignDesc), ctypes.c_int, ctypes.POINTER(_vp)]
    L.ws_destroy.argtypes = [_vp]
    L.ws_destroy.restype = None
    L.ws_dims.argtypes = [_vp, _c_i64p]
    L.ws_topology_len.argtypes = [_vp, ctypes.c_int]
    L.ws_topology_len.restype = ctypes.c_int64
    L.ws_get_topology.argtypes = [_vp, ctypes.c_int, _c_i64p]
    L.ws_set_values.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp]
    L.ws_perturb_values.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                    ctypes.c_double, _vp]
    L.ws_run.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_double,
                         ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp]
    L.ws_run_kernel.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                ctypes.c_int, ctypes.c_int, _vp]
    L.ws_get.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp]
    L.ws_set_state.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp]
    L.ws_device_ptr.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp), _c_i64p]
    L.ws_value_ptr.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp), _c_i64p]
    L.ws_summary.argtypes = [_vp, ctypes.c_int, _c_f64p, _vp]
    L.ws_last_launch_count.argtypes = [_vp]
    _ip = ctypes.POINTER(ctypes.c_int)
    L.ws_kernel_times.argtypes = [_vp, _ip, _ip, ctypes.POINTER(ctypes.c_float), ctypes.c_int]
    L.ws_set_probe.argtypes = [_vp, _vp]
    i64, vp, d = ctypes.c_int64, _vp, ctypes.c_double
    L.ws_rc_level.argtypes = [i64, vp, i64, vp, vp, vp, i64, vp, vp, vp, vp, i64, vp, vp, vp, vp,
                              ctypes.c_int]
    L.ws_forward_level.argtypes = [i64, vp, i64, vp, vp, vp, i64, vp, vp, vp, i64, vp, vp, vp, i64,
                                   vp, vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp]
    L.ws_backward_level.argtypes = [i64, vp, i64, vp, vp, i64, vp, vp, vp, i64, vp, i64, vp, vp, vp]
    _lib = L
    return L


def check(rc):
    """Map a status code to the reference's exception types."""
    if rc == WS_OK:
        return
    L = lib()
    msg = (L.ws_last_error() or b"").decode(errors="replace")
    if rc == WS_ERR_VALUE:
        raise ValueError(msg)
    if rc == WS_ERR_CYCLE:
        raise CycleError(int(L.ws_last_error_pin()))
    if rc == WS_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"warpstar: {msg}")


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)
