"""Device-resident design context (the fast path behind the drop-in API).

``DeviceDesign`` owns one ``ws_ctx``: the design's topology lives on the GPU
as int32 CSR arrays built there (levels, net/member/arc groupings), and each
of ``n_corners`` value slots holds FP64 values plus the full TimingState and
GradientState of that corner.  Results stay in HBM; they are handed out as
numpy copies (``get``) or as zero-copy torch CUDA tensors (``tensor``).

Everything numeric runs in libwarpstar_b200.so; this module only marshals
pointers.  Streams are torch streams (``torch.cuda.current_stream()`` by
default), so CUDA-event timing and torch.distributed collectives compose
with the engine's kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import check, lib, ptr
from .netlist import RawDesign

_LATE = slice(2, 4)


_CUDA_STREAM_LEGACY = 1   # cudaStreamLegacy: torch's default stream has handle 0


def _stream_handle(stream):
    """The cudaStream_t the engine enqueues on: the caller's torch stream.
    Torch's default stream reports handle 0, which the C ABI would read as
    "the context's own stream"; it is passed as cudaStreamLegacy instead so
    the engine's copies and kernels stay ordered with the caller's torch work
    (a default-stream ``torch.add`` followed by ``set_values``)."""
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                h = torch.cuda.current_stream().cuda_stream
                return ctypes.c_void_p(h or _CUDA_STREAM_LEGACY)
        except Exception:  # torch absent / no device: the library's own stream
            pass
        return ctypes.c_void_p(0)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream or _CUDA_STREAM_LEGACY)
    return ctypes.c_void_p(stream.cuda_stream or _CUDA_STREAM_LEGACY)


class _CudaArray:
    """__cuda_array_interface__ view of device memory owned by the context."""

    def __init__(self, dptr, shape, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8",
                                         "data": (int(dptr), False), "version": 3,
                                         "strides": None}
        self._owner = owner


class DeviceDesign:
    """One design on the device with ``n_corners`` value/state slots."""

    def __init__(self, raw: RawDesign, n_corners: int = 1, validate: bool = True):
        raw = raw.normalized()
        if validate:
            # what the device build relies on (tree order, one driver per pin,
            # increasing LUT axes); the full model check is design_io.validate
            from .design_io import check_engine_invariants
            check_engine_invariants(raw)
        self.raw = raw
        L = lib()
        d = _lib.DesignDesc()
        d.n_pins, d.n_nets, d.n_members = raw.n_pins, raw.n_nets, raw.n_members
        d.n_arcs, d.n_luts = raw.n_arcs, raw.n_luts
        d.n_pi, d.n_ep = len(raw.pi_pin), len(raw.ep_pin)
        d.lut_s_len, d.lut_l_len, d.lut_t_len = (len(raw.lut_s_flat), len(raw.lut_l_flat),
                                                  len(raw.lut_t_flat))
        d.clock_period = raw.clock_period
        for f in ("net_root", "net_mptr", "mem_pin", "mem_parent_pin", "mem_res", "mem_cap",
                  "root_cap", "arc_from", "arc_to", "arc_dlut", "arc_slut", "lut_s_ptr",
                  "lut_l_ptr", "lut_t_ptr", "lut_s_flat", "lut_l_flat", "lut_t_flat", "pi_pin",
                  "pi_arrival", "pi_slew", "ep_pin", "ep_required"):
            setattr(d, f, ptr(getattr(raw, f)))
        h = ctypes.c_void_p()
        check(L.ws_create(ctypes.byref(d), int(n_corners), ctypes.byref(h)))
        self._h = h
        dims = np.zeros(_lib.DIMS_LEN, dtype=np.int64)
        check(L.ws_dims(h, dims.ctypes.data_as(_lib._c_i64p)))
        (self.n_pins, self.n_nets, self.n_members, self.n_arcs, self.n_pi, self.n_ep,
         self.n_levels, self.n_luts, self.n_corners, self.max_in, self.max_m) = map(int, dims)
        self.clock_period = raw.clock_period

    # -- lifetime ---------------------------------------------------------
    @classmethod
    def from_file(cls, path: str, n_corners: int = 1, verify: bool = True) -> "DeviceDesign":
        """Ingest a design written by ingest.save_raw (hash-verified)."""
        from .ingest import load_raw
        return cls(load_raw(path, verify=verify), n_corners=n_corners)

    def close(self):
        if getattr(self, "_h", None):
            lib().ws_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- topology ------------------------------------------------------------
    def topology(self, name: str) -> np.ndarray:
        """A FlatDesign/LevelSchedule/CsrNetlist index array (int64, host)."""
        L = lib()
        f = _lib.TOPO[name]
        n = L.ws_topology_len(self._h, f)
        if n < 0:
            check(_lib.WS_ERR_VALUE)
        out = np.empty(int(n), dtype=np.int64)
        if n:
            check(L.ws_get_topology(self._h, f, out.ctypes.data_as(_lib._c_i64p)))
        if name in ("arc_dlut", "arc_slut"):
            out = out.reshape(-1, 4)
        if name == "is_endpoint":
            out = out.astype(bool)
        return out

    def levels(self):
        ptr_ = self.topology("level_ptr")
        nets = self.topology("level_nets")
        return [nets[ptr_[i]:ptr_[i + 1]] for i in range(len(ptr_) - 1)]

    # -- values ----------------------------------------------------------------
    def set_values(self, corner: int, stream=None, **arrays):
        """Replace value arrays of one corner (numpy host arrays or torch CUDA
        tensors): mem_res, mem_cap, root_cap, lut_t_flat, pi_arrival, pi_slew,
        ep_required; position model: xy, res0, cap0, wire (see placement.py)."""
        L = lib()
        for name, a in arrays.items():
            f = _lib.VALUE_FIELDS[name]
            on_dev = 0
            if hasattr(a, "is_cuda"):
                # torch tensor: device memory (D2D) or (pinned) host memory (async H2D)
                import torch
                src = a
                a = a.contiguous()
                if a.dtype != torch.float64:
                    raise TypeError(f"{name}: expected float64")
                p, on_dev = ctypes.c_void_p(a.data_ptr()), 1 if a.is_cuda else 0
                keep = a
                temp_host = (not a.is_cuda) and a is not src
            else:
                keep = np.ascontiguousarray(a, dtype=np.float64)
                p = ptr(keep)
                temp_host = False   # pageable H2D: staged before the call returns
            n = ctypes.c_int64()
            dp = ctypes.c_void_p()
            check(L.ws_value_ptr(self._h, corner, f, ctypes.byref(dp), ctypes.byref(n)))
            if (keep.numel() if hasattr(keep, "numel") else keep.size) != n.value:
                raise ValueError(f"{name}: expected {n.value} values")
            check(L.ws_set_values(self._h, corner, f, p, on_dev, _stream_handle(stream)))
            if temp_host:   # a contiguous copy of a pinned tensor: let the DMA land first
                self.sync(stream)
            del keep

    def perturb(self, corner: int, base_corner: int, seed: int, sigma: float = 0.01, stream=None):
        """C4 placement-loop stand-in: scale mem_res / mem_cap / root_cap of
        ``base_corner`` by 1 + sigma*clip(N(0,1), +-3) into ``corner``."""
        check(lib().ws_perturb_values(self._h, corner, base_corner, ctypes.c_uint64(seed),
                                      float(sigma), _stream_handle(stream)))

    def value_tensor(self, name: str, corner: int = 0):
        return self._tensor(lib().ws_value_ptr, _lib.VALUE_FIELDS[name], corner, name)

    # -- run ---------------------------------------------------------------------
    def run(self, flags: int, corner: int = 0, n_corners: int = 1, gamma: float | None = None,
            loss: str = "hinge", reduce_width: int = 8, granularity: int = 10, stream=None,
            grad_stream=None):
        g = 0.01 * self.clock_period if gamma is None else float(gamma)
        if loss not in _lib.LOSS_KINDS:
            raise ValueError(f"unknown loss kind {loss!r} (expected one of {tuple(_lib.LOSS_KINDS)})")
        check(lib().ws_run(self._h, corner, n_corners, flags, g, _lib.LOSS_KINDS[loss],
                           int(reduce_width), int(granularity), _stream_handle(stream),
                           _stream_handle(grad_stream) if grad_stream is not None else None))
        return g

    def last_launch_count(self) -> int:
        return int(lib().ws_last_launch_count(self._h))

    def kernel_times(self):
        """[(kind, level, ms)] of the last RUN_TIMED pass (fusion.py kinds)."""
        cap = 8 * (self.n_levels + 4)
        kind = (ctypes.c_int * cap)()
        level = (ctypes.c_int * cap)()
        ms = (ctypes.c_float * cap)()
        n = lib().ws_kernel_times(self._h, kind, level, ms, cap)
        if n < 0:
            check(_lib.WS_ERR_VALUE)
        return [(int(kind[i]), int(level[i]), float(ms[i])) for i in range(n)]

    # -- results -------------------------------------------------------------------
    def _shape(self, name):
        if name in ("load", "net_delay", "impulse", "slew", "arrival", "required", "slack"):
            return (self.n_pins, 4)
        if name == "arc_delay":
            return (self.n_arcs, 4)
        if name in ("lse_arrival", "adjoint"):
            return (self.n_pins, 2)
        if name in ("arc_weights", "d_arc", "d_arc_sum"):
            return (self.n_arcs, 2)
        if name in ("d_edge", "d_edge_sum"):
            return (self.n_members, 2)
        if name == "summary":
            return (3,)
        if name in ("d_res", "d_cap"):
            return (self.n_members, 2)
        if name == "d_root_cap":
            return (self.n_nets, 2)
        if name in ("d_slew", "d_xy", "xy"):
            return (self.n_pins, 2)
        if name == "d_len":
            return (self.n_members,)
        if name == "wire":
            return (8,)
        if name in ("mem_res", "mem_cap", "res0", "cap0"):
            return (self.n_members, 4)
        if name == "root_cap":
            return (self.n_nets, 4)
        if name in ("pi_arrival", "pi_slew"):
            return (self.n_pi, 4)
        if name == "ep_required":
            return (self.n_ep, 4)
        return (-1,)

    def get(self, name: str, corner: int = 0, stream=None) -> np.ndarray:
        out = np.empty(self._shape(name), dtype=np.float64)
        if out.size:
            check(lib().ws_get(self._h, corner, _lib.STATE_FIELDS[name], ptr(out), 0,
                               _stream_handle(stream)))
        return out

    def get_many(self, names, corner: int = 0) -> dict:
        """Several result arrays of one corner as numpy arrays in PINNED host
        memory: all device-to-host copies are queued on the current stream
        back to back (full copy-engine bandwidth, no pageable staging) and
        synchronised once.  The buffers come from torch's caching host
        allocator, so repeated calls reuse them."""
        import torch
        host = {}
        for n in names:
            src = self.tensor(n, corner)
            h = torch.empty(tuple(src.shape), dtype=torch.float64, pin_memory=True)
            if h.numel():
                h.copy_(src, non_blocking=True)
            host[n] = h
        torch.cuda.current_stream().synchronize()
        return {n: h.numpy() for n, h in host.items()}

    def set_state(self, corner: int = 0, stream=None, **arrays):
        """Overwrite result arrays of one corner (host numpy arrays)."""
        L = lib()
        for name, a in arrays.items():
            a = np.ascontiguousarray(a, dtype=np.float64)
            if a.size != int(np.prod(self._shape(name))):
                raise ValueError(f"{name}: expected shape {self._shape(name)}")
            if a.size:
                check(L.ws_set_state(self._h, corner, _lib.STATE_FIELDS[name], ptr(a), 0,
                                     _stream_handle(stream)))
                self.sync(stream)   # `a` may be a temporary; the copy must land first

    def sync(self, stream=None):
        try:
            import torch
            if torch.cuda.is_available():
                (stream or torch.cuda.current_stream()).synchronize()
        except ImportError:
            pass

    def _tensor(self, getter, field, corner, name):
        import torch
        dp = ctypes.c_void_p()
        n = ctypes.c_int64()
        check(getter(self._h, corner, field, ctypes.byref(dp), ctypes.byref(n)))
        shape = self._shape(name)
        if n.value == 0:
            return torch.zeros(shape, dtype=torch.float64, device="cuda")
        return torch.as_tensor(_CudaArray(dp.value, shape, self), device="cuda")

    def tensor(self, name: str, corner: int = 0):
        """Zero-copy torch view of a result array in HBM (valid while the
        DeviceDesign lives)."""
        return self._tensor(lib().ws_device_ptr, _lib.STATE_FIELDS[name], corner, name)

    def summary(self, corner: int = 0, stream=None):
        """(TNS, WNS, loss) of the corner's last pass."""
        out = np.zeros(3, dtype=np.float64)
        check(lib().ws_summary(self._h, corner, out.ctypes.data_as(_lib._c_f64p),
                               _stream_handle(stream)))
        return float(out[0]), float(out[1]), float(out[2])
