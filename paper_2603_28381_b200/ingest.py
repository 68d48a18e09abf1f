"""On-disk ingest format for a design.

The reference reads designs as canonical JSON (netlist.py:399-559) and
re-flattens them on every run; at C3 generate + flatten costs ~98 s.  Here a
design is stored as the flat arrays the device build consumes (``RawDesign``,
the reference's own orders: nets, members, arcs, LUT pool, seeds) in one
uncompressed ``.npz``, together with a sha256 content hash over the arrays
in a fixed order (the analogue of reports.py:30-36 ``design_hash``, which
hashes the canonical JSON).  ``load_raw`` verifies the hash and the array
shapes before anything reaches the device; ``DeviceDesign`` ingests the
result directly (flatten + levelize + CSR on the device, ~0.1 s at C3).
"""

from __future__ import annotations

import hashlib
import os

import numpy as np

from .netlist import RawDesign

FORMAT = "warpstar-raw"
VERSION = 1
ARRAYS = ("net_root", "net_mptr", "mem_pin", "mem_parent_pin", "mem_res", "mem_cap", "root_cap",
          "arc_from", "arc_to", "arc_dlut", "arc_slut", "lut_s_ptr", "lut_l_ptr", "lut_t_ptr",
          "lut_s_flat", "lut_l_flat", "lut_t_flat", "pi_pin", "pi_arrival", "pi_slew", "ep_pin",
          "ep_required")


class DesignFileError(ValueError):
    """Malformed or corrupted design file (the reference raises
    DesignFormatError for malformed documents, netlist.py:48-53)."""


def raw_hash(raw: RawDesign) -> str:
    """sha256 over (n_pins, clock_period, every array's dtype, shape and
    bytes) in ARRAYS order, after normalisation to the C-ABI dtypes."""
    r = raw.normalized()
    h = hashlib.sha256()
    h.update(f"{FORMAT}/{VERSION}/{int(r.n_pins)}/{float(r.clock_period).hex()}".encode())
    for name in ARRAYS:
        a = np.ascontiguousarray(getattr(r, name))
        h.update(f"|{name}:{a.dtype.str}:{a.shape}|".encode())
        h.update(a.tobytes())
    return h.hexdigest()


def save_raw(path: str, raw: RawDesign) -> str:
    """Write ``raw`` to ``path`` (.npz); returns its content hash."""
    r = raw.normalized()
    digest = raw_hash(r)
    arrays = {name: getattr(r, name) for name in ARRAYS}
    tmp = path + ".tmp.npz"
    np.savez(tmp, _format=np.array(FORMAT), _version=np.array(VERSION),
             _n_pins=np.array(int(r.n_pins)), _clock_period=np.array(float(r.clock_period)),
             _hash=np.array(digest), **arrays)
    os.replace(tmp, path)
    return digest


def load_raw(path: str, verify: bool = True) -> RawDesign:
    """Read a design written by save_raw; with ``verify`` the content hash
    must match (DesignFileError otherwise)."""
    try:
        z = np.load(path, allow_pickle=False)
    except (OSError, ValueError) as e:
        raise DesignFileError(f"{path}: not a design file ({e})") from None
    with z:
        files = set(z.files)
        need = {"_format", "_version", "_n_pins", "_clock_period", "_hash", *ARRAYS}
        if not need <= files:
            raise DesignFileError(f"{path}: missing {sorted(need - files)}")
        if str(z["_format"]) != FORMAT or int(z["_version"]) != VERSION:
            raise DesignFileError(f"{path}: format {str(z['_format'])!r} v{int(z['_version'])}, "
                                  f"expected {FORMAT!r} v{VERSION}")
        raw = RawDesign(n_pins=int(z["_n_pins"]), clock_period=float(z["_clock_period"]),
                        **{name: z[name] for name in ARRAYS}).normalized()
        stored = str(z["_hash"])
    if verify and raw_hash(raw) != stored:
        raise DesignFileError(f"{path}: content hash mismatch (corrupted or edited file)")
    raw.meta["hash"] = stored
    raw.meta["source"] = os.path.abspath(path)
    return raw
