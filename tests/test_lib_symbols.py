"""The C-ABI library loads without a GPU and exports every symbol that
include/warpstar.h declares (no compute calls here)."""

import ctypes
import os
import re

from paper_2603_28381_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(REPO, "include", "warpstar.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ws_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_abi_version_and_error_path_without_gpu():
    L = _lib.lib()
    assert L.ws_abi_version() == 1
    # a null descriptor is rejected before any device work
    h = ctypes.c_void_p()
    rc = L.ws_create(None, 1, ctypes.byref(h))
    assert rc == _lib.WS_ERR_VALUE
    assert b"null" in L.ws_last_error()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    try:
        _lib.lib()
    except ImportError as e:
        assert "no CPU fallback" in str(e)
    else:
        raise AssertionError("expected ImportError")
