"""RC kernel variants — the CTE scheme (the paper's Algorithm 2 ablation,
WS_RC_SCHEME=cte) and the pin-order streaming kernel (WS_RC_SCHEME=pin):
bitwise the same RC outputs and pass as the default member-order streaming
RC kernel on star designs (heavy tail up to 508 members) and on RC-tree
designs.  Likewise the star-net root loads folded inside the member blocks
(WS_RC_ROOTS=fold, the corner-batch default; nets that run past a block's
end read their tail from global) against the separate net blocks."""

import os

import numpy as np
import pytest

import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G

pytestmark = pytest.mark.gpu
FIELDS = ("load", "net_delay", "impulse", "arrival", "slew", "required", "slack", "adjoint")


def _run(raw, scheme, var="WS_RC_SCHEME"):
    old = os.environ.get(var)
    os.environ[var] = scheme
    try:
        dev = ws.DeviceDesign(raw)
    finally:
        if old is None:
            del os.environ[var]
        else:
            os.environ[var] = old
    dev.run(_lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED)
    out = {f: dev.get(f) for f in FIELDS}
    dev.close()
    return out


@pytest.mark.parametrize("cfg", ["c1", "c1tree", "c2"])
@pytest.mark.parametrize("scheme", ["cte", "pin"])
def test_rc_schemes_bitwise(cfg, scheme):
    raw = G.generate_raw({"c1": G.config_c1(), "c1tree": G.config_c1("random_tree"),
                          "c2": G.config_c2()}[cfg])
    a, b = _run(raw, "flat"), _run(raw, scheme)
    for f in FIELDS:
        assert np.array_equal(a[f], b[f]), f


@pytest.mark.parametrize("cfg", ["c1", "c1tree", "c2"])
def test_rc_root_fold_bitwise(cfg):
    raw = G.generate_raw({"c1": G.config_c1(), "c1tree": G.config_c1("random_tree"),
                          "c2": G.config_c2()}[cfg])
    a, b = _run(raw, "net", "WS_RC_ROOTS"), _run(raw, "fold", "WS_RC_ROOTS")
    for f in FIELDS:
        assert np.array_equal(a[f], b[f]), f
