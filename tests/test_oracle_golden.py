"""Pin the CPU oracle (oracle/sta_oracle.c) to the reference's own outputs.

The golden fixtures were produced by running the reference (stasim, compiled
backend) on the reference's test designs and generator designs
(tests/golden/make_golden.py).  The oracle must reproduce the hard pass, the
FlatDesign index arrays, the level schedule, the CSR and TNS/WNS bit for bit,
and the gradients to within libm-vs-numpy exp/log ulps.
"""

import numpy as np
import pytest

from golden_util import G_FIELDS, ST_FIELDS, grad_close, load, max_rel, names, raw_ns
from oracle import oracle as O

CASES = names()


@pytest.mark.parametrize("name", CASES)
def test_oracle_flatten_bit_exact(name):
    g = load(name)
    flat = O.flatten_raw(raw_ns(g))
    for k, v in g.items():
        if k.startswith("flat_"):
            assert np.array_equal(getattr(flat, k[5:]), v), k
    lv = np.concatenate(flat.levels) if flat.levels else np.zeros(0, np.int64)
    assert np.array_equal(lv, g["levels_nets"])
    assert np.array_equal(np.cumsum([0] + [len(x) for x in flat.levels]), g["levels_ptr"])
    assert np.array_equal(flat.level_of, g["level_of"])
    assert np.array_equal(flat.pin_list, g["csr_pin_list"])
    assert np.array_equal(flat.net_index, g["csr_net_index"])


@pytest.mark.parametrize("name", CASES)
def test_oracle_engine_bit_exact(name):
    g = load(name)
    flat = O.flatten_raw(raw_ns(g))
    st = O.run_engine(flat)
    for f in ST_FIELDS:
        assert np.array_equal(getattr(st, f), g["st_" + f]), f
    assert O.tns(st, flat) == g["tns"]
    assert O.wns(st, flat) == g["wns"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_gradients(name):
    g = load(name)
    flat = O.flatten_raw(raw_ns(g))
    st = O.run_engine(flat)
    gs = O.timing_gradients(flat, st, gamma=float(g["gamma"]))
    for f in G_FIELDS:
        assert grad_close(getattr(gs, f), g["g_" + f], rtol=1e-12), (f, max_rel(getattr(gs, f), g["g_" + f]))
    assert gs.loss == pytest.approx(float(g["g_loss"]), rel=1e-13)
    if "gs_loss" in g:
        gp = O.timing_gradients(flat, st, gamma=float(g["gamma"]), loss="softplus")
        for f in G_FIELDS:
            assert grad_close(getattr(gp, f), g["gs_" + f], rtol=1e-12), f
        assert gp.loss == pytest.approx(float(g["gs_loss"]), rel=1e-13)


def test_oracle_lut_kats():
    # test_sta.py:187-201 on the oracle's interpolation
    from types import SimpleNamespace
    f = SimpleNamespace(lut_s_ptr=np.array([0, 2]), lut_l_ptr=np.array([0, 2]),
                        lut_t_ptr=np.array([0, 4]), lut_s_flat=np.array([0.0, 1.0]),
                        lut_l_flat=np.array([0.0, 1.0]), lut_t_flat=np.array([0.0, 1.0, 2.0, 3.0]))
    for s, l, want in ((0, 0, 0.0), (0, 1, 1.0), (1, 0, 2.0), (1, 1, 3.0), (0.5, 0.5, 1.5),
                       (5.0, 0.0, 2.0), (-5.0, 1.0, 1.0), (1.0, 99.0, 3.0)):
        assert O.interpolate(f, 0, s, l) == want
