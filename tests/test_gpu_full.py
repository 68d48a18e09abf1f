"""Full-size parity: BASELINE configs C1 / C2 / C3 on the device vs the CPU
oracle (oracle/sta_oracle.c, itself pinned to the reference by
test_oracle_golden.py) on identical generator inputs, plus the multi-corner
batch and the placement-loop perturbation.

C2 = 995,808 pins (heavy-tail fanout, max 508), C3 = 2,490,236 pins.
"""

import numpy as np
import pytest

from golden_util import G_FIELDS, ST_FIELDS, grad_close, max_rel
import paper_2603_28381_b200 as ws
from paper_2603_28381_b200 import _lib, generator as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu

FLAT_FIELDS = ("net_ptr", "net_root", "root_kind", "mem_pin", "mem_parent_loc", "mem_net",
               "mem_local", "net_in_ptr", "net_in_arc", "mem_out_ptr", "mem_out_arc", "net_m",
               "net_a", "net_o", "member_of_pin", "root_net_of_pin", "is_endpoint", "arc_dlut",
               "arc_slut")

_cache = {}


def setup(cfg_name):
    if cfg_name not in _cache:
        cfg = {"c1": G.config_c1(), "c1tree": G.config_c1("random_tree"),
               "c2": G.config_c2(), "c3": G.config_c3()}[cfg_name]
        raw = G.generate_raw(cfg)
        ofl = O.flatten_raw(raw)
        _cache[cfg_name] = (raw, ofl)
    return _cache[cfg_name]


def check_flat(dev, ofl):
    for f in FLAT_FIELDS:
        assert np.array_equal(dev.topology(f), getattr(ofl, f)), f
    lv = dev.levels()
    assert len(lv) == ofl.n_levels
    for a, b in zip(lv, ofl.levels):
        assert np.array_equal(a, b)
    assert np.array_equal(dev.topology("csr_pin_list"), ofl.pin_list)
    assert np.array_equal(dev.topology("csr_net_index"), ofl.net_index)


@pytest.mark.parametrize("cfg_name", ["c1", "c1tree", "c2", "c3"])
def test_full_size_parity(cfg_name):
    raw, ofl = setup(cfg_name)
    dev = ws.DeviceDesign(raw)
    check_flat(dev, ofl)
    ost = O.run_engine(ofl)
    flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED
    gamma = dev.run(flags)
    for f in ST_FIELDS:
        got = dev.get(f)
        assert np.array_equal(got, getattr(ost, f)), (f, max_rel(got, getattr(ost, f)))
    tns, wns, loss = dev.summary()
    assert tns == O.tns(ost, ofl)
    assert wns == O.wns(ost, ofl)
    og = O.timing_gradients(ofl, ost, gamma=gamma)
    for f in G_FIELDS:
        assert grad_close(dev.get(f), getattr(og, f)), (f, max_rel(dev.get(f), getattr(og, f)))
    assert loss == pytest.approx(og.loss, rel=1e-9)
    # two-stream and persistent modes are bitwise identical to the fused single stream
    ref = {f: dev.get(f) for f in ST_FIELDS + G_FIELDS}
    for extra in (_lib.RUN_TWO_STREAM, _lib.RUN_PERSISTENT):
        dev.run(_lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | extra)
        for f in ST_FIELDS + G_FIELDS:
            assert np.array_equal(dev.get(f), ref[f]), (extra, f)
        assert dev.summary()[2] == loss
    dev.close()


def corner_values(raw, k):
    """corner k scales res by 0.85+0.02k, caps and LUT
    tables by 0.90+0.0125k."""
    fr, fc = 0.85 + 0.02 * k, 0.90 + 0.0125 * k
    return dict(mem_res=raw.mem_res * fr, mem_cap=raw.mem_cap * fc, root_cap=raw.root_cap * fc,
                lut_t_flat=raw.lut_t_flat * fc)


@pytest.mark.parametrize("cfg_name", ["c1", "c3"])
def test_corner_batch_matches_single_and_oracle(cfg_name):
    raw, ofl = setup(cfg_name)
    nc = 4
    dev = ws.DeviceDesign(raw, n_corners=nc)
    for k in range(nc):
        dev.set_values(k, **corner_values(raw, k))
    flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED
    dev.run(flags, corner=0, n_corners=nc)
    batch = [{f: dev.get(f, k) for f in ST_FIELDS + G_FIELDS} for k in range(nc)]
    sums = [dev.summary(k) for k in range(nc)]
    for k in range(nc):
        dev.run(flags, corner=k, n_corners=1)
        for f in ST_FIELDS + G_FIELDS:
            assert np.array_equal(dev.get(f, k), batch[k][f]), (k, f)
        assert dev.summary(k) == sums[k]
    k = nc - 1
    import copy
    o2 = copy.copy(ofl)
    for name, v in corner_values(raw, k).items():
        setattr(o2, name, v.reshape(getattr(ofl, name).shape))
    ost = O.run_engine(o2)
    for f in ST_FIELDS:
        assert np.array_equal(batch[k][f], getattr(ost, f)), f
    dev.close()


def test_placement_perturbation_parity():
    raw, ofl = setup("c1")
    dev = ws.DeviceDesign(raw, n_corners=2)
    flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED
    for t in (0, 99, 199):
        dev.perturb(1, 0, seed=1000 + t, sigma=0.01)
        res = dev.value_tensor("mem_res", 1).cpu().numpy()
        fac = res / raw.mem_res
        assert np.all(fac >= 0.97 - 1e-12) and np.all(fac <= 1.03 + 1e-12)
        assert np.allclose(fac, fac[:, :1])          # one factor per member
        cap = dev.value_tensor("mem_cap", 1).cpu().numpy()
        rc = dev.value_tensor("root_cap", 1).cpu().numpy()
        dev.run(flags, corner=1)
        import copy
        o2 = copy.copy(ofl)
        o2.mem_res, o2.mem_cap, o2.root_cap = res, cap, rc
        ost = O.run_engine(o2)
        for f in ST_FIELDS:
            assert np.array_equal(dev.get(f, 1), getattr(ost, f)), (t, f)
        og = O.timing_gradients(o2, ost, gamma=0.01 * raw.clock_period)
        for f in G_FIELDS:
            assert grad_close(dev.get(f, 1), getattr(og, f)), (t, f)
    dev.close()


@pytest.mark.parametrize("cfg_name", ["c1tree", "c2"])
def test_softplus_loss_full_size(cfg_name):
    """Softplus endpoint loss (diff.py:192-212: max(v,0) + g log1p(exp(-|v|/g)),
    seed sigmoid(v/g)) at full size, custom gamma, all modes."""
    raw, ofl = setup(cfg_name)
    dev = ws.DeviceDesign(raw)
    ost = O.run_engine(ofl)
    gamma = 0.02 * ofl.clock_period
    og = O.timing_gradients(ofl, ost, gamma=gamma, loss="softplus")
    ref = None
    for extra in (_lib.RUN_FUSED, _lib.RUN_TWO_STREAM, _lib.RUN_PERSISTENT, 0):
        dev.run(_lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | extra, gamma=gamma, loss="softplus")
        got = {f: dev.get(f) for f in G_FIELDS}
        for f in G_FIELDS:
            assert grad_close(got[f], getattr(og, f)), (extra, f)
        assert dev.summary()[2] == pytest.approx(og.loss, rel=1e-9)
        if ref is None:
            ref = got
        else:
            for f in G_FIELDS:
                assert np.array_equal(got[f], ref[f]), (extra, f)
    dev.close()


@pytest.mark.parametrize("gran", [1, 7, 60])
def test_two_stream_granularity_bitwise(gran):
    """fusion.py:151-157 event granularity g: the two-stream pass equals the
    fused pass bitwise for any g (only the overlap changes)."""
    raw, ofl = setup("c1")
    dev = ws.DeviceDesign(raw)
    base = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
    dev.run(base | _lib.RUN_FUSED)
    ref = {f: dev.get(f) for f in ST_FIELDS + G_FIELDS}
    dev.run(base | _lib.RUN_TWO_STREAM, granularity=gran)
    for f in ST_FIELDS + G_FIELDS:
        assert np.array_equal(dev.get(f), ref[f]), (gran, f)
    dev.close()
