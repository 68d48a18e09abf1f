"""Host-side API logic that needs no device: config validation, the LSE
helpers' known answers (test_diff.py:19-66) and the kernel-graph structure
the two-stream executor launches (test_fusion.py:38-82)."""

import math

import numpy as np
import pytest

from paper_2603_28381_b200 import (FusionConfig, Kernel, LseConfig, build_kernel_graph,
                                   default_gamma, get_backend, available_backends, backend_name,
                                   lse, lse_grad)


def test_lse_kats():
    cfg = LseConfig(0.37)
    for x in (-5.0, 0.0, 1e-9, 3.25e4):
        assert lse([x], cfg) == x
    assert lse([0.0, 0.0], LseConfig(1.0)) == pytest.approx(math.log(2.0), rel=1e-15)
    assert lse([1.0, 2.0, 3.0], LseConfig(0.5)) == pytest.approx(3.0714658142499496, rel=1e-14)
    w = lse_grad([7.0] * 4, LseConfig(0.3))
    assert np.array_equal(w, np.full(4, 0.25))
    with pytest.raises(ValueError):
        LseConfig(0.0)
    with pytest.raises(ValueError):
        LseConfig(float("inf"))
    with pytest.raises(ValueError):
        lse([], LseConfig(1.0))
    assert default_gamma(2e-9) == pytest.approx(2e-11, rel=1e-15)


def test_lse_bounds():
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(1, 12))
        xs = rng.normal(scale=10.0 ** rng.integers(-9, 2), size=n)
        g = float(10.0 ** rng.uniform(-12, 0))
        v = lse(xs, LseConfig(g))
        assert xs.max() <= v <= xs.max() + g * math.log(n)


def test_graph_structure():
    g = build_kernel_graph(3, None, granularity=1)
    assert g.sta_order == ["net_rc:0", "cell_delay_at:0", "net_rc:1", "cell_delay_at:1",
                           "net_rc:2", "cell_delay_at:2", "slack_bwd:2", "slack_bwd:1",
                           "slack_bwd:0"]
    assert g.grad_order == ["lse_fwd:0", "lse_fwd:1", "lse_fwd:2", "grad_bwd:2", "grad_bwd:1",
                            "grad_bwd:0"]
    g10 = build_kernel_graph(30, None, granularity=10)
    cross = sorted((e.src, e.dst) for e in g10.edges if e.src.startswith("cell_delay_at"))
    assert cross == [("cell_delay_at:19", "lse_fwd:10"), ("cell_delay_at:29", "lse_fwd:20"),
                     ("cell_delay_at:9", "lse_fwd:0")]
    assert any(e.src == "slack_bwd:29" and e.dst == "grad_bwd:29" for e in g10.edges)
    with pytest.raises(ValueError, match="missing cost entry"):
        build_kernel_graph(2, {("net_rc", 0): 1.0}, granularity=1)


def test_configs_validate():
    with pytest.raises(ValueError):
        FusionConfig(granularity=0)
    with pytest.raises(ValueError):
        FusionConfig(contention=0.5)
    with pytest.raises(ValueError):
        FusionConfig(mode="fibers")
    with pytest.raises(ValueError):
        Kernel("x", "grad", "net_rc", 0, 1.0)
    with pytest.raises(ValueError):
        Kernel("x", "sta", "net_rc", 0, -1.0)


def test_backend_registry():
    assert backend_name() == "cuda"
    assert set(available_backends()) == {"cuda"}
    with pytest.raises(ValueError):
        get_backend("gpu")
    with pytest.raises(ValueError):
        get_backend("python")
