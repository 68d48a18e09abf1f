"""Operation fusion on CUDA streams (drop-in for stasim/fusion.py:38-160, 421-450).

The reference models two "streams" with Python threads and events
(fusion.py:383-407) and reports a *simulated* makespan.  Here the streams are
real CUDA streams inside one ``ws_run`` call:

* ``mode="threads"`` / ``"streams"`` (WS_RUN_TWO_STREAM): stream S runs RC, the
  forward levels and the backward levels; stream G runs the LSE levels and the
  gradient levels.  After the last forward level of each granularity-g group S
  records an event that gates that group's LSE work on G, and G's gradient
  backward additionally waits on S's backward of the top level — exactly the
  cross edges of ``build_kernel_graph`` (fusion.py:151-157).  G overlaps the
  forward levels still running on S.
* ``mode="interleaved"`` (WS_RUN_FUSED): one stream, forward+LSE and
  backward+gradient fused into single per-level kernels.

Both run the same device functions as ``execute_sequential`` so all outputs
are bitwise identical (fusion.py:6-9); the returned ``FusedResult`` carries
CUDA-event-measured times instead of simulated cycles.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib
from .diff import GradientState, LseConfig, default_gamma
from .flatten import device_of
from .sta import TimingState

STA_STREAM = "sta"
GRAD_STREAM = "grad"
STA_KINDS = ("net_rc", "cell_delay_at", "slack_bwd")
GRAD_KINDS = ("lse_fwd", "grad_bwd")
MODES = ("interleaved", "threads", "streams")


class FusionError(RuntimeError):
    """Dependency discipline violated."""


@dataclass
class Kernel:
    id: str
    stream: str
    kind: str
    level: int
    cost: float

    def __post_init__(self):
        if self.cost < 0:
            raise ValueError("kernel cost must be non-negative")
        if (self.kind in STA_KINDS) != (self.stream == STA_STREAM):
            raise ValueError(f"kind {self.kind!r} does not belong to stream {self.stream!r}")


@dataclass
class EventEdge:
    src: str
    dst: str


@dataclass
class FusionConfig:
    granularity: int = 10
    contention: float = 1.0
    mode: str = "interleaved"
    gamma: float | None = None
    loss: str = "hinge"
    reduce_width: int = 8

    def __post_init__(self):
        if self.granularity < 1:
            raise ValueError("granularity must be >= 1")
        if self.contention < 1.0:
            raise ValueError("contention factor must be >= 1.0")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")


@dataclass
class KernelGraph:
    kernels: dict
    edges: list
    sta_order: list
    grad_order: list
    event_granularity: int
    n_levels: int

    def cross_deps(self, kid: str) -> list:
        return [e.src for e in self.edges if e.dst == kid]


def build_kernel_graph(schedule, costs=None, granularity: int = 10) -> KernelGraph:
    """The stream/event structure the two-stream executor launches
    (fusion.py:113-160).  ``costs`` maps (kind, level) -> cost; optional here
    (measured timings replace the reference's simulated cycles)."""
    n_levels = schedule if isinstance(schedule, int) else schedule.n_levels
    if granularity < 1:
        raise ValueError("granularity must be >= 1")

    def kernel(kind, li):
        stream = STA_STREAM if kind in STA_KINDS else GRAD_STREAM
        cost = 0.0
        if costs is not None:
            try:
                cost = float(costs[(kind, li)])
            except KeyError:
                raise ValueError(f"missing cost entry for ({kind!r}, level {li})")
        return Kernel(id=f"{kind}:{li}", stream=stream, kind=kind, level=li, cost=cost)

    kernels, sta_order, grad_order = {}, [], []
    for li in range(n_levels):
        for kind in ("net_rc", "cell_delay_at"):
            k = kernel(kind, li)
            kernels[k.id] = k
            sta_order.append(k.id)
    for li in range(n_levels - 1, -1, -1):
        k = kernel("slack_bwd", li)
        kernels[k.id] = k
        sta_order.append(k.id)
    for li in range(n_levels):
        k = kernel("lse_fwd", li)
        kernels[k.id] = k
        grad_order.append(k.id)
    for li in range(n_levels - 1, -1, -1):
        k = kernel("grad_bwd", li)
        kernels[k.id] = k
        grad_order.append(k.id)
    edges = []
    for g0 in range(0, n_levels, granularity):
        g1 = min(g0 + granularity, n_levels) - 1
        edges.append(EventEdge(f"cell_delay_at:{g1}", f"lse_fwd:{g0}"))
    if n_levels:
        edges.append(EventEdge(f"slack_bwd:{n_levels - 1}", f"grad_bwd:{n_levels - 1}"))
    return KernelGraph(kernels=kernels, edges=edges, sta_order=sta_order, grad_order=grad_order,
                       event_granularity=granularity, n_levels=n_levels)


@dataclass
class FusedResult:
    """Measured execution record of one pipeline run."""

    mode: str
    makespan_ms: float
    n_kernels: int
    graph: KernelGraph


def _run(design, schedule, cfg: FusionConfig, flags: int, mode: str):
    import torch
    from .diff import _flat_of
    flat = _flat_of(design, schedule)
    cfg = cfg or FusionConfig()
    gamma = cfg.gamma if cfg.gamma is not None else default_gamma(flat.clock_period)
    LseConfig(gamma)
    dev = device_of(flat)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    dev.run(flags, gamma=gamma, loss=cfg.loss, reduce_width=cfg.reduce_width,
            granularity=cfg.granularity)
    e1.record(s)
    e1.synchronize()
    st = TimingState.from_device(dev, 0, n_levels=flat.n_levels)
    gs = GradientState.from_device(dev, 0, gamma, cfg.loss, flat=flat)
    res = FusedResult(mode=mode, makespan_ms=float(e0.elapsed_time(e1)),
                      n_kernels=dev.last_launch_count(),
                      graph=build_kernel_graph(flat.n_levels, None, cfg.granularity))
    return st, gs, res


def execute_sequential(design, schedule=None, geometry=None, cfg: FusionConfig | None = None,
                       cost_model=None):
    """Every STA kernel, then every gradient kernel, on one stream
    (fusion.py:421-432)."""
    return _run(design, schedule, cfg, _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD,
                "sequential")


def execute_fused(design, schedule=None, geometry=None, cfg: FusionConfig | None = None,
                  cost_model=None):
    """Fused pipeline (fusion.py:435-450): two CUDA streams with event gating
    ("threads"/"streams"), or single-stream per-level kernel fusion
    ("interleaved")."""
    cfg = cfg or FusionConfig()
    base = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
    if cfg.mode == "interleaved":
        return _run(design, schedule, cfg, base | _lib.RUN_FUSED, "interleaved")
    return _run(design, schedule, cfg, base | _lib.RUN_TWO_STREAM, "streams")
