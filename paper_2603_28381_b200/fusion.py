"""Operation fusion on CUDA streams (drop-in for stasim/fusion.py:38-160, 287-450).

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

``PipelineRun`` is the kernel-by-kernel form of the same graph
(fusion.py:287-333): ``execute(kernel, deps)`` refuses, with
``FusionError``, a kernel whose dependencies have not run, and otherwise
launches exactly that kernel on the device (ws_run_kernel).
``execute_graph`` drives every kernel of ``build_kernel_graph`` through it.

The reference's two-lane makespan *simulator* (fusion.py:163-265) is not part
of this package: scripts/makespan_c3.py feeds the per-kernel costs measured
here (``measured_kernel_costs``) to the reference's own
``schedule_sequential`` / ``schedule_fused``.
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

    def is_acyclic(self) -> bool:
        """Kahn over stream orders + event edges (fusion.py KernelGraph)."""
        succ = {k: [] for k in self.kernels}
        indeg = {k: 0 for k in self.kernels}
        for order in (self.sta_order, self.grad_order):
            for a, b in zip(order, order[1:]):
                succ[a].append(b)
                indeg[b] += 1
        for e in self.edges:
            succ[e.src].append(e.dst)
            indeg[e.dst] += 1
        ready = [k for k, d in indeg.items() if d == 0]
        seen = 0
        while ready:
            k = ready.pop()
            seen += 1
            for n in succ[k]:
                indeg[n] -= 1
                if indeg[n] == 0:
                    ready.append(n)
        return seen == len(self.kernels)


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


KIND_NAMES = {0: "net_rc", 1: "cell_delay_at", 2: "slack_bwd", 3: "lse_fwd", 4: "grad_bwd"}


def measured_kernel_costs(dev, n_levels: int, gamma: float | None = None, loss: str = "hinge",
                          repeats: int = 5) -> dict:
    """(kind, level) -> ms measured on the device: RUN_TIMED sequential passes
    (one CUDA event after every launch; median of `repeats`).  The RC of all
    levels is one streaming launch, charged to net_rc:0; launches outside the
    graph (free pins, adjoint finish, summary) are folded into the
    neighbouring kernel of the same stream.  The makespan model that consumes
    these costs is the reference's own (scripts/makespan_ref.py)."""
    import statistics
    flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_TIMED
    runs = []
    for _ in range(repeats + 1):
        dev.run(flags, gamma=gamma, loss=loss)
        runs.append(dev.kernel_times())
    runs = runs[1:]                        # first run warms up
    costs = {(k, li): 0.0 for li in range(n_levels) for k in KIND_NAMES.values()}
    for i, (kind, level, _) in enumerate(runs[0]):
        ms = statistics.median(r[i][2] for r in runs)
        if kind in KIND_NAMES:
            costs[(KIND_NAMES[kind], level)] += ms
        elif i > 0:                        # fold "other" into the previous kernel
            pk, pl, _ = runs[0][i - 1]
            if pk in KIND_NAMES:
                costs[(KIND_NAMES[pk], pl)] += ms
    return costs


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


# ---------------------------------------------------------------------------
# kernel-by-kernel execution with the dependency discipline (fusion.py:287-333)

KIND_IDS = {"net_rc": 0, "cell_delay_at": 1, "slack_bwd": 2, "lse_fwd": 3, "grad_bwd": 4}


class PipelineRun:
    """One design's pipeline, one graph kernel at a time on the device.

    ``execute(kernel, deps)`` raises ``FusionError`` when any dependency has
    not executed yet (the reference's _PipelineRun.execute), else launches
    the kernel (ws_run_kernel: the same device functions as ws_run) and marks
    it done.  ``finalize()`` adds the pins finished after the level loop and
    the TNS / WNS / loss, and returns (TimingState, GradientState)."""

    def __init__(self, design, cfg: "FusionConfig | None" = None, schedule=None):
        from .diff import _flat_of
        self.cfg = cfg or FusionConfig()
        self.flat = _flat_of(design, schedule)
        self.gamma = self.cfg.gamma if self.cfg.gamma is not None else default_gamma(self.flat.clock_period)
        LseConfig(self.gamma)
        self.dev = device_of(self.flat)
        self.done = set()

    def _launch(self, kind_id, level):
        from ._lib import LOSS_KINDS, check, lib
        from .engine import _stream_handle
        if self.cfg.loss not in LOSS_KINDS:
            raise ValueError(f"unknown loss kind {self.cfg.loss!r}")
        check(lib().ws_run_kernel(self.dev._h, 0, int(kind_id), int(level), float(self.gamma),
                                  LOSS_KINDS[self.cfg.loss], int(self.cfg.reduce_width),
                                  _stream_handle(None)))

    def execute(self, kernel: Kernel, deps: list):
        missing = [d for d in deps if d not in self.done]
        if missing:
            raise FusionError(f"kernel {kernel.id} ran before its dependencies {missing}")
        if kernel.kind not in KIND_IDS:
            raise ValueError(f"unknown kernel kind {kernel.kind!r}")
        self._launch(KIND_IDS[kernel.kind], kernel.level)
        self.done.add(kernel.id)

    def finalize(self):
        self._launch(5, 0)
        st = TimingState.from_device(self.dev, 0, n_levels=self.flat.n_levels)
        gs = GradientState.from_device(self.dev, 0, self.gamma, self.cfg.loss, flat=self.flat)
        return st, gs


def execute_graph(design, schedule=None, cfg: FusionConfig | None = None):
    """Every kernel of ``build_kernel_graph`` through ``PipelineRun`` in a
    dependency-respecting order (stream predecessors and event sources
    first): bitwise the sequential pass."""
    cfg = cfg or FusionConfig()
    run = PipelineRun(design, cfg, schedule)
    g = build_kernel_graph(run.flat.n_levels, None, cfg.granularity)
    pred = {}
    for order in (g.sta_order, g.grad_order):
        for a, b in zip(order, order[1:]):
            pred[b] = a
    pending = [list(g.sta_order), list(g.grad_order)]
    while pending[0] or pending[1]:
        progressed = False
        for lane in pending:
            while lane:
                kid = lane[0]
                deps = ([pred[kid]] if kid in pred else []) + g.cross_deps(kid)
                if any(d not in run.done for d in deps):
                    break
                run.execute(g.kernels[kid], deps)
                lane.pop(0)
                progressed = True
        if not progressed:
            raise FusionError("kernel graph has no runnable kernel (cyclic dependencies)")
    return run.finalize()
