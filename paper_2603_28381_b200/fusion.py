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


# ---------------------------------------------------------------------------
# makespan model (fusion.py:163-265): the reference's two-lane schedule over
# per-kernel costs.  Here the costs can be MEASURED on the device
# (measured_kernel_costs), which validates the model against the real
# two-stream run (makespan_report).

@dataclass
class ScheduleResult:
    records: list
    makespan: float
    overlap_fraction: float
    sta_finish: float
    grad_cycles: float
    overlapped_grad_cycles: float

    def _times(self):
        got = getattr(self, "_times_cache", None)
        if got is None:
            got = {r["id"]: (r["start"], r["finish"]) for r in self.records}
            self._times_cache = got
        return got

    def start(self, kid):
        return self._times()[kid][0]

    def finish(self, kid):
        return self._times()[kid][1]


def _result(graph: KernelGraph, times: dict) -> ScheduleResult:
    records, sta_fin = [], 0.0
    for kid in graph.sta_order + graph.grad_order:
        k = graph.kernels[kid]
        s, f = times[kid]
        records.append({"id": kid, "stream": k.stream, "kind": k.kind, "level": k.level,
                        "start": s, "finish": f})
        if k.stream == STA_STREAM:
            sta_fin = max(sta_fin, f)
    grad = sum(r["finish"] - r["start"] for r in records if r["stream"] == GRAD_STREAM)
    over = sum(max(0.0, min(r["finish"], sta_fin) - r["start"]) for r in records
               if r["stream"] == GRAD_STREAM)
    return ScheduleResult(records=records, makespan=max((f for _, f in times.values()), default=0.0),
                          overlap_fraction=over / grad if grad > 0 else 0.0, sta_finish=sta_fin,
                          grad_cycles=grad, overlapped_grad_cycles=over)


def schedule_sequential(graph: KernelGraph) -> ScheduleResult:
    """One lane: the sta stream's kernels, then the grad stream's."""
    times, t = {}, 0.0
    for kid in graph.sta_order + graph.grad_order:
        c = graph.kernels[kid].cost
        times[kid] = (t, t + c)
        t += c
    return _result(graph, times)


def schedule_fused(graph: KernelGraph, contention: float = 1.0) -> ScheduleResult:
    """Two lanes: the sta lane never waits; a grad kernel starts when its lane
    is free and its event sources finished, at `contention` x cost while the
    sta lane is still busy."""
    times, t = {}, 0.0
    for kid in graph.sta_order:
        c = graph.kernels[kid].cost
        times[kid] = (t, t + c)
        t += c
    sta_total, t = t, 0.0
    for kid in graph.grad_order:
        start = max([t] + [times[d][1] for d in graph.cross_deps(kid)])
        c = graph.kernels[kid].cost * (contention if start < sta_total else 1.0)
        times[kid] = (start, start + c)
        t = start + c
    return _result(graph, times)


def check_schedule(graph: KernelGraph, result: ScheduleResult) -> list:
    """Stream order, event edges, makespan = last finish."""
    problems = []
    for order in (graph.sta_order, graph.grad_order):
        for a, b in zip(order, order[1:]):
            if result.start(b) < result.finish(a):
                problems.append(f"stream order violated: {b} starts before {a} ends")
    for e in graph.edges:
        if result.start(e.dst) < result.finish(e.src):
            problems.append(f"event violated: {e.dst} starts before {e.src} ends")
    last = max((r["finish"] for r in result.records), default=0.0)
    if result.makespan != last:
        problems.append("makespan is not the last finish")
    return problems


KIND_NAMES = {0: "net_rc", 1: "cell_delay_at", 2: "slack_bwd", 3: "lse_fwd", 4: "grad_bwd"}


def measured_kernel_costs(dev, n_levels: int, gamma: float | None = None, loss: str = "hinge",
                          repeats: int = 5) -> dict:
    """(kind, level) -> ms measured on the device: RUN_TIMED sequential passes
    (one CUDA event after every launch; median of `repeats`).  The RC of all
    levels is one streaming launch, charged to net_rc:0; launches outside the
    graph (free pins, adjoint finish, summary) are folded into the
    neighbouring kernel of the same stream."""
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


def makespan_report(design, schedule=None, cfg: "FusionConfig | None" = None, repeats: int = 5) -> dict:
    """The reference's makespan model (schedule_sequential / schedule_fused)
    on MEASURED kernel costs, next to the measured sequential, two-stream and
    fused (interleaved) passes of the same design.

    Events between launches serialise the programmatic-dependent-launch
    overlap of the untimed pass, so the raw per-launch deltas are calibrated
    to the measured sequential pass (same proportions, same total).  The
    model's two-lane prediction is then compared with the measured two-stream
    pass, and the contention factor that reproduces it is fitted (the
    reference's ``contention`` knob, fusion.py:227-249)."""
    from .diff import _flat_of
    import torch
    cfg = cfg or FusionConfig()
    flat = _flat_of(design, schedule)
    gamma = cfg.gamma if cfg.gamma is not None else default_gamma(flat.clock_period)
    dev = device_of(flat)
    raw_costs = measured_kernel_costs(dev, flat.n_levels, gamma, cfg.loss, repeats)

    def measure(flags):
        ts = []
        for i in range(repeats + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev.run(flags, gamma=gamma, loss=cfg.loss, granularity=cfg.granularity)
            e1.record()
            e1.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1))
        return sorted(ts)[len(ts) // 2]

    base = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
    seq_ms = measure(base)
    two_ms = measure(base | _lib.RUN_TWO_STREAM)
    fused_ms = measure(base | _lib.RUN_FUSED)
    total = sum(raw_costs.values()) or 1.0
    costs = {k: v * seq_ms / total for k, v in raw_costs.items()}
    g = build_kernel_graph(flat.n_levels, costs, cfg.granularity)
    seq, fus = schedule_sequential(g), schedule_fused(g, 1.0)
    lo, hi = 1.0, 8.0                       # contention reproducing the two-stream run
    if schedule_fused(g, hi).makespan < two_ms:
        fit = None
    elif fus.makespan >= two_ms:
        fit = 1.0
    else:
        for _ in range(50):
            mid = 0.5 * (lo + hi)
            lo, hi = (mid, hi) if schedule_fused(g, mid).makespan < two_ms else (lo, mid)
        fit = 0.5 * (lo + hi)
    return {"raw_event_sum_ms": total, "model_sequential_ms": seq.makespan,
            "model_fused_ms": fus.makespan, "model_overlap_fraction": fus.overlap_fraction,
            "measured_sequential_ms": seq_ms, "measured_two_stream_ms": two_ms,
            "measured_interleaved_ms": fused_ms, "fitted_contention": fit,
            "problems": check_schedule(g, fus) + check_schedule(g, seq)}


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
