#!/usr/bin/env python
"""Benchmark: differentiable STA fwd+bwd pass on the 2.5M-pin netlist (C3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full differentiable STA pass over the synthetic superblue-shaped
C3 netlist (2,490,236 pins): init, RC, 60 forward levels with
the LSE smooth forward, endpoint hinge loss, 60 backward levels with the
gradient adjoint, slack, TNS/WNS — inputs resident in HBM.  Under torchrun
(N>1) every rank runs its own corner of the C5 corner set (corner k = rank,
weak scaling) and the ranks all-reduce WNS (MIN), TNS and loss (SUM) and the
gradients d_arc/d_edge (SUM) over NCCL each step.

value = whole-job ms per pass = max-over-ranks device time of K steps / (K*N).
``e2e`` is the same pass through the public API with the step's value inputs
(mem_res, mem_cap, root_cap) copied from pinned host memory and TNS/WNS/loss
read back every step.  ``--impl reference`` times the reference's own CPU
implementation (stasim run_engine + timing_gradients, from oracle/_ref) on
this host.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "ms per fwd+bwd STA pass on 2.5M-pin netlist; achieved HBM GB/s; corners/s @1-8 GPU"
L2_BYTES = 126 * 1024 * 1024


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def algorithmic_bytes(P, M, N, A, I, E):
    """BASELINE.md §3 / SURVEY.md §8(d): compulsory bytes of one fwd+bwd pass."""
    return 256 * P + 92 * M + 44 * N + 108 * A + 68 * I + 36 * E


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def corner_values(raw, k):
    """C5 corner k: res x(0.85+0.02k); caps, LUT tables x(0.90+0.0125k)."""
    fr, fc = 0.85 + 0.02 * k, 0.90 + 0.0125 * k
    return dict(mem_res=raw.mem_res * fr, mem_cap=raw.mem_cap * fc, root_cap=raw.root_cap * fc,
                lut_t_flat=raw.lut_t_flat * fc)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU reference (the --impl reference arm and the cpu_baseline object)

def reference_flat(raw):
    """The reference's FlatDesign for `raw`, assembled from the oracle's
    flatten (pinned bit-exact to the reference's flatten by
    tests/test_oracle_golden.py) — the reference's own flatten() would need
    ~100 s of Python object construction at C3."""
    from oracle import oracle as O
    of = O.flatten_raw(raw)
    # the pip-installed unmodified reference (baseline/_ref),
    # else the same sources built by oracle/build_ref.sh
    ref = next((d for d in (os.path.join(REPO, "baseline", "_ref"), os.path.join(REPO, "oracle", "_ref"))
                if os.path.isdir(os.path.join(d, "stasim"))), None)
    if ref is not None:
        sys.path.insert(0, ref)
        import stasim  # the unmodified reference
        from stasim.flatten import FlatDesign, LevelSchedule
        from stasim.backend import backend_name
        fields = {f: getattr(of, f) for f in FlatDesign.__dataclass_fields__
                  if f not in ("design", "schedule", "_level_cache")}
        flat = FlatDesign(design=None, schedule=LevelSchedule(of.levels, of.level_of), **fields)
        return flat, "reference", f"stasim {stasim.__version__} ({backend_name()} backend)"
    return of, "port", "oracle/sta_oracle.c (C restatement)"


def time_reference(raw, max_passes, budget_s):
    flat, kind, what = reference_flat(raw)
    if kind == "reference":
        from stasim.warp import run_engine
        from stasim.diff import timing_gradients

        def one():
            st = run_engine(flat)
            timing_gradients(flat, state=st)
    else:
        from oracle import oracle as O

        def one():
            st = O.run_engine(flat)
            O.timing_gradients(flat, st)
    t0 = time.perf_counter()
    one()                                   # warm-up (lazy level_view caches)
    warm = time.perf_counter() - t0
    n = int(max(1, min(max_passes, budget_s // max(warm, 1e-3))))
    times = []
    for _ in range(n):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    return {"ms": 1e3 * statistics.median(times), "passes": n, "kind": kind, "what": what,
            "times_ms": [round(1e3 * t, 1) for t in times]}


def corner_batch(raw, rank, world, flags, steps, dist=None, n_total=16):
    """C5: 16 corners of the C3 netlist sharded round-robin
    over the ranks (corner k -> rank k mod world, 16/world per GPU), all of a
    rank's corners in ONE ws_run (blockIdx.y = corner), then the batch
    objective's NCCL exchange: TNS / loss SUM, WNS MIN, d_arc / d_edge SUM
    (the gradient of sum_k loss_k).  Device time with CUDA events, max over
    ranks; corners/s is the whole job's."""
    import torch
    import paper_2603_28381_b200 as ws
    from paper_2603_28381_b200.corners import combine_local, reduce_batch
    mine = [k for k in range(n_total) if k % world == rank]
    nc = len(mine)
    dev = ws.DeviceDesign(raw, n_corners=nc)
    for i, k in enumerate(mine):
        dev.set_values(i, **corner_values(raw, k))
    stream = torch.cuda.current_stream()
    d_arc = [dev.tensor("d_arc", i) for i in range(nc)]
    d_edge = [dev.tensor("d_edge", i) for i in range(nc)]
    summ = [dev.tensor("summary", i) for i in range(nc)]
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")

    def step():
        dev.run(flags, corner=0, n_corners=nc, stream=stream)
        ga, ge = d_arc[0].clone(), d_edge[0].clone()
        for i in range(1, nc):
            ga += d_arc[i]
            ge += d_edge[i]
        sm = combine_local(summ)
        if dist is not None:
            reduce_batch(sm, ga, ge)
        return sm

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    if dist is not None:
        dist.barrier()
    for i in range(steps):
        flush.fill_(i)
        evs[i][0].record(stream)
        sm = step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    tot = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms = float(tot.item()) / steps
    out = {"workload": "C5: %d corners of the C3 netlist, corner k -> rank k mod N, a rank's "
                       "corners in one ws_run, NCCL TNS/loss SUM, WNS MIN, d_arc/d_edge SUM" % n_total,
           "corners_per_gpu": nc, "ms_per_batch": round(ms, 4),
           "corners_per_s": round(n_total / (ms * 1e-3), 2), "steps": steps,
           "batch_result": {"tns": float(sm[0]), "wns": float(sm[1]), "loss": float(sm[2])}}
    dev.close()
    return out


def candidate_batch(raw, rank, world, steps, dist=None, n_total=16, sigma_um=0.5):
    """Placement-candidate batch (north_star): 16 candidate
    placements of C3 (cells moved by N(0, sigma) with seed 2000 + c),
    candidate c on rank c mod N, a rank's candidates in ONE ws_run (wire RC ->
    batched pass -> position gradients per candidate), then the candidates'
    (TNS, WNS, loss) and dL/dxy all-gathered in candidate order (no
    reduction: candidates are alternatives).  Device time, max over ranks."""
    import torch
    import paper_2603_28381_b200 as ws
    from paper_2603_28381_b200 import placement as PL
    from paper_2603_28381_b200.corners import best_candidate, corners_of_rank, gather_candidates
    mine = corners_of_rank(n_total, rank, world)
    nc = len(mine)
    pl = PL.synthetic_placement(raw, seed=3)
    dev = ws.DeviceDesign(raw, n_corners=nc)
    timers = []
    for i, c in enumerate(mine):
        rng = np.random.default_rng(2000 + c)
        xy = pl.xy + sigma_um * rng.standard_normal(pl.cell_xy.shape)[pl.cell_of_pin]
        timers.append(PL.PlacementTimer(dev, PL.Placement(xy, pl.res0, pl.cap0, pl.wire, pl.cell_of_pin,
                                                          pl.cell_xy, pl.pin_offset), corner=i))
    flags = timers[0].flags
    stream = torch.cuda.current_stream()
    summ = [dev.tensor("summary", i) for i in range(nc)]
    dxy = [dev.tensor("d_xy", i) for i in range(nc)]

    def step():
        dev.run(flags, corner=0, n_corners=nc, gamma=timers[0].gamma, stream=stream)
        s = torch.stack(summ)
        if dist is not None:
            return gather_candidates(s, torch.stack(dxy))
        return s, torch.stack(dxy)

    for _ in range(5):                       # first calls in a process are slower
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    if dist is not None:
        dist.barrier()
    for i in range(steps):
        evs[i][0].record(stream)
        s, _ = step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    tot = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms = float(tot.item()) / steps
    b = best_candidate(s)
    out = {"workload": "%d placement candidates of C3 (cells moved by N(0, %.1f um)), candidate c -> "
                       "rank c mod N, a rank's candidates in one ws_run with position gradients, "
                       "(TNS, WNS, loss) and dL/dxy all-gathered" % (n_total, sigma_um),
           "candidates_per_gpu": nc, "ms_per_batch": round(ms, 4),
           "candidates_per_s": round(n_total / (ms * 1e-3), 2), "steps": steps,
           "best": {"candidate": b, "loss": float(s[b, 2]), "tns": float(s[b, 0])}}
    dev.close()
    return out


def c2_sta(steps=20):
    """C2: the ICCAD-2015-shaped 995,808-pin heavy-tail
    netlist, forward AT / RAT / slack + TNS/WNS only (run_engine), one B200;
    CUDA events per pass, a >L2 buffer rewritten between passes.  Roofline
    on B_sta."""
    import torch
    import paper_2603_28381_b200 as ws
    from paper_2603_28381_b200 import _lib, generator as G
    raw = G.generate_raw(G.config_c2())
    dev = ws.DeviceDesign(raw)
    flags = _lib.RUN_HARD | _lib.RUN_GRAPH
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(3):
        dev.run(flags, stream=stream)
    ts = []
    for i in range(steps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dev.run(flags, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    P, M, N, A, I, E = dev.n_pins, dev.n_members, dev.n_nets, dev.n_arcs, dev.n_pi, dev.n_ep
    B = 224 * P + 76 * M + 44 * N + 76 * A + 68 * I + 36 * E
    peak, _ = measured_peaks()
    tns, wns, _ = dev.summary()
    out = {"workload": "C2 ICCAD-2015-shaped 995,808-pin heavy-tail netlist: forward AT/RAT/slack + "
                       "TNS/WNS (run_engine)", "pins": P, "levels": dev.n_levels,
           "ms_per_pass": round(ms, 4), "algorithmic_bytes": B,
           "achieved_gbs": round(B / (ms * 1e-3) / 1e9, 1), "frac": round(B / (ms * 1e-3) / 1e9 / peak, 4),
           "launches": dev.last_launch_count(), "tns": tns, "wns": wns}
    dev.close()
    return out


def placement_loop(raw, n_inv=200, sigma_um=0.5, seed=1000):
    """C4: the timing-driven placement loop — n_inv STA
    fwd+bwd invocations on the C3 netlist with perturbed pin coordinates,
    each returning loss / TNS / WNS and dL/dxy (position gradients).

    Invocation t moves every cell by N(0, sigma_um) (seed + t, pins follow
    their cell; coordinates generated on the device before the timed loop),
    then one ws_run does wire RC -> RC -> forward + LSE -> backward +
    adjoint -> position gradients.  Device time: CUDA events around all
    n_inv invocations (each = D2D install of its coordinates + ws_run).  e2e:
    the same loop through the public API with each invocation's positions
    copied from pinned host memory and loss / TNS / WNS read back."""
    import torch
    import paper_2603_28381_b200 as ws
    from paper_2603_28381_b200 import placement as PL
    pl = PL.synthetic_placement(raw, seed=3)
    dev = ws.DeviceDesign(raw, n_corners=2)     # corner 1: the e2e's second input slot
    timer = PL.PlacementTimer(dev, pl)
    PL.PlacementTimer(dev, pl, corner=1)
    stream = torch.cuda.current_stream()
    cell_xy = torch.as_tensor(pl.cell_xy, device="cuda")
    cop = torch.as_tensor(pl.cell_of_pin, device="cuda")
    off = torch.as_tensor(pl.pin_offset, device="cuda")
    xy = dev.value_tensor("xy")          # the corner's position array in HBM
    summ = dev.tensor("summary")
    # every invocation's coordinates, generated on the device up front (the
    # placer's input stream; 8 GB of HBM at C3): cell k of invocation t moves
    # by N(0, sigma) from torch's Philox stream seeded seed + t
    xy_all = torch.empty((n_inv,) + tuple(off.shape), dtype=torch.float64, device="cuda")
    gen = torch.Generator(device="cuda")
    for t in range(n_inv):
        gen.manual_seed(seed + t)
        disp = torch.randn(cell_xy.shape, generator=gen, device="cuda", dtype=torch.float64)
        torch.add((cell_xy + sigma_um * disp).index_select(0, cop), off, out=xy_all[t])

    def invocation(t):
        xy.copy_(xy_all[t])
        dev.run(timer.flags, gamma=timer.gamma, stream=stream)

    for t in range(3):
        invocation(t)
    torch.cuda.synchronize()
    launches = dev.last_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(n_inv):
        invocation(t)
    e1.record(stream)
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1)
    loss_last = dev.summary()
    # e2e: positions from pinned host memory (copy stream, straight into one
    # of two corner slots so invocation t+1's copy overlaps invocation t),
    # summary back, every invocation
    rng = np.random.default_rng(seed)
    host_xy = [torch.from_numpy(np.ascontiguousarray(
        pl.xy + sigma_um * rng.standard_normal(pl.cell_xy.shape)[pl.cell_of_pin])).pin_memory()
        for _ in range(2)]
    h_out = torch.zeros(3, dtype=torch.float64).pin_memory()
    xys = [dev.value_tensor("xy", b) for b in range(2)]
    summs = [dev.tensor("summary", b) for b in range(2)]
    cstream = torch.cuda.Stream()
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]

    def copy_in(t):
        b = t % 2
        cstream.wait_event(consumed[b])
        with torch.cuda.stream(cstream):
            xys[b].copy_(host_xy[t % 2], non_blocking=True)
        copied[b].record(cstream)

    def e2e_inv(t, nxt=True):
        b = t % 2
        stream.wait_event(copied[b])
        if nxt:
            copy_in(t + 1)
        dev.run(timer.flags, corner=b, gamma=timer.gamma, stream=stream)
        consumed[b].record(stream)
        h_out.copy_(summs[b], non_blocking=True)

    for b in range(2):
        consumed[b].record(stream)
    copy_in(0)
    e2e_inv(0)
    e2e_inv(1, nxt=False)
    n_e2e = min(n_inv, 50)
    torch.cuda.synchronize()
    e0.record(stream)
    cstream.wait_event(e0)
    copy_in(0)
    for t in range(n_e2e):
        e2e_inv(t, nxt=t + 1 < n_e2e)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / n_e2e
    dev.close()
    return {"workload": "C4 timing-driven placement loop on C3: %d STA fwd+bwd invocations with "
                        "perturbed pin coordinates (cells moved by N(0, %.1f um)), position "
                        "gradients dL/dxy every invocation" % (n_inv, sigma_um),
            "invocations": n_inv, "total_ms": round(dev_ms, 3),
            "ms_per_invocation": round(dev_ms / n_inv, 4),
            "launches_per_invocation": launches,
            "e2e": {"ms_per_invocation": round(e2e_ms, 4), "invocations": n_e2e,
                    "h2d_bytes_per_step": int(host_xy[0].numel() * 8), "d2h_bytes_per_step": 24},
            "last": {"tns": loss_last[0], "wns": loss_last[1], "loss": loss_last[2]}}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--mode", default="fused",
                    choices=("persistent", "fused", "streams", "sequential"))
    ap.add_argument("--graph", type=int, default=1)
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--workload", default="c3", choices=("c1", "c2", "c3"))
    ap.add_argument("--corners", type=int, default=1,
                    help="also measure the C5 16-corner batch (corner_batch key); 0: skip")
    ap.add_argument("--placement", type=int, default=200,
                    help="C4 placement-loop invocations reported under placement_loop (0: skip)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2603_28381_b200 import generator as G
    cfg = {"c1": G.config_c1(), "c2": G.config_c2(), "c3": G.config_c3()}[args.workload]
    workload = {"c1": "C1 10k-pin", "c2": "C2 1M-pin heavy-tail",
                "c3": "C3 synthetic superblue-shaped 2.5M-pin"}[args.workload]
    config = {"workload": f"{workload} differentiable STA fwd+bwd (hinge-TNS gradients)",
              "generator": cfg.to_doc(), "corners_per_gpu": 1,
              "parallelism": f"corner-sharded x{args.gpus} (weak)"}

    if args.impl == "reference":
        if rank != 0:
            return 0
        t0 = time.time()
        raw = G.generate_raw(cfg)
        log(f"[ref] generated {raw.n_pins} pins in {time.time() - t0:.1f}s")
        budget = max(30.0, min(150.0, 6.0 * (args.steps + args.warmup)))
        r = time_reference(raw, max_passes=args.steps, budget_s=budget)
        cores = 1
        line = {"impl": "reference", "metric": METRIC, "value": round(r["ms"], 3), "unit": "ms",
                "n_gpus": args.gpus, "steps": r["passes"], "warmup": 1,
                "ms_per_step": round(r["ms"], 3), "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator)",
                "config": config,
                "cpu_baseline": {"value": round(r["ms"], 3), "unit": "ms", "cores": cores,
                                 "kind": r["kind"],
                                 "sample": f"{r['passes']} full C3 passes after 1 warm-up "
                                           f"({r['what']}, single-threaded by construction, "
                                           f"{cpu_model()})"},
                "e2e": {"value": round(r["ms"], 3), "unit": "ms", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    # WS_BENCH_SHARE_GPU=1 (testing only): every rank on cuda:0 over gloo, so
    # the N>1 path can be exercised on a one-GPU box
    share = os.environ.get("WS_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    # one explicit stream for everything the bench enqueues (flush, events,
    # engine passes, collectives): nothing can reorder around the timed work
    torch.cuda.set_stream(torch.cuda.Stream())
    dist = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2603_28381_b200 as ws
    from paper_2603_28381_b200 import _lib
    from paper_2603_28381_b200.corners import reduce_batch

    t0 = time.time()
    raw = G.generate_raw(cfg)
    t_gen = time.time() - t0
    t0 = time.time()
    dev = ws.DeviceDesign(raw, n_corners=2)     # corner 1: the e2e's second input slot
    torch.cuda.synchronize()
    t_build = time.time() - t0
    if world > 1 or rank > 0:
        for b in range(2):
            dev.set_values(b, **corner_values(raw, rank))
    log(f"[rank {rank}] {raw.n_pins} pins, {dev.n_levels} levels; generate {t_gen:.1f}s, "
        f"device build {t_build * 1e3:.0f} ms")

    flags = _lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD
    flags |= {"persistent": _lib.RUN_PERSISTENT, "fused": _lib.RUN_FUSED,
              "streams": _lib.RUN_TWO_STREAM, "sequential": 0}[args.mode]
    if args.graph:
        flags |= _lib.RUN_GRAPH
    stream = torch.cuda.current_stream()
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")

    # zero-copy torch views of the corner's results in HBM
    d_arc, d_edge, summ = dev.tensor("d_arc"), dev.tensor("d_edge"), dev.tensor("summary")

    def step():
        dev.run(flags, stream=stream)

    def collectives():
        if world > 1:
            # the batch objective: TNS / loss SUM, WNS MIN, gradients SUM
            reduce_batch(summ, d_arc, d_edge)

    for _ in range(max(3, args.warmup)):
        step()
        collectives()
    torch.cuda.synchronize()
    launches = dev.last_launch_count()

    # ---- timed region: K passes, each bracketed by CUDA events on the launch
    # stream; a >L2 buffer is rewritten between passes (outside the events)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i)
            evs[i][0].record(stream)
            step()
            collectives()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    per = [a.elapsed_time(b) for a, b in evs]
    tot = torch.tensor([sum(per)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_step = float(tot.item()) / args.steps
    value = ms_step / world
    tns, wns, loss = dev.summary()

    # ---- e2e through the public API with pinned host inputs
    vals = corner_values(raw, rank) if (world > 1 or rank > 0) else dict(
        mem_res=raw.mem_res, mem_cap=raw.mem_cap, root_cap=raw.root_cap)
    h_in = {k: torch.from_numpy(np.ascontiguousarray(vals[k])).pin_memory()
            for k in ("mem_res", "mem_cap", "root_cap")}
    h_out = torch.zeros(3, dtype=torch.float64).pin_memory()
    h2d = sum(t.numel() for t in h_in.values()) * 8
    d2h = h_out.numel() * 8

    # Each step's RC inputs go H2D straight into one of two corner slots of
    # the context (corner i % 2; both share the topology), so step i+1's copy
    # overlaps step i's pass and no device-to-device install competes with
    # the copy engine.  The step then runs its slot and reads TNS / WNS / loss
    # back.  Every step's H2D and D2H is inside the timed region.
    cstream = torch.cuda.Stream()
    views = [{k: dev.value_tensor(k, b) for k in h_in} for b in range(2)]
    summs = [dev.tensor("summary", b) for b in range(2)]
    grads = [(dev.tensor("d_arc", b), dev.tensor("d_edge", b)) for b in range(2)]
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]

    def stage_copy(i):
        b = i % 2
        cstream.wait_event(consumed[b])
        with torch.cuda.stream(cstream):
            for k, v in h_in.items():
                views[b][k].copy_(v, non_blocking=True)
        copied[b].record(cstream)

    def e2e_step(i, prefetch_next=True):
        b = i % 2
        stream.wait_event(copied[b])
        if prefetch_next:
            stage_copy(i + 1)
        dev.run(flags, corner=b, stream=stream)
        consumed[b].record(stream)
        if world > 1:
            reduce_batch(summs[b], *grads[b])
        h_out.copy_(summs[b], non_blocking=True)

    for b in range(2):
        consumed[b].record(stream)
    stage_copy(0)
    e2e_step(0)
    e2e_step(1, prefetch_next=False)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ke = max(3, min(args.steps, 10))
    windows = []
    for _ in range(3):                       # median of three pipelined windows of ke steps
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0.record(stream)
        cstream.wait_event(e0)
        stage_copy(0)                        # the first timed step's inputs
        for i in range(ke):
            e2e_step(i, prefetch_next=i + 1 < ke)
        e1.record(stream)
        torch.cuda.synchronize()
        windows.append(e0.elapsed_time(e1))
    e2e_tot = torch.tensor([sorted(windows)[1]], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(e2e_tot, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_tot.item()) / ke / world

    # per-kernel-class breakdown of the same pass: a fused pass with a CUDA
    # event after every launch (the events serialise the PDL overlap, so the
    # classes sum to more than the pass), and the ncu-measured DRAM bytes of
    # each class (profiles/traffic_*.json) over its event time
    kclass = None
    if rank == 0:
        tflags = (flags & ~_lib.RUN_GRAPH) | _lib.RUN_TIMED
        runs = []
        for _ in range(4):
            dev.run(tflags, stream=stream)
            runs.append(dev.kernel_times())
        names = {0: "k_rc_flat (+free pins)", 1: "k_fwd<1,1> (fwd+LSE level)",
                 2: "k_bwd<1,1> (bwd+grad level)", 5: "k_fin_summary"}
        acc = {}
        for kt in runs[1:]:
            for kind, lvl, ms in kt:
                a = acc.setdefault(kind, [0, 0.0])
                a[0] += 1
                a[1] += ms
        traffic_pk = {}
        tp = os.path.join(REPO, "profiles", "traffic_r01.json")
        if os.path.exists(tp):
            try:
                for k, v in json.load(open(tp)).get("per_kernel", {}).items():
                    for key, nm in (("k_rc_flat", 0), ("k_fwd<", 1), ("k_bwd<", 2), ("k_fin_summary", 5)):
                        if key in k:
                            traffic_pk[nm] = v["dram_bytes"] / max(1, v["launches"])
            except Exception:
                traffic_pk = {}
        kclass = []
        for kind in (1, 2, 0, 5):
            if kind not in acc:
                continue
            n, tot = acc[kind]
            avg_us = 1e3 * tot / n
            row = {"kernel": names[kind], "launches_per_pass": n // (len(runs) - 1),
                   "avg_launch_us": round(avg_us, 2)}
            if kind in traffic_pk:
                row["dram_bytes_per_launch"] = int(traffic_pk[kind])
                row["dram_gbs"] = round(traffic_pk[kind] / (avg_us * 1e-6) / 1e9, 1)
            kclass.append(row)

    cb = pb = None
    if args.corners and 16 % world == 0:
        cb = corner_batch(raw, rank, world, flags, steps=max(3, min(args.steps, 10)), dist=dist)
        pb = candidate_batch(raw, rank, world, steps=6, dist=dist)

    if rank == 0:
        P, M, N, A, I, E = (dev.n_pins, dev.n_members, dev.n_nets, dev.n_arcs, dev.n_pi, dev.n_ep)
        B = algorithmic_bytes(P, M, N, A, I, E)
        peak, peak_src = measured_peaks()
        achieved = B / (ms_step * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(REPO, "profiles", "traffic_r01.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get("bytes_per_pass")
            except Exception:
                traffic = None
        line = {"metric": METRIC, "value": round(value, 4), "unit": "ms", "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 4),
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference generator port, BASELINE.md §2 C3; corner k values per rank)",
                "config": dict(config, mode=args.mode, cuda_graph=bool(args.graph),
                               l2="inputs larger than L2 (1.03 GB/pass vs 126 MB) and a 252 MB "
                                  "buffer rewritten between timed passes"),
                "corners_per_s": round(1e3 / value, 2),
                "achieved_hbm_gbs": round(achieved, 1),
                "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                             "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                             "kernel": "whole pass (one ws_run: %d launches)" % launches,
                             "algorithmic_bytes_per_pass": B, "peak_source": peak_src},
                "e2e": {"value": round(e2e_ms, 4), "unit": "ms", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h,
                        "how": "public API (DeviceDesign value_tensor views / run / summary view): "
                               "each step's pinned H2D on a copy stream straight into one of two "
                               "corner slots, so step i+1's copy overlaps step i's pass; D2H of "
                               "TNS/WNS/loss every step"},
                "gpu_launches": launches * args.steps,
                "clocks": clk.summary(),
                "result": {"tns": tns, "wns": wns, "loss": loss},
                "init": {"generate_s": round(t_gen, 2), "device_build_ms": round(t_build * 1e3, 1)}}
        if kclass:
            line["roofline"]["kernel_classes"] = kclass
        if cb is not None:
            line["corner_batch"] = cb
        if pb is not None:
            line["candidate_batch"] = pb
        if args.placement and world == 1:
            line["placement_loop"] = placement_loop(raw, n_inv=args.placement)
        if args.corners and world == 1:
            line["c2_sta"] = c2_sta()
        if args.cpu_baseline and world == 1:
            r = time_reference(raw, max_passes=3, budget_s=25.0)
            line["cpu_baseline"] = {"value": round(r["ms"], 3), "unit": "ms", "cores": 1,
                                    "kind": r["kind"],
                                    "sample": f"{r['passes']} full C3 passes after 1 warm-up "
                                              f"({r['what']}; {cpu_model()})"}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    dev.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
