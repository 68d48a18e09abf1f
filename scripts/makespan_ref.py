"""The reference's two-lane makespan model (stasim/fusion.py:163-265) run on
costs MEASURED on the device.

The model itself is NOT restated in this repo: this script imports the
unmodified reference (baseline/_ref, else oracle/_ref) and calls its own
``build_kernel_graph`` / ``schedule_sequential`` / ``schedule_fused`` /
``check_schedule`` on the per-kernel costs of
``paper_2603_28381_b200.fusion.measured_kernel_costs``, next to the measured
sequential, two-stream and interleaved passes of the same design.
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def reference_fusion():
    for d in (os.path.join(REPO, "baseline", "_ref"), os.path.join(REPO, "oracle", "_ref")):
        if os.path.isdir(os.path.join(d, "stasim")):
            if d not in sys.path:
                sys.path.insert(0, d)
            import stasim.fusion as RF
            return RF
    return None


def makespan_report(flat, granularity=10, loss="hinge", repeats=5):
    """Events between launches serialise the programmatic-dependent-launch
    overlap of the untimed pass, so the raw per-launch deltas are calibrated
    to the measured sequential pass (same proportions, same total); the
    reference's model then predicts the two-lane makespan, and the contention
    factor reproducing the measured two-stream pass is fitted (the
    reference's ``contention`` knob)."""
    import torch
    from paper_2603_28381_b200 import _lib, fusion as F
    from paper_2603_28381_b200.diff import default_gamma
    from paper_2603_28381_b200.flatten import device_of
    RF = reference_fusion()
    if RF is None:
        raise RuntimeError("the reference is not installed (baseline/_ref or oracle/_ref)")
    gamma = default_gamma(flat.clock_period)
    dev = device_of(flat)
    raw_costs = F.measured_kernel_costs(dev, flat.n_levels, gamma, loss, repeats)

    def measure(flags):
        ts = []
        for i in range(repeats + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev.run(flags, gamma=gamma, loss=loss, granularity=granularity)
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
    g = RF.build_kernel_graph(flat.n_levels, costs, granularity)
    seq = RF.schedule_sequential(g)
    fus = RF.schedule_fused(g, 1.0)
    lo, hi = 1.0, 8.0
    if RF.schedule_fused(g, hi).makespan < two_ms:
        fit = None
    elif fus.makespan >= two_ms:
        fit = 1.0
    else:
        for _ in range(50):
            mid = 0.5 * (lo + hi)
            lo, hi = (mid, hi) if RF.schedule_fused(g, mid).makespan < two_ms else (lo, mid)
        fit = 0.5 * (lo + hi)
    return {"model": "reference stasim.fusion (unmodified)", "raw_event_sum_ms": total,
            "model_sequential_ms": seq.makespan, "model_fused_ms": fus.makespan,
            "model_overlap_fraction": fus.overlap_fraction, "measured_sequential_ms": seq_ms,
            "measured_two_stream_ms": two_ms, "measured_interleaved_ms": fused_ms,
            "fitted_contention": fit,
            "problems": RF.check_schedule(g, fus) + RF.check_schedule(g, seq)}
