"""Corner / placement-candidate batches across GPUs.

A single design does not shard (levels serialize), so the unit of
distribution is a whole corner: corner k runs on rank k mod G, each rank
running the full pass for its corners.  One exchange per batch step: the
batch objective sum_k loss_k and TNS are SUM-reduced, WNS MIN-reduced, and
the gradients d_arc / d_edge SUM-reduced (the gradient of the summed
objective).  The tensors are the engine's zero-copy views, so the NCCL
collectives run on the engine's stream right after the pass.

The reference's only analog is its bench process pool (bench.py:188-191).
"""

from __future__ import annotations


def corners_of_rank(n_corners: int, rank: int, world: int) -> list:
    """Round-robin corner ownership: corner k on rank k mod world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return [k for k in range(n_corners) if k % world == rank]


def corner_scales(k: int):
    """C5 corner k: res x (0.85 + 0.02k); caps and LUT
    tables x (0.90 + 0.0125k)."""
    return 0.85 + 0.02 * k, 0.90 + 0.0125 * k


def corner_values(raw, k: int) -> dict:
    fr, fc = corner_scales(k)
    return dict(mem_res=raw.mem_res * fr, mem_cap=raw.mem_cap * fc, root_cap=raw.root_cap * fc,
                lut_t_flat=raw.lut_t_flat * fc)


def reduce_batch(summary, d_arc=None, d_edge=None, group=None):
    """In-place batch reduction over the process group.

    summary: fp64 tensor [3] = (TNS, WNS, loss) of this rank's corners (for
    several local corners, pre-combine them with ``combine_local``).
    TNS, loss: SUM; WNS: MIN; d_arc, d_edge: SUM."""
    import torch
    import torch.distributed as dist
    sl = torch.stack([summary[0], summary[2]])
    dist.all_reduce(sl, op=dist.ReduceOp.SUM, group=group)
    wn = summary[1:2].clone()
    dist.all_reduce(wn, op=dist.ReduceOp.MIN, group=group)
    summary[0] = sl[0]
    summary[2] = sl[1]
    summary[1] = wn[0]
    for g in (d_arc, d_edge):
        if g is not None:
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group)
    return summary


def combine_local(summaries):
    """(TNS, WNS, loss) of several corners on one rank -> one row, in corner
    order (sum, min, sum)."""
    import torch
    s = torch.stack(list(summaries))
    return torch.stack([s[:, 0].sum(), s[:, 1].min(), s[:, 2].sum()])


def gather_candidates(summaries, d_xy=None, group=None, n_candidates=None):
    """Placement-candidate batch (north_star: "multiple placement candidates
    in a timing-driven placement batch"): candidates are
    independent, so nothing is reduced — every rank's (TNS, WNS, loss) rows and
    position gradients are gathered in candidate order.

    summaries: [k, 3] fp64 tensor of this rank's k candidates; d_xy: [k, P, 2]
    or None.  Candidate c lives on rank c mod world as its (c // world)-th
    local candidate (corners_of_rank); returns ([n, 3], [n, P, 2]) in global
    candidate order.  ``n_candidates`` (default world*k) may leave the ranks
    with unequal counts (n % world != 0): every rank then pads to
    ceil(n/world) rows so the all_gather shapes agree, and the padding is
    dropped after the reorder."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    k = summaries.shape[0]
    if n_candidates is None:
        n_candidates = world * k
    kmax = -(-n_candidates // world)           # ceil: every rank sends kmax rows
    if k != len(corners_of_rank(n_candidates, rank, world)):
        raise ValueError(f"rank {rank} holds {k} candidates, expected "
                         f"{len(corners_of_rank(n_candidates, rank, world))} of {n_candidates}")

    def gather(t):
        t = t.contiguous()
        if k < kmax:                            # uneven split: pad to a common shape
            pad = torch.zeros((kmax - k,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            t = torch.cat([t, pad])
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        out = torch.stack(parts)          # out[r, i] is candidate i * world + r
        out = out.transpose(0, 1).reshape((world * kmax,) + tuple(t.shape[1:]))
        return out[:n_candidates]         # padding rows sort last; drop them

    s = gather(summaries)
    g = gather(d_xy) if d_xy is not None else None
    return s, g


def best_candidate(summaries):
    """Index of the candidate with the smallest loss (ties: lowest index)."""
    import torch
    loss = summaries[:, 2]
    return int(torch.argmin(loss).item())
