"""Multi-GPU host logic on CPU: world_size-2 gloo run of the corner-batch
reduction (paper_2603_28381_b200/corners.py) used by bench.py --gpus N.

Each rank owns its round-robin corners of a golden design, evaluates them
with the oracle (the checker; the device path is covered by the gpu tests),
and reduces (TNS, WNS, loss) and the gradients with ``reduce_batch``; rank 0
compares against all corners evaluated serially.
"""

import copy
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_28381_b200 import corners as CO

N_CORNERS = 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _corner_result(name, k):
    from golden_util import load, raw_ns
    from oracle import oracle as O
    g = load(name)
    ns = raw_ns(g)
    base = O.flatten_raw(ns)
    fl = copy.copy(base)
    fr, fc = CO.corner_scales(k)
    fl.mem_res = base.mem_res * fr
    fl.mem_cap = base.mem_cap * fc
    fl.root_cap = base.root_cap * fc
    fl.lut_t_flat = base.lut_t_flat * fc
    st = O.run_engine(fl)
    gr = O.timing_gradients(fl, st, gamma=0.01 * ns.clock_period)
    summ = torch.tensor([O.tns(st, fl), O.wns(st, fl), gr.loss], dtype=torch.float64)
    return summ, torch.from_numpy(gr.d_arc.copy()), torch.from_numpy(gr.d_edge.copy())


def _worker(rank, world, port, name, out):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        mine = CO.corners_of_rank(N_CORNERS, rank, world)
        res = [_corner_result(name, k) for k in mine]
        summ = CO.combine_local([r[0] for r in res])
        d_arc = sum(r[1] for r in res)
        d_edge = sum(r[2] for r in res)
        CO.reduce_batch(summ, d_arc, d_edge)
        if rank == 0:
            torch.save({"summ": summ, "d_arc": d_arc, "d_edge": d_edge}, out)
    finally:
        dist.destroy_process_group()


def test_corner_assignment_round_robin():
    assert CO.corners_of_rank(16, 3, 8) == [3, 11]
    allk = sorted(k for r in range(4) for k in CO.corners_of_rank(16, r, 4))
    assert allk == list(range(16))
    with pytest.raises(ValueError):
        CO.corners_of_rank(4, 2, 2)


@pytest.mark.parametrize("name", ["kat_chain5_viol", "gen_c1_star"])
def test_gloo_world2_batch_reduction(tmp_path, name):
    out = str(tmp_path / "r0.pt")
    mp.spawn(_worker, args=(2, _free_port(), name, out), nprocs=2, join=True)
    got = torch.load(out)
    ref = [_corner_result(name, k) for k in range(N_CORNERS)]
    exp = CO.combine_local([r[0] for r in ref])
    # TNS / loss: sums of 2 partial sums vs a 4-term sum — fp64 reassociation only
    np.testing.assert_allclose(got["summ"][[0, 2]].numpy(), exp[[0, 2]].numpy(), rtol=1e-12)
    assert float(got["summ"][1]) == float(exp[1])                       # MIN is exact
    np.testing.assert_allclose(got["d_arc"].numpy(), sum(r[1] for r in ref).numpy(), rtol=1e-12)
    np.testing.assert_allclose(got["d_edge"].numpy(), sum(r[2] for r in ref).numpy(), rtol=1e-12)


def _cand_worker(rank, world, port, out, n=6):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        mine = CO.corners_of_rank(n, rank, world)
        summ = torch.stack([torch.tensor([-1.0 * c, -0.1 * c, 10.0 - c], dtype=torch.float64)
                            for c in mine])
        dxy = torch.stack([torch.full((5, 2), float(c), dtype=torch.float64) for c in mine])
        s, g = CO.gather_candidates(summ, dxy, n_candidates=n)
        if rank == 0:
            torch.save({"s": s, "g": g, "best": CO.best_candidate(s)}, out)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_candidate_gather(tmp_path):
    """Placement candidates: rank r holds candidates r, r+2, r+4; the gather
    returns all six in candidate order; the best is the lowest loss."""
    out = str(tmp_path / "c.pt")
    mp.spawn(_cand_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = torch.load(out)
    assert got["s"][:, 0].tolist() == [-float(c) for c in range(6)]
    assert all(float(got["g"][c, 0, 0]) == float(c) for c in range(6))
    assert got["best"] == 5


def test_gloo_world2_candidate_gather_uneven(tmp_path):
    """5 candidates on 2 ranks (3 + 2): rank 1 pads to 3 rows so the
    all_gather shapes agree; the result is the 5 candidates in order."""
    out = str(tmp_path / "c5.pt")
    mp.spawn(_cand_worker, args=(2, _free_port(), out, 5), nprocs=2, join=True)
    got = torch.load(out)
    assert got["s"].shape == (5, 3) and got["g"].shape == (5, 5, 2)
    assert got["s"][:, 0].tolist() == [-float(c) for c in range(5)]
    assert all(float(got["g"][c, 0, 0]) == float(c) for c in range(5))
    assert got["best"] == 4


def _engine_worker(rank, world, port, name, out):
    """One rank on the shared cuda:0: its round-robin corners of the design
    in ONE batched ws_run (with the in-kernel batch gradient sum), then the
    batch exchange over gloo."""
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    import paper_2603_28381_b200 as ws
    from paper_2603_28381_b200 import _lib
    from golden_util import load, raw_of
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        raw = raw_of(load(name))
        mine = CO.corners_of_rank(N_CORNERS, rank, world)
        dev = ws.DeviceDesign(raw, n_corners=len(mine))
        for i, k in enumerate(mine):
            dev.set_values(i, **CO.corner_values(raw, k))
        dev.run(_lib.RUN_HARD | _lib.RUN_LSE | _lib.RUN_GRAD | _lib.RUN_FUSED | _lib.RUN_CORNER_SUM,
                corner=0, n_corners=len(mine), gamma=0.01 * raw.clock_period)
        summ = CO.combine_local([dev.tensor("summary", i) for i in range(len(mine))]).cpu()
        d_arc = dev.tensor("d_arc_sum").cpu()
        d_edge = dev.tensor("d_edge_sum").cpu()
        CO.reduce_batch(summ, d_arc, d_edge)
        if rank == 0:
            torch.save({"summ": summ, "d_arc": d_arc, "d_edge": d_edge}, out)
        dev.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["gen_c1_star", "multi_out"])
def test_gloo_world2_engine_batch_on_shared_gpu(tmp_path, name):
    """The multi-GPU data plane with real engine outputs: 2 ranks sharing
    cuda:0, each running its corners through the C-ABI, reduced over gloo;
    rank 0's batch TNS / WNS / loss and gradient sums against the oracle's
    serial evaluation of all 4 corners."""
    out = str(tmp_path / "e0.pt")
    mp.spawn(_engine_worker, args=(2, _free_port(), name, out), nprocs=2, join=True)
    got = torch.load(out)
    ref = [_corner_result(name, k) for k in range(N_CORNERS)]
    exp = CO.combine_local([r[0] for r in ref])
    assert float(got["summ"][1]) == float(exp[1])
    np.testing.assert_allclose(got["summ"][[0, 2]].numpy(), exp[[0, 2]].numpy(), rtol=1e-9)
    for key, idx in (("d_arc", 1), ("d_edge", 2)):
        e = sum(r[idx] for r in ref).numpy()
        scale = max(float(np.abs(e).max()), 1e-300)
        np.testing.assert_allclose(got[key].numpy(), e, rtol=1e-4, atol=1e-9 * scale)
