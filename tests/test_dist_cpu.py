"""Multi-rank slab protocol on CPU (gloo, world_size 2 and 3).

Each rank owns the axis-0 slab given by the library's own partition rule
(hjb_slab_partition), exchanges halo planes with torch.distributed
send/recv, sweeps its planes with the CPU oracle, all-reduces max|dV| and
applies the solve() loop logic (solver.cpp:347-369).  This is the protocol
hjb_solve_sharded_dev runs with NCCL on GPUs; the gathered result must equal
the unsharded solve bitwise, with the same iteration count.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj
from paper_2101_05916_b200.sharded import slab_partition

from cases import band_np


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    g = hj.Grid([(-5.0, 5.0, 11), (-2.0, 2.0, 7), (-0.35, 0.35, 6), (-1.5, 1.5, 5)])
    model = configs.planar_model()
    db = hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    c = band_np(g, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=400)
    return g, model, db, c, cfg


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Restatement
    ora = Restatement(threads=1)
    g, model, db, c, cfg = _problem()
    n0 = g.dim(0).n
    s0 = g.size() // n0
    b, e = slab_partition(n0, world, rank)
    dt = ora.cfl_dt(g, model, db, cfg.cfl_factor)
    v = c.copy()  # full-size array; only planes [b-1, e+1) are ever valid here
    nxt = v.copy()
    hist = []
    min_res, first = float("inf"), None
    it = 0
    converged = False
    while it < cfg.max_iters:
        # halo exchange: first owned plane to rank-1, last to rank+1
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(v[b * s0:(b + 1) * s0].copy()), rank - 1))
            lo = torch.empty(s0, dtype=torch.float64)
            reqs.append(dist.irecv(lo, rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(v[(e - 1) * s0:e * s0].copy()), rank + 1))
            hi = torch.empty(s0, dtype=torch.float64)
            reqs.append(dist.irecv(hi, rank + 1))
        for q in reqs:
            q.wait()
        if rank > 0:
            v[(b - 1) * s0:b * s0] = lo.numpy()
        if rank < world - 1:
            v[e * s0:(e + 1) * s0] = hi.numpy()
        local = ora.sweep_planes(g, model, db, v, c, dt, b, e, nxt)
        t = torch.tensor([local], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        residual = float(t.item()) / dt
        v, nxt = nxt, v
        it += 1
        hist.append(residual)
        if residual < cfg.tolerance:
            converged = True
            break
        if first is None:
            first = residual
        min_res = min(min_res, residual)
        assert residual <= 10 * max(min_res, first)
    slab = torch.from_numpy(v[b * s0:e * s0].copy())
    gathered = [None] * world
    dist.all_gather_object(gathered, (b, e, slab.numpy(), it, converged, hist))
    if rank == 0:
        full = np.empty(g.size())
        for (bb, ee, arr, _, _, _) in gathered:
            full[bb * s0:ee * s0] = arr
        np.savez(out_path, value=full, iterations=it, converged=converged, history=np.array(hist))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_protocol_matches_unsharded(tmp_path, oracle, world):
    out = tmp_path / "res.npz"
    mp.spawn(_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    r = np.load(out)
    g, model, db, c, cfg = _problem()
    want = oracle.solve(hj.ScalarField(g, c), hj.ScalarField(g, c), model, db, cfg)
    assert int(r["iterations"]) == want.iterations
    assert bool(r["converged"]) == want.converged
    assert np.array_equal(r["history"], want.residual_history)
    assert np.array_equal(r["value"], want.value.values())


def test_partition_rule():
    for n0, P in ((101, 8), (51, 4), (11, 3), (7, 7)):
        spans = [slab_partition(n0, P, r) for r in range(P)]
        assert spans[0][0] == 0 and spans[-1][1] == n0
        assert all(spans[i][1] == spans[i + 1][0] for i in range(P - 1))
        sizes = [e - b for b, e in spans]
        assert max(sizes) - min(sizes) <= 1
    assert slab_partition(101, 8, 0) == (0, 13) and slab_partition(101, 8, 7) == (89, 101)
    with pytest.raises(hj.InvalidArgument):
        slab_partition(3, 4, 0)


# stage table of a TVD-RK step: (input, output, kind) with buffers
# 'v' (V_n), 's1', 's2', 'n' (V_{n+1}); kind as in k_ho4t / hj_oracle.c
_STAGES = {1: [("v", "n", 0)], 2: [("v", "s1", 0), ("s1", "n", 1)],
           3: [("v", "s1", 0), ("s1", "s2", 2), ("s2", "n", 3)]}


def _ho_worker(rank, world, port, out_path, order, rk):
    """Sharded ENO/TVD-RK solve: halo width R = order planes per side,
    exchanged before EVERY stage, max|dV| all-reduced after the
    last stage."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Restatement
    ora = Restatement(threads=1)
    g, model, db, c, cfg = _problem()
    n0 = g.dim(0).n
    s0 = g.size() // n0
    b, e = slab_partition(n0, world, rank)
    R = order
    dt = ora.cfl_dt(g, model, db, cfg.cfl_factor)
    buf = {k: c.copy() for k in ("v", "s1", "s2", "n")}

    def exchange(a):
        reqs, lo, hi = [], None, None
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(a[b * s0:(b + R) * s0].copy()), rank - 1))
            lo = torch.empty(R * s0, dtype=torch.float64)
            reqs.append(dist.irecv(lo, rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(a[(e - R) * s0:e * s0].copy()), rank + 1))
            hi = torch.empty(R * s0, dtype=torch.float64)
            reqs.append(dist.irecv(hi, rank + 1))
        for q in reqs:
            q.wait()
        if lo is not None:
            a[(b - R) * s0:b * s0] = lo.numpy()
        if hi is not None:
            a[e * s0:(e + R) * s0] = hi.numpy()

    hist, it, converged = [], 0, False
    min_res, first = float("inf"), None
    while it < 60:
        local = 0.0
        for src, dst, kind in _STAGES[rk]:
            exchange(buf[src])
            local = ora.ho_stage_planes(g, model, db, buf[src], buf["v"], c, dt, order, kind, b, e,
                                        buf[dst])
        t = torch.tensor([local], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        residual = float(t.item()) / dt
        buf["v"], buf["n"] = buf["n"], buf["v"]
        it += 1
        hist.append(residual)
        if residual < cfg.tolerance:
            converged = True
            break
        if first is None:
            first = residual
        min_res = min(min_res, residual)
        assert residual <= 10 * max(min_res, first)
    gathered = [None] * world
    dist.all_gather_object(gathered, (b, e, buf["v"][b * s0:e * s0].copy(), it, converged, hist))
    if rank == 0:
        full = np.empty(g.size())
        for (bb, ee, arr, _, _, _) in gathered:
            full[bb * s0:ee * s0] = arr
        np.savez(out_path, value=full, iterations=it, converged=converged, history=np.array(hist))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,order,rk", [(2, 3, 3), (3, 2, 2)])
def test_high_order_slab_protocol_matches_unsharded(tmp_path, oracle, world, order, rk):
    out = tmp_path / "res.npz"
    mp.spawn(_ho_worker, args=(world, _free_port(), str(out), order, rk), nprocs=world, join=True)
    r = np.load(out)
    g, model, db, c, cfg = _problem()
    cfg = hj.SolveConfig(tolerance=cfg.tolerance, max_iters=60, spatial_order=order,
                         time_order=rk)
    want = oracle.solve(hj.ScalarField(g, c), hj.ScalarField(g, c), model, db, cfg)
    assert int(r["iterations"]) == want.iterations
    assert np.array_equal(r["history"], want.residual_history)
    assert np.array_equal(r["value"], want.value.values())
