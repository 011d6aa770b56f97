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


def _plan(n0, world, rank, R):
    """Boundary / interior planes of a rank (the split hjb_shard.cu's
    plane_split makes, in global plane numbers)."""
    b, e = slab_partition(n0, world, rank)
    has_lo, has_hi = rank > 0, rank < world - 1
    lo_end = b + R if has_lo else b
    hi_beg = e - R if has_hi else e
    if world == 1:
        return b, e, [], [(b, e)]
    if lo_end >= hi_beg:
        return b, e, [(b, e)], []
    bnd = ([(b, lo_end)] if has_lo else []) + ([(hi_beg, e)] if has_hi else [])
    return b, e, bnd, [(lo_end, hi_beg)]


def _pipelined_worker(rank, world, port, out_path, order, rk):
    """The round-2 protocol of hjb_solve_sharded_dev, step by step on CPU:
    per stage the BOUNDARY planes are swept first and the stage OUTPUT's
    boundary planes travel (isend/irecv) while the INTERIOR planes sweep;
    the residual all-reduce of sweep k is asynchronous and its epilogue is
    applied only after sweep k + 1 was issued (pipelined); a stop at sweep k
    keeps V_{k+1}, which the speculative sweep k + 1 does not overwrite."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Restatement
    ora = Restatement(threads=1)
    g, model, db, c, cfg = _problem()
    max_iters = 60 if (order > 1 or rk > 1) else cfg.max_iters
    n0 = g.dim(0).n
    s0 = g.size() // n0
    R = order
    b, e, bnd, inner = _plan(n0, world, rank, R)
    dt = ora.cfl_dt(g, model, db, cfg.cfl_factor)
    vbuf = [c.copy(), c.copy()]
    sbuf = {"s1": c.copy(), "s2": c.copy()}

    def exchange_start(a):
        reqs, got = [], []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(a[b * s0:(b + R) * s0].copy()), rank - 1))
            lo = torch.empty(R * s0, dtype=torch.float64)
            reqs.append(dist.irecv(lo, rank - 1))
            got.append(((b - R) * s0, lo))
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(a[(e - R) * s0:e * s0].copy()), rank + 1))
            hi = torch.empty(R * s0, dtype=torch.float64)
            reqs.append(dist.irecv(hi, rank + 1))
            got.append((e * s0, hi))
        return reqs, got, a

    def exchange_finish(x):
        reqs, got, a = x
        for q in reqs:
            q.wait()
        for off, t in got:
            a[off:off + t.numel()] = t.numpy()

    exchange_finish(exchange_start(vbuf[0]))  # halos of V_0
    stages = _STAGES[rk]
    hist, it, converged, stopped = [], 0, False, False
    min_res, first = float("inf"), None
    pending = None
    k = 0
    while True:
        vn, out = vbuf[k & 1], vbuf[(k + 1) & 1]
        names = {"v": vn, "n": out, **sbuf}
        local = 0.0
        for src, dst, kind in stages:
            def run(ranges):
                m = 0.0
                for pb, pe in ranges:
                    if order == 1 and rk == 1:
                        m = max(m, ora.sweep_planes(g, model, db, names[src], c, dt, pb, pe,
                                                    names[dst]))
                    else:
                        m = max(m, ora.ho_stage_planes(g, model, db, names[src], vn, c, dt, order,
                                                       kind, pb, pe, names[dst]))
                return m
            local = run(bnd)  # the final stage's max|V_{n+1} - V_n| is the sweep's
            x = exchange_start(names[dst])  # travels while the interior sweeps
            local = max(local, run(inner))
            exchange_finish(x)
        t = torch.tensor([local], dtype=torch.float64)
        work = dist.all_reduce(t, op=dist.ReduceOp.MAX, async_op=True)
        if pending is not None:  # epilogue of sweep k - 1, after sweep k was issued
            pw, pt = pending
            pw.wait()
            residual = float(pt.item()) / dt
            it += 1
            hist.append(residual)
            if residual < cfg.tolerance:
                converged = stopped = True
            else:
                if first is None:
                    first = residual
                min_res = min(min_res, residual)
                assert residual <= 10 * max(min_res, first)
            if it >= max_iters:
                stopped = True
        if stopped:
            work.wait()  # the speculative sweep's all-reduce completes too
            break
        pending = (work, t)
        k += 1
    final = vbuf[it & 1]  # V_it: untouched by the speculative sweep
    gathered = [None] * world
    dist.all_gather_object(gathered, (b, e, final[b * s0:e * s0].copy(), it, converged, hist))
    if rank == 0:
        full = np.empty(g.size())
        for (bb, ee, arr, _, _, _) in gathered:
            full[bb * s0:ee * s0] = arr
        np.savez(out_path, value=full, iterations=it, converged=converged, history=np.array(hist))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,order,rk", [(2, 1, 1), (3, 1, 1), (2, 3, 3), (3, 2, 2)])
def test_pipelined_overlap_protocol_matches_unsharded(tmp_path, oracle, world, order, rk):
    out = tmp_path / "res.npz"
    mp.spawn(_pipelined_worker, args=(world, _free_port(), str(out), order, rk), nprocs=world,
             join=True)
    r = np.load(out)
    g, model, db, c, cfg = _problem()
    if order > 1 or rk > 1:
        cfg = hj.SolveConfig(tolerance=cfg.tolerance, max_iters=60, spatial_order=order,
                             time_order=rk)
    want = oracle.solve(hj.ScalarField(g, c), hj.ScalarField(g, c), model, db, cfg)
    assert int(r["iterations"]) == want.iterations
    assert bool(r["converged"]) == want.converged
    assert np.array_equal(r["history"], want.residual_history)
    assert np.array_equal(r["value"], want.value.values())


def test_plane_split_covers_slab():
    """Boundary + interior ranges tile every rank's slab exactly once."""
    for n0, world, R in ((101, 8, 1), (101, 8, 3), (11, 3, 3), (17, 4, 2), (9, 2, 1)):
        for rank in range(world):
            b, e, bnd, inner = _plan(n0, world, rank, R)
            planes = sorted(p for lo, hi in bnd + inner for p in range(lo, hi))
            assert planes == list(range(b, e))


def _cpp_plan(n0, world, rank, R):
    """hjb_slab_plan (the C++ the sharded drivers run) in global planes."""
    from paper_2101_05916_b200.sharded import slab_plan
    p = slab_plan(n0, world, rank, R)
    gl = lambda x: x - p["cbeg"] + p["global_begin"]  # noqa: E731
    bnd = [(gl(p["b0"]), gl(p["e0"]))] if p["e0"] > p["b0"] else []
    if p["e1"] > p["b1"]:
        bnd.append((gl(p["b1"]), gl(p["e1"])))
    inner = [(gl(p["i0"]), gl(p["i1"]))] if p["i1"] > p["i0"] else []
    return p, gl, bnd, inner


@pytest.mark.parametrize("n0,world,R", [(101, 8, 1), (101, 8, 3), (11, 3, 3), (17, 4, 2),
                                        (9, 2, 1), (51, 1, 2), (101, 2, 3), (12, 4, 3)])
def test_cpp_slab_plan_matches_protocol(n0, world, R):
    """The native per-rank plan (geometry, halo planes, boundary-first split)
    is the one the CPU protocol tests above run: owned ranges tile the axis,
    every halo a rank receives is exactly the planes its neighbour sends, the
    planes a rank sends lie in its boundary ranges (swept before the
    exchange starts), and boundary + interior tile the slab once."""
    plans = [_cpp_plan(n0, world, r, R) for r in range(world)]
    nxt = 0
    for r, (p, gl, bnd, inner) in enumerate(plans):
        b, e = slab_partition(n0, world, r)
        assert (p["global_begin"], p["owned"]) == (b, e - b) and b == nxt
        nxt = e
        assert (p["cbeg"], p["cend"] - p["cbeg"]) == (R if r > 0 else 0, e - b)
        assert p["nloc"] == p["owned"] + R * ((r > 0) + (r < world - 1)) and p["halo"] == R
        planes = sorted(q for lo, hi in bnd + inner for q in range(lo, hi))
        assert planes == list(range(b, e))
        if world > 1:
            assert sorted(bnd + inner) == sorted(_plan(n0, world, r, R)[2] + _plan(n0, world, r, R)[3])
        sends = [p["send_lo"]] if r > 0 else []
        sends += [p["send_hi"]] if r < world - 1 else []
        for s in sends:  # the exchanged planes are produced by the boundary pass
            assert all(any(lo <= gl(s + i) < hi for lo, hi in bnd) for i in range(R))
        if r < world - 1:
            q, gq = plans[r + 1][0], plans[r + 1][1]
            assert [gl(p["send_hi"] + i) for i in range(R)] == [gq(q["recv_lo"] + i) for i in range(R)]
            assert [gl(p["recv_hi"] + i) for i in range(R)] == [gq(q["send_lo"] + i) for i in range(R)]
            assert p["recv_hi"] == p["cend"] and q["recv_lo"] == 0
        else:
            assert p["send_hi"] == p["recv_hi"] == -1
    assert nxt == n0
