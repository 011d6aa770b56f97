"""GPU side of the slab partition: plane-range sweeps of the 4D kernel compose
to the full sweep, and the NCCL-driven sharded solve (1 rank on this box)
equals the single-GPU solve bitwise."""
import numpy as np
import pytest
import torch

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj
from paper_2101_05916_b200 import sharded

from cases import band_np, same

pytestmark = pytest.mark.gpu


def _setup(dims):
    g = hj.Grid([(-5.0, 5.0, dims[0]), (-2.0, 2.0, dims[1]), (-0.35, 0.35, dims[2]),
                 (-1.5, 1.5, dims[3])])
    return g, configs.planar_model(), hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])


@pytest.mark.parametrize("world", [2, 3, 8])
def test_slab_sweeps_compose_to_full_sweep(gpu_ctx, oracle, world):
    g, model, db = _setup((17, 9, 8, 11))
    rng = np.random.default_rng(1)
    c = band_np(g, 0, -4.0, 4.0)
    v = c + 0.2 * rng.random(g.size())
    dt = oracle.cfl_dt(g, model, db, 0.8)
    want = oracle.vi_step(hj.ScalarField(g, v), hj.ScalarField(g, c), model, db, dt)
    vt = torch.tensor(v, device="cuda")
    ct = torch.tensor(c, device="cuda")
    full = np.empty(g.size())
    s0 = g.size() // g.dim(0).n
    maxes = []
    for r in range(world):
        b, e = sharded.slab_partition(g.dim(0).n, world, r)
        out = torch.empty_like(vt)
        torch.cuda.synchronize()
        maxes.append(sharded.sweep_planes_dev(g, model, db, vt.data_ptr(), ct.data_ptr(), b, e, dt,
                                              out.data_ptr(), ctx=gpu_ctx))
        full[b * s0:e * s0] = out.cpu().numpy()[b * s0:e * s0]
    assert same(full, want)
    assert max(maxes) == float(np.max(np.abs(want - v)))


@pytest.mark.parametrize("scheme,diss", [(hj.GODUNOV, hj.PER_NODE),
                                         (hj.LAX_FRIEDRICHS, hj.PER_NODE),
                                         (hj.LAX_FRIEDRICHS, hj.GLOBAL)])
def test_sharded_single_rank_equals_solve(gpu_ctx, scheme, diss):
    w = configs.config2(21)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=150, scheme=scheme, dissipation=diss)
    ref = hj.solve(hj.ScalarField(w.grid, c), hj.ScalarField(w.grid, c), w.model, w.dbounds(), cfg,
                   ctx=gpu_ctx)
    ct = torch.tensor(c, device="cuda")
    out = torch.empty_like(ct)
    torch.cuda.synchronize()
    comm = sharded.Comm(gpu_ctx, 0, 1, "cuda")
    try:
        r = sharded.solve_sharded_dev(comm, w.grid, w.model, w.dbounds(), ct.data_ptr(),
                                      ct.data_ptr(), out.data_ptr(), cfg, gpu_ctx,
                                      history_capacity=150)
    finally:
        comm.close()
    assert r.iterations == ref.iterations == 150
    assert same(r.residual_history, ref.residual_history)
    assert same(out.cpu().numpy(), ref.value.values())


@pytest.mark.parametrize("world,order,kind", [(2, 3, 0), (3, 3, 3), (8, 2, 1), (3, 1, 2)])
def test_ho_slab_stages_compose_to_full_stage(gpu_ctx, oracle, world, order, kind):
    """The high-order stage kernel on plane ranges (halo planes read from
    the full arrays) composes to the oracle's full-grid stage."""
    g, model, db = _setup((23, 9, 8, 11))
    rng = np.random.default_rng(3)
    c = band_np(g, 0, -4.0, 4.0)
    vn = c + 0.2 * rng.random(g.size())
    vs = vn + 0.05 * rng.random(g.size())
    dt = oracle.cfl_dt(g, model, db, 0.8)
    want = np.empty(g.size())
    want_dv = oracle.ho_stage_planes(g, model, db, vs, vn, hj.ScalarField(g, c), dt, order, kind,
                                     0, g.dim(0).n, want)
    vst, vnt, ct = (torch.tensor(x, device="cuda") for x in (vs, vn, c))
    full = np.empty(g.size())
    s0 = g.size() // g.dim(0).n
    maxes = []
    for r in range(world):
        b, e = sharded.slab_partition(g.dim(0).n, world, r)
        out = torch.empty_like(vst)
        torch.cuda.synchronize()
        maxes.append(sharded.ho_stage_planes_dev(g, model, db, vst.data_ptr(), vnt.data_ptr(),
                                                 ct.data_ptr(), dt, order, kind, b, e,
                                                 out.data_ptr(), ctx=gpu_ctx))
        full[b * s0:e * s0] = out.cpu().numpy()[b * s0:e * s0]
    assert same(full, want)
    assert max(maxes) == want_dv


@pytest.mark.parametrize("scheme,diss", [(hj.GODUNOV, hj.PER_NODE), (hj.LAX_FRIEDRICHS, hj.PER_NODE),
                                         (hj.LAX_FRIEDRICHS, hj.GLOBAL)],
                         ids=["godunov", "lf_per_node", "lf_global"])
@pytest.mark.parametrize("order,rk", [(2, 2), (3, 3)])
def test_sharded_single_rank_high_order_equals_solve(gpu_ctx, order, rk, scheme, diss):
    w = configs.config2(17)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=1e-5, max_iters=40, spatial_order=order, time_order=rk,
                         scheme=scheme, dissipation=diss)
    ref = hj.solve(hj.ScalarField(w.grid, c), hj.ScalarField(w.grid, c), w.model, w.dbounds(), cfg,
                   ctx=gpu_ctx)
    ct = torch.tensor(c, device="cuda")
    out = torch.empty_like(ct)
    torch.cuda.synchronize()
    comm = sharded.Comm(gpu_ctx, 0, 1, "cuda")
    try:
        r = sharded.solve_sharded_dev(comm, w.grid, w.model, w.dbounds(), ct.data_ptr(),
                                      ct.data_ptr(), out.data_ptr(), cfg, gpu_ctx,
                                      history_capacity=40)
    finally:
        comm.close()
    assert r.iterations == ref.iterations
    assert same(r.residual_history, ref.residual_history)
    assert same(out.cpu().numpy(), ref.value.values())


# ------------------------------------------- in-process ranks (world > 1)
# hjb_solve_sharded_local_dev runs the per-rank plans of the NCCL path
# (slab geometry, halo offsets, boundary planes first, interior while the
# halos travel on a second stream, per-rank epilogues) for P ranks on one
# device; the halo planes move by device copies.  Bitwise vs hjb_solve.

def _local(gpu_ctx, w, c, cfg, P, cap):
    ct = torch.tensor(c, device="cuda")
    out = torch.full_like(ct, float("nan"))
    torch.cuda.synchronize()
    r = sharded.solve_sharded_local_dev(P, w.grid, w.model, w.dbounds(), ct.data_ptr(),
                                        ct.data_ptr(), out.data_ptr(), cfg, gpu_ctx,
                                        history_capacity=cap)
    return r, out.cpu().numpy()


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("overlap", ["1", "0"])
def test_local_ranks_first_order_equal_solve(gpu_ctx, monkeypatch, P, overlap):
    monkeypatch.setenv("HJB_SHARD_OVERLAP", overlap)
    w = configs.config2(21)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=150)
    ref = hj.solve(hj.ScalarField(w.grid, c), hj.ScalarField(w.grid, c), w.model, w.dbounds(), cfg,
                   ctx=gpu_ctx)
    r, v = _local(gpu_ctx, w, c, cfg, P, 150)
    assert r.iterations == ref.iterations == 150 and r.dt == ref.dt
    assert same(r.residual_history, ref.residual_history)
    assert same(v, ref.value.values())


@pytest.mark.parametrize("scheme,diss,P", [(hj.LAX_FRIEDRICHS, hj.PER_NODE, 3),
                                           (hj.LAX_FRIEDRICHS, hj.GLOBAL, 2)])
def test_local_ranks_lax_friedrichs_equal_solve(gpu_ctx, scheme, diss, P):
    w = configs.config2(21)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=120, scheme=scheme, dissipation=diss)
    ref = hj.solve(hj.ScalarField(w.grid, c), hj.ScalarField(w.grid, c), w.model, w.dbounds(), cfg,
                   ctx=gpu_ctx)
    r, v = _local(gpu_ctx, w, c, cfg, P, 120)
    assert r.iterations == ref.iterations
    assert same(r.residual_history, ref.residual_history)
    assert same(v, ref.value.values())


@pytest.mark.parametrize("order,rk,P,scheme", [(3, 3, 2, hj.GODUNOV), (3, 3, 3, hj.GODUNOV),
                                               (2, 2, 4, hj.GODUNOV), (1, 3, 5, hj.GODUNOV),
                                               (3, 3, 2, hj.LAX_FRIEDRICHS),
                                               (2, 2, 3, hj.LAX_FRIEDRICHS)])
def test_local_ranks_high_order_equal_solve(gpu_ctx, order, rk, P, scheme):
    """ENO/TVD-RK slabs: halos of R = ENO order planes after every stage."""
    w = configs.config2(21)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=30, scheme=scheme)
    cfg.spatial_order, cfg.time_order = order, rk
    ref = hj.solve(hj.ScalarField(w.grid, c), hj.ScalarField(w.grid, c), w.model, w.dbounds(), cfg,
                   ctx=gpu_ctx)
    r, v = _local(gpu_ctx, w, c, cfg, P, 30)
    assert r.iterations == ref.iterations == 30
    assert same(r.residual_history, ref.residual_history)
    assert same(v, ref.value.values())


def test_local_ranks_irregular_grid(gpu_ctx):
    """Odd extents on every axis, 3 ranks of 6/6/5 planes, first and third order."""
    g, model, db = _setup((17, 9, 8, 11))
    rng = np.random.default_rng(5)
    c = band_np(g, 0, -4.0, 4.0)
    init = c + 0.3 * rng.random(g.size())
    for order, rk in ((1, 1), (3, 3)):
        cfg = hj.SolveConfig(tolerance=1e-6, max_iters=25)
        cfg.spatial_order, cfg.time_order = order, rk
        ref = hj.solve(hj.ScalarField(g, init), hj.ScalarField(g, c), model, db, cfg, ctx=gpu_ctx)
        it = torch.tensor(init, device="cuda")
        ct = torch.tensor(c, device="cuda")
        out = torch.empty_like(it)
        torch.cuda.synchronize()
        r = sharded.solve_sharded_local_dev(3, g, model, db, it.data_ptr(), ct.data_ptr(),
                                            out.data_ptr(), cfg, gpu_ctx, history_capacity=25)
        assert r.iterations == ref.iterations
        assert same(r.residual_history, ref.residual_history)
        assert same(out.cpu().numpy(), ref.value.values())


def test_local_ranks_converge_in_reference_iteration_count(gpu_ctx):
    """4 in-process ranks solve config 2 at 21^4 to tol 5e-3: the reference's
    16 685 iterations and V* (golden fixture from oracle/_ref)."""
    import json
    from pathlib import Path
    meta = json.loads((Path(__file__).resolve().parent / "golden" / "golden_fullsize.json")
                      .read_text())["conv21"]
    w = configs.config2(21)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=200000)
    r, v = _local(gpu_ctx, w, c, cfg, 4, 0)
    assert r.iterations == meta["iterations"] == 16685 and r.converged
    import hashlib
    assert hashlib.sha256(np.ascontiguousarray(v + 0.0).tobytes()).hexdigest() == meta["value_sha256"]


def test_local_ranks_thin_slab_rejected(gpu_ctx):
    """n0 = 11 over 4 ranks gives 3/3/3/2 planes: ENO3 needs 3 on EVERY rank,
    so the solve fails up front (the NCCL path checks this before any
    collective, so no rank can block in NCCL while another returns)."""
    w = configs.config2(11)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(max_iters=5)
    cfg.spatial_order, cfg.time_order = 3, 3
    with pytest.raises(hj.Unsupported):
        _local(gpu_ctx, w, c, cfg, 4, 5)


@pytest.mark.parametrize("order,rk,P", [(1, 1, 2), (1, 1, 8), (3, 3, 3), (2, 2, 4)])
def test_local_ranks_signal_protocol_equal_solve(gpu_ctx, monkeypatch, order, rk, P):
    """The NCCL transport's default protocol on in-process ranks: ONE launch
    per rank and stage with the boundary items first; the transfer stream
    waits on the launch's boundary flag (cuStreamWaitValue32), moves the
    halos and re-arms it; host-driven loop with one-batch lookahead."""
    monkeypatch.setenv("HJB_SHARD_SIGNAL", "1")
    w = configs.config2(21)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=60)
    cfg.spatial_order, cfg.time_order = order, rk
    ref = hj.solve(hj.ScalarField(w.grid, c), hj.ScalarField(w.grid, c), w.model, w.dbounds(), cfg,
                   ctx=gpu_ctx)
    r, v = _local(gpu_ctx, w, c, cfg, P, 60)
    assert r.iterations == ref.iterations == 60
    assert same(r.residual_history, ref.residual_history)
    assert same(v, ref.value.values())


def test_local_ranks_signal_protocol_converges(gpu_ctx, monkeypatch):
    """Convergence (the loop stops mid-batch; the extra batch's launches find
    done set and still release the transfer stream's flag wait)."""
    monkeypatch.setenv("HJB_SHARD_SIGNAL", "1")
    w = configs.config2(11)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=200000)
    ref = hj.solve(hj.ScalarField(w.grid, c), hj.ScalarField(w.grid, c), w.model, w.dbounds(), cfg,
                   ctx=gpu_ctx)
    r, v = _local(gpu_ctx, w, c, cfg, 3, 0)
    assert r.converged and r.iterations == ref.iterations
    assert same(v, ref.value.values())


# Peer-store halos (HJB_SHARD_P2P=1): the slab sweep kernels store their
# boundary planes straight into the neighbours' halo planes and publish an
# epoch to the neighbours' flags; the next stage's stream waits on its own
# flags.  In-process ranks exercise the same kernels, offsets and flags with
# same-device pointers (the NCCL driver maps the neighbours' buffers over
# CUDA IPC instead).

@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("scheme", ["godunov", "lf_per_node", "lf_global"])
def test_local_ranks_peer_store_equal_solve(gpu_ctx, monkeypatch, P, scheme):
    monkeypatch.setenv("HJB_SHARD_P2P", "1")
    w = configs.config2(21)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=120)
    if scheme != "godunov":
        cfg.scheme = hj.LAX_FRIEDRICHS
        cfg.dissipation = hj.GLOBAL if scheme == "lf_global" else hj.PER_NODE
    ref = hj.solve(hj.ScalarField(w.grid, c), hj.ScalarField(w.grid, c), w.model, w.dbounds(), cfg,
                   ctx=gpu_ctx)
    r, v = _local(gpu_ctx, w, c, cfg, P, 120)
    assert r.iterations == ref.iterations == 120 and r.dt == ref.dt
    assert same(r.residual_history, ref.residual_history)
    assert same(v, ref.value.values())


def test_local_ranks_peer_store_irregular_grid(gpu_ctx, monkeypatch):
    """Odd extents, 3 ranks with unequal slabs, peer-store halos."""
    monkeypatch.setenv("HJB_SHARD_P2P", "1")
    g = hj.Grid([(-5.0, 5.0, 17), (-2.0, 2.0, 9), (-0.35, 0.35, 8), (-1.5, 1.5, 11)])
    model = configs.planar_model()
    db = hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    c = band_np(g, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=1e-5, max_iters=60)
    ref = hj.solve(hj.ScalarField(g, c), hj.ScalarField(g, c), model, db, cfg, ctx=gpu_ctx)
    ct = torch.tensor(c, device="cuda")
    out = torch.full_like(ct, float("nan"))
    torch.cuda.synchronize()
    r = sharded.solve_sharded_local_dev(3, g, model, db, ct.data_ptr(), ct.data_ptr(),
                                        out.data_ptr(), cfg, gpu_ctx, history_capacity=60)
    assert r.iterations == ref.iterations and same(r.residual_history, ref.residual_history)
    assert same(out.cpu().numpy(), ref.value.values())


def test_local_ranks_peer_store_converge_in_reference_iteration_count(gpu_ctx, monkeypatch):
    """4 in-process ranks with peer-store halos solve config 2 at 21^4 to tol
    5e-3: the reference's 16 685 iterations and V* (golden fixture), i.e. the
    epoch protocol holds over every batch, the stop and the extra batch."""
    import json
    import hashlib
    from pathlib import Path
    monkeypatch.setenv("HJB_SHARD_P2P", "1")
    meta = json.loads((Path(__file__).resolve().parent / "golden" / "golden_fullsize.json")
                      .read_text())["conv21"]
    w = configs.config2(21)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=200000)
    r, v = _local(gpu_ctx, w, c, cfg, 4, 0)
    assert r.iterations == meta["iterations"] == 16685 and r.converged
    assert hashlib.sha256(np.ascontiguousarray(v + 0.0).tobytes()).hexdigest() == meta["value_sha256"]


def _mp_probe(np_, n, iters, tol=0.0, order=1):
    """Run scripts/p2p_same_gpu_probe.py in np_ processes on this one GPU with
    the peer-store communicator; one JSON report per rank."""
    import json
    import os
    import socket
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, P2P_COMM="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={np_}",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           str(root / "scripts" / "p2p_same_gpu_probe.py"), str(n), str(iters), str(tol), str(order)]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    # the ranks share one stdout pipe: two reports can land on one line
    reps, dec = [], json.JSONDecoder()
    for ln in out.stdout.splitlines():
        pos = ln.find("{")
        while pos >= 0:
            obj, end = dec.raw_decode(ln, pos)
            reps.append(obj)
            pos = ln.find("{", end)
    assert out.returncode == 0 and len(reps) == np_, out.stdout[-2000:] + out.stderr[-2000:]
    return reps


@pytest.mark.parametrize("np_", [2, 3])
def test_peer_store_comm_multiprocess_equal_solve(np_):
    """The NCCL-free peer-store communicator between PROCESSES (CUDA IPC
    control blocks and V buffers, halos stored by the sweep kernels, residual
    and CFL-scan all-reduces through the ranks' mailboxes), here with all
    ranks on this one GPU: every rank's slab and residual history equal the
    single-process solve bit for bit."""
    for rep in _mp_probe(np_, 21, 60):
        assert rep["ok"] and rep["bitwise"] and rep["history_equal"], rep
        assert rep["iterations"] == rep["ref_iterations"] == 60


def test_peer_store_comm_multiprocess_converges():
    """Two processes to convergence (config 2 at 21^4, tol 5e-3): the
    reference's 16 685 iterations, V bitwise (epochs, mailbox slots and the
    stop across thousands of positions)."""
    for rep in _mp_probe(2, 21, 200000, 5e-3):
        assert rep["ok"] and rep["bitwise"] and rep["converged"], rep
        assert rep["iterations"] == rep["ref_iterations"] == 16685


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("order,rk,scheme", [(2, 2, "godunov"), (3, 3, "godunov"), (3, 3, "lf")])
def test_local_ranks_peer_store_high_order_equal_solve(gpu_ctx, monkeypatch, P, order, rk, scheme):
    """Peer-store halos for ENO / TVD-RK slabs: every stage's boundary planes
    (ghost cells of the ENO3 layout included) go straight into the
    neighbours' stage buffers; bitwise vs the single-GPU solve."""
    monkeypatch.setenv("HJB_SHARD_P2P", "1")
    w = configs.config2(21)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=20, spatial_order=order, time_order=rk)
    if scheme == "lf":
        cfg.scheme = hj.LAX_FRIEDRICHS
    ref = hj.solve(hj.ScalarField(w.grid, c), hj.ScalarField(w.grid, c), w.model, w.dbounds(), cfg,
                   ctx=gpu_ctx)
    r, v = _local(gpu_ctx, w, c, cfg, P, 20)
    assert r.iterations == ref.iterations == 20 and r.dt == ref.dt
    assert same(r.residual_history, ref.residual_history)
    assert same(v, ref.value.values())


def test_peer_store_comm_multiprocess_eno3_rk3():
    """ENO3 + TVD-RK3 slabs (config 3's scheme) between 3 processes on the
    NCCL-free communicator: bitwise vs the single-process solve."""
    for rep in _mp_probe(3, 21, 10, 0.0, 3):
        assert rep["ok"] and rep["bitwise"] and rep["history_equal"], rep
        assert rep["iterations"] == rep["ref_iterations"] == 10
