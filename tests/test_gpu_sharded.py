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
