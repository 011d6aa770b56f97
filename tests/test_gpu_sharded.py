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


def test_sharded_single_rank_equals_solve(gpu_ctx):
    w = configs.config2(21)
    c = band_np(w.grid, 0, -4.0, 4.0)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=150)
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
