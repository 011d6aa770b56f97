"""GPU ENO/TVD-RK stages against the repo's CPU restatement (parity unpinned
by the reference, which has no high-order scheme): bitwise values, residual
histories and iteration counts."""
import numpy as np
import pytest

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj

from cases import per_node_case, quad_setup, same, with_iters, workload_case

pytestmark = pytest.mark.gpu


def _cases():
    out = []
    for order, rk in ((1, 2), (2, 2), (3, 3), (2, 3), (3, 1)):
        for scheme, diss in ((hj.GODUNOV, hj.PER_NODE), (hj.LAX_FRIEDRICHS, hj.PER_NODE),
                             (hj.LAX_FRIEDRICHS, hj.GLOBAL)):
            out.append((order, rk, scheme, diss))
    return out


@pytest.mark.parametrize("order,rk,scheme,diss", _cases())
def test_high_order_solve_matches_restatement(gpu_ctx, oracle, order, rk, scheme, diss):
    for case in (with_iters(quad_setup(21), 60), with_iters(workload_case(configs.config2(9)), 12),
                 with_iters(per_node_case(13), 40)):
        cfg = hj.SolveConfig(**case.cfg.__dict__)
        cfg.spatial_order, cfg.time_order, cfg.scheme, cfg.dissipation = order, rk, scheme, diss
        want = oracle.solve(case.init_field(), case.c_field(), case.model, case.db, cfg)
        got = hj.solve(case.init_field(), case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
        assert got.iterations == want.iterations, case.name
        assert same(got.residual_history, want.residual_history), case.name
        assert same(got.value.values(), want.value.values()), case.name


def test_forced_stage_machinery_is_the_reference_update(gpu_ctx, oracle):
    case = with_iters(workload_case(configs.config2(11)), 40)
    want = oracle.solve(case.init_field(), case.c_field(), case.model, case.db, case.cfg)
    cfg = hj.SolveConfig(**case.cfg.__dict__)
    cfg.flags = 1
    got = hj.solve(case.init_field(), case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
    assert same(got.value.values(), want.value.values())
    assert same(got.residual_history, want.residual_history)


def test_config1_eno2_rk2(gpu_ctx, oracle):
    """BASELINE config 1 as named: ENO2 + TVD-RK2, CFL 0.8, tol 1e-4."""
    case = workload_case(configs.config1())
    cfg = hj.SolveConfig(**case.cfg.__dict__)
    cfg.spatial_order, cfg.time_order = 2, 2
    want = oracle.solve(case.init_field(), case.c_field(), case.model, case.db, cfg)
    got = hj.solve(case.init_field(), case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
    assert got.converged and got.iterations == want.iterations
    assert same(got.value.values(), want.value.values())


def test_high_order_vi_step(gpu_ctx, oracle):
    case = workload_case(configs.config2(9))
    rng = np.random.default_rng(2)
    v = hj.ScalarField(case.grid, case.c + 0.2 * rng.random(case.grid.size()))
    for order, rk in ((2, 2), (3, 3)):
        cfg = hj.SolveConfig(spatial_order=order, time_order=rk, max_iters=1, tolerance=1e-300)
        want = oracle.solve(v, case.c_field(), case.model, case.db, cfg)
        dt = oracle.cfl_dt(case.grid, case.model, case.db, 0.8)
        got = hj.vi_step(v, case.c_field(), case.model, case.db, dt, cfg, ctx=gpu_ctx)
        assert same(got.values(), want.value.values())


@pytest.mark.parametrize("dims", [(13, 8, 11, 6), (7, 9, 5, 12), (17, 21, 19, 23), (9, 7, 6, 33)])
@pytest.mark.parametrize("order,rk", [(3, 3), (2, 2), (1, 3)])
def test_ho4d_irregular_grids(gpu_ctx, oracle, dims, order, rk):
    """The 4D ENO/TVD-RK kernel (k_ho4d: padded layout, axis-0 march,
    chunked planes, odd contiguous extents) against the restatement."""
    from cases import band_np
    n0, n1, n2, n3 = dims
    g = hj.Grid([(-5.0, 5.0, n0), (-2.0, 2.0, n1), (-0.35, 0.35, n2), (-1.5, 1.5, n3)])
    model = configs.planar_model()
    db = hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    cfg = hj.SolveConfig(tolerance=1e-5, max_iters=12, spatial_order=order, time_order=rk)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


def test_ho4d_matches_generic_kernel(gpu_ctx, monkeypatch):
    case = with_iters(workload_case(configs.config2(21)), 10)
    cfg = hj.SolveConfig(**case.cfg.__dict__)
    cfg.spatial_order, cfg.time_order = 3, 3
    fast = hj.solve(case.init_field(), case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
    monkeypatch.setenv("HJB_FAST", "0")
    gen = hj.solve(case.init_field(), case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
    assert same(fast.value.values(), gen.value.values())
    assert same(fast.residual_history, gen.residual_history)


_LF_HO_MODELS = {
    "planar_d0": (lambda: configs.planar_model(), [hj.Interval(-0.5, 0.5)],
                  [(-5.0, 5.0), (-2.0, 2.0), (-0.35, 0.35), (-1.5, 1.5)]),
    "planar_d1": (lambda: hj.NearHoverPlanar4D("x", d_row=1), [hj.Interval(-0.3, 0.7)],
                  [(-5.0, 5.0), (-2.0, 2.0), (-0.35, 0.35), (-1.5, 1.5)]),
    "twin": (lambda: hj.TwinDoubleIntegrator(), [hj.Interval(-0.2, 0.2), hj.Interval(-0.1, 0.3)],
             [(-1.0, 1.0)] * 4),
}


@pytest.mark.parametrize("diss", [hj.PER_NODE, hj.GLOBAL], ids=["per_node", "global"])
@pytest.mark.parametrize("order,rk", [(3, 3), (2, 2), (1, 3)])
@pytest.mark.parametrize("dims", [(13, 8, 11, 6), (7, 9, 5, 12), (5, 3, 4, 7)])
@pytest.mark.parametrize("model", list(_LF_HO_MODELS))
def test_ho4t_lax_friedrichs(gpu_ctx, oracle, diss, order, rk, dims, model):
    """ENO1-3 + TVD-RK with the Lax-Friedrichs Hamiltonian in the TMA-staged
    4D kernel (replicated ghost faces on every axis, per-node / global alpha)
    against the restatement, bitwise."""
    from cases import band_np
    mk, ivs, boxes = _LF_HO_MODELS[model]
    g = hj.Grid([(lo, hi, n) for (lo, hi), n in zip(boxes, dims)])
    db = hj.IntervalField.constant(g, ivs)
    c = hj.ScalarField(g, band_np(g, 0, 0.6 * boxes[0][0], 0.6 * boxes[0][1]))
    cfg = hj.SolveConfig(tolerance=1e-6, max_iters=10, spatial_order=order, time_order=rk,
                         scheme=hj.LAX_FRIEDRICHS, dissipation=diss)
    want = oracle.solve(c, c, mk(), db, cfg)
    got = hj.solve(c, c, mk(), db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


@pytest.mark.parametrize("diss", [hj.PER_NODE, hj.GLOBAL], ids=["per_node", "global"])
def test_ho4t_lax_friedrichs_matches_generic(gpu_ctx, monkeypatch, diss):
    case = with_iters(workload_case(configs.config2(21)), 8)
    cfg = hj.SolveConfig(**case.cfg.__dict__)
    cfg.spatial_order, cfg.time_order = 3, 3
    cfg.scheme, cfg.dissipation = hj.LAX_FRIEDRICHS, diss
    fast = hj.solve(case.init_field(), case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
    monkeypatch.setenv("HJB_FAST", "0")
    gen = hj.solve(case.init_field(), case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
    assert same(fast.value.values(), gen.value.values())
    assert same(fast.residual_history, gen.residual_history)


@pytest.mark.parametrize("model", sorted(_LF_HO_MODELS))
@pytest.mark.parametrize("dims", [(13, 8, 11, 6), (6, 17, 9, 101), (11, 23, 5, 70), (5, 3, 4, 7),
                                  (3, 5, 2, 9)])
def test_eno3g_godunov_shapes(gpu_ctx, oracle, model, dims):
    """k_eno3g (ENO3 Godunov, face-shared choices, edge-patched TMA boxes)
    on every fast-path model shape, multi-segment axis-3 rows and partial
    tiles, against the restatement."""
    mk, bounds, box = _LF_HO_MODELS[model]
    g = hj.Grid([(lo, hi, n) for (lo, hi), n in zip(box, dims)])
    m = mk()
    db = hj.IntervalField.constant(g, bounds)
    rng = np.random.default_rng(sum(dims))
    c = hj.ScalarField(g, rng.random(g.size()) - 0.6)
    init = hj.ScalarField(g, c.values() + 0.3 * rng.random(g.size()))
    cfg = hj.SolveConfig(tolerance=1e-9, max_iters=6, spatial_order=3, time_order=3)
    want = oracle.solve(init, c, m, db, cfg)
    got = hj.solve(init, c, m, db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


def test_eno3g_matches_ho4t(gpu_ctx, monkeypatch):
    """The face-shared ENO3 kernel and the per-cell k_ho4t agree bitwise on
    a config-2 grid large enough for several tiles and plane chunks."""
    case = with_iters(workload_case(configs.config2(41)), 5)
    cfg = hj.SolveConfig(**case.cfg.__dict__)
    cfg.spatial_order, cfg.time_order = 3, 3
    new = hj.solve(case.init_field(), case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
    monkeypatch.setenv("HJB_HO_ENO3G", "0")
    old = hj.solve(case.init_field(), case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
    assert same(new.value.values(), old.value.values())
    assert same(new.residual_history, old.residual_history)
