"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bitwise (IEEE ==) values, identical iteration counts and residual histories,
on the same seeded inputs (BASELINE.json north_star: |dV| <= 1e-9, identical
signs, identical iteration count — bitwise equality implies all three).
"""
import numpy as np
import pytest

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj

from cases import (band_np, fmax_np, per_node_case, quad_setup, same, solve_cases, with_iters,
                   workload_case)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case,iters", solve_cases(), ids=lambda x: getattr(x, "name", str(x)))
def test_solve_matches_oracle(gpu_ctx, oracle, case, iters):
    case = with_iters(case, iters)
    init, c = case.init_field(), case.c_field()
    want = oracle.solve(init, c, case.model, case.db, case.cfg)
    got = hj.solve(init, c, case.model, case.db, case.cfg, ctx=gpu_ctx)
    assert got.dt == want.dt
    assert got.iterations == want.iterations
    assert got.converged == want.converged
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


def test_config1_converges_like_reference(gpu_ctx):
    case = workload_case(configs.config1())
    r = hj.solve(case.init_field(), case.c_field(), case.model, case.db, case.cfg, ctx=gpu_ctx)
    assert r.converged and r.iterations == 146
    assert int(np.sum(r.value.values() <= 0)) == 4544


@pytest.mark.parametrize("order", [1, 3])
def test_solve_with_one_field_as_init_and_constraint(gpu_ctx, oracle, order):
    """hjb_solve copies an aliased init/constraint (the reference's cold
    solve(c, c, ...), sim.cpp:282) once; the result is the two-buffer one,
    and the host field is left untouched."""
    case = with_iters(workload_case(configs.config2(13)), 40)
    cfg = hj.SolveConfig(**case.cfg.__dict__)
    cfg.spatial_order = cfg.time_order = order
    c = case.c_field()
    before = c.values().copy()
    want = oracle.solve(case.init_field(), case.c_field(), case.model, case.db, cfg)
    got = hj.solve(c, c, case.model, case.db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations == 40
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())
    assert np.array_equal(c.values(), before)


@pytest.mark.parametrize("n,iters", [(21, 200), (51, 10)])
def test_config2_k_iterations(gpu_ctx, oracle, n, iters):
    case = with_iters(workload_case(configs.config2(n)), iters)
    init, c = case.init_field(), case.c_field()
    want = oracle.solve(init, c, case.model, case.db, case.cfg)
    got = hj.solve(init, c, case.model, case.db, case.cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations == iters
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


@pytest.mark.parametrize("scheme,diss", [(hj.GODUNOV, hj.PER_NODE), (hj.LAX_FRIEDRICHS, hj.PER_NODE),
                                         (hj.LAX_FRIEDRICHS, hj.GLOBAL)])
def test_vi_step_matches_oracle(gpu_ctx, oracle, scheme, diss):
    for case in (quad_setup(31), per_node_case(17), workload_case(configs.config2(9))):
        case.cfg.scheme = scheme
        case.cfg.dissipation = diss
        rng = np.random.default_rng(5)
        v = hj.ScalarField(case.grid, case.c + 0.3 * rng.random(case.grid.size()))
        dt = oracle.cfl_dt(case.grid, case.model, case.db, 0.8)
        assert hj.cfl_dt(case.grid, case.model, case.db, 0.8, ctx=gpu_ctx) == dt
        want = oracle.vi_step(v, case.c_field(), case.model, case.db, dt, case.cfg)
        got = hj.vi_step(v, case.c_field(), case.model, case.db, dt, case.cfg, ctx=gpu_ctx)
        assert same(got.values(), want), case.name


def test_errors_match_reference(gpu_ctx):
    m = hj.ConstantAdvection([0.0])
    g = hj.Grid([(0.0, 1.0, 11)])
    db = hj.IntervalField.constant(g, [])
    with pytest.raises(hj.SolverRuntimeError):
        hj.cfl_dt(g, m, db, 0.8, ctx=gpu_ctx)
    m = hj.ConstantAdvection([1.0])
    dt = hj.cfl_dt(g, m, db, 0.8, ctx=gpu_ctx)
    v = hj.ScalarField(g, g.coords(0))
    c = hj.ScalarField(g, fill=-100.0)
    with pytest.raises(hj.InvalidArgument):
        hj.vi_step(v, c, m, db, 10 * dt, ctx=gpu_ctx)
    with pytest.raises(hj.InvalidArgument):
        hj.solve(v, c, m, db, hj.SolveConfig(cfl_factor=1.5), ctx=gpu_ctx)
    with pytest.raises(hj.InvalidArgument):
        hj.solve(v, c, m, db, hj.SolveConfig(tolerance=0.0), ctx=gpu_ctx)
    q = quad_setup(11)
    with pytest.raises(hj.InvalidArgument):  # rank mismatch
        hj.solve(v, c, q.model, hj.IntervalField.constant(g, [hj.Interval(-1, 1)]), ctx=gpu_ctx)


def test_resample_seed_jump_match_oracle(gpu_ctx, oracle):
    rng = np.random.default_rng(11)
    src_g, dst_g = configs.planar_grid(7), configs.planar_grid(13)
    f = hj.ScalarField(src_g, rng.standard_normal(src_g.size()))
    assert same(hj.resample(f, dst_g, ctx=gpu_ctx).values(), oracle.resample(f, dst_g))
    assert hj.max_adjacent_jump(f, ctx=gpu_ctx) == oracle.max_adjacent_jump(f)
    c = hj.ScalarField(dst_g, band_np(dst_g, 0, -4.0, 4.0))
    assert same(hj.seed_from(f, dst_g, c, ctx=gpu_ctx).values(), oracle.seed_from(f, dst_g, c))
    g = configs.planar_grid(9)
    assert same(hj.signed_distance_band(g, 0, -4.0, 4.0, ctx=gpu_ctx).values(),
                oracle.signed_distance_band(g, 0, -4.0, 4.0))


def test_coarse_to_fine_matches_oracle(gpu_ctx, oracle):
    case = quad_setup(41)
    coarse = hj.Grid([(0.0, 3.2, 21), (-5.0, 5.0, 21)])
    want = oracle.solve_coarse_to_fine(case.c_field(), case.model, case.db, coarse, case.cfg)
    got = hj.solve_coarse_to_fine(case.c_field(), case.model, case.db, coarse, case.cfg, ctx=gpu_ctx)
    for x, y in ((got.coarse, want.coarse), (got.fine, want.fine)):
        assert x.iterations == y.iterations
        assert same(x.value.values(), y.value.values())
    warm = got.fine.value
    case2 = quad_setup(41, dbar=0.4)
    want = oracle.solve_coarse_to_fine(case2.c_field(), case2.model, case2.db, coarse, case2.cfg, warm)
    got = hj.solve_coarse_to_fine(case2.c_field(), case2.model, case2.db, coarse, case2.cfg, warm,
                                  ctx=gpu_ctx)
    assert got.fine.iterations == want.fine.iterations
    assert same(got.fine.value.values(), want.fine.value.values())


def test_determinism_and_invariants_101(gpu_ctx):
    """Size-independent properties at the config-3 size (101^4): two runs are
    bitwise identical, V >= c exactly, cold evolution is non-decreasing."""
    w = configs.config3(101, max_iters=3)
    case = workload_case(w)
    init, c = case.init_field(), case.c_field()
    r1 = hj.solve(init, c, case.model, case.db, case.cfg, ctx=gpu_ctx)
    r2 = hj.solve(init, c, case.model, case.db, case.cfg, ctx=gpu_ctx)
    assert same(r1.value.values(), r2.value.values())
    assert same(r1.residual_history, r2.residual_history)
    v = r1.value.values()
    assert np.all(v >= case.c)
    assert np.all(v >= init.values() - 1e-12)


@pytest.mark.parametrize("dims", [(13, 8, 11, 6), (7, 9, 5, 12), (17, 21, 19, 23), (33, 5, 6, 101)])
def test_fast4d_irregular_grids(gpu_ctx, oracle, dims):
    """Odd/even contiguous extents, partial tiles and chunked marches of the
    specialised 4D kernel against the oracle."""
    n0, n1, n2, n3 = dims
    g = hj.Grid([(-5.0, 5.0, n0), (-2.0, 2.0, n1), (-0.35, 0.35, n2), (-1.5, 1.5, n3)])
    model = configs.planar_model()
    db = hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=40)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


def test_fast4d_matches_generic_kernel(gpu_ctx, monkeypatch):
    """The specialised kernel and the generic one produce identical bits."""
    case = with_iters(workload_case(configs.config2(21)), 30)
    init, c = case.init_field(), case.c_field()
    fast = hj.solve(init, c, case.model, case.db, case.cfg, ctx=gpu_ctx)
    monkeypatch.setenv("HJB_FAST", "0")
    gen = hj.solve(init, c, case.model, case.db, case.cfg, ctx=gpu_ctx)
    assert same(fast.value.values(), gen.value.values())
    assert same(fast.residual_history, gen.residual_history)


def test_multilevel_three_levels_matches_oracle(gpu_ctx, oracle):
    """Config-5 style 3-level chain (obstacles, wind 0.6) at reduced size:
    7^4 -> 13^4 -> 25^4, bitwise per level."""
    ws = configs.config5(levels=(7, 13, 25), tol=5e-3)
    fine = ws[-1]
    c = hj.ScalarField(fine.grid, fine.constraint(band_np, fmax_np))
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=300)
    want = oracle.solve_multilevel(c, fine.model, fine.dbounds(), [w.grid for w in ws[:-1]], cfg)
    got = hj.solve_multilevel(c, fine.model, fine.dbounds(), [w.grid for w in ws[:-1]], cfg,
                              ctx=gpu_ctx)
    for x, y in zip(got.levels, want.levels):
        assert x.iterations == y.iterations
        assert same(x.residual_history, y.residual_history)
        assert same(x.value.values(), y.value.values())


@pytest.mark.parametrize("fast", ["1", "0"])
def test_nan_cell_never_wins_the_residual(gpu_ctx, monkeypatch, fast):
    """A NaN in V (possible only through unchecked inputs) is skipped by the
    max|dV| reduction as by the reference's `if (dv > max_dv)`
    (solver.cpp:181-182); the fast kernel takes its rescan path here.  The
    NaN node itself is clamped to c (std::max(c, NaN) == c)."""
    monkeypatch.setenv("HJB_FAST", fast)
    case = with_iters(workload_case(configs.config2(13)), 1)
    rng = np.random.default_rng(11)
    v0 = case.c + 0.25 * rng.random(case.grid.size())
    k = case.grid.linear_index((6, 6, 6, 6))
    v0[k] = np.nan
    init = hj.ScalarField(case.grid, v0, check=False)
    r = hj.solve(init, case.c_field(), case.model, case.db, case.cfg, ctx=gpu_ctx)
    out = r.value.values()
    assert out[k] == case.c[k]
    dv = np.abs(out - v0)
    want = dv[np.isfinite(dv)].max() / r.dt
    assert r.iterations == 1 and r.residual_history[0] == want


@pytest.mark.parametrize("nch,tab_global", [("1", "0"), ("3", "0"), ("7", "1"), ("13", "0")])
def test_fast4d_item_schedule_and_tables(gpu_ctx, oracle, monkeypatch, nch, tab_global):
    """The persistent kernel's work items (tile x chunk of planes, dynamic
    schedule) and both slope-table paths (shared-memory staged / global)
    give the oracle's bits; chunk counts that do not divide the axis."""
    monkeypatch.setenv("HJB_NCH", nch)
    monkeypatch.setenv("HJB_TAB_GLOBAL", tab_global)
    g = hj.Grid([(-5.0, 5.0, 29), (-2.0, 2.0, 13), (-0.35, 0.35, 11), (-1.5, 1.5, 9)])
    model = configs.planar_model()
    db = hj.IntervalField.constant(g, [hj.Interval(-0.7, 0.3)])
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=25)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


@pytest.mark.parametrize("wind", [(0.0, 0.0), (-3.0, -2.5), (2.5, 3.0), (-0.2, 0.9)])
def test_fast4d_slope_shapes(gpu_ctx, oracle, wind):
    """Disturbance intervals that make the wind row non-decreasing,
    non-increasing, V-shaped or linear over the whole grid (every Godunov
    shape branch of the fast kernel) against the oracle."""
    g = hj.Grid([(-5.0, 5.0, 15), (-2.0, 2.0, 9), (-0.35, 0.35, 7), (-1.5, 1.5, 11)])
    model = configs.planar_model()
    db = hj.IntervalField.constant(g, [hj.Interval(*wind)])
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    cfg = hj.SolveConfig(tolerance=1e-5, max_iters=30)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


@pytest.mark.parametrize("dims", [(2, 2, 2, 2), (2, 3, 2, 3), (3, 2, 5, 2), (5, 4, 3, 7)])
@pytest.mark.parametrize("order,rk", [(1, 1), (3, 3), (2, 2)])
def test_smallest_grids(gpu_ctx, oracle, dims, order, rk):
    """Two-node axes: every face is an edge face (ghost rule everywhere), the
    stencil halo exceeds the grid, one-tile / one-plane marches."""
    n0, n1, n2, n3 = dims
    g = hj.Grid([(-5.0, 5.0, n0), (-2.0, 2.0, n1), (-0.35, 0.35, n2), (-1.5, 1.5, n3)])
    model = configs.planar_model()
    db = hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0) + 0.01 * np.arange(g.size()) / g.size())
    cfg = hj.SolveConfig(tolerance=1e-6, max_iters=25, spatial_order=order, time_order=rk)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


def test_max_iters_zero_and_time_horizon(gpu_ctx, oracle):
    case = workload_case(configs.config2(9))
    init = hj.ScalarField(case.grid, case.c + 0.1)
    cfg = hj.SolveConfig(tolerance=1e-6, max_iters=0)
    got = hj.solve(init, case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
    want = oracle.solve(init, case.c_field(), case.model, case.db, cfg)
    assert got.iterations == want.iterations == 0
    assert same(got.value.values(), init.values())
    for order in (1, 2, 3):
        cfg = hj.SolveConfig(tolerance=1e-9, max_iters=1000, time_horizon=0.05,
                             spatial_order=order, time_order=order)
        want = oracle.solve(case.c_field(), case.c_field(), case.model, case.db, cfg)
        got = hj.solve(case.c_field(), case.c_field(), case.model, case.db, cfg, ctx=gpu_ctx)
        assert got.iterations == want.iterations < 1000
        assert got.iterations * got.dt >= 0.05 > (got.iterations - 1) * got.dt
        assert same(got.value.values(), want.value.values())


def _lf_models():
    return [("planar_d0", configs.planar_model(), [hj.Interval(-0.5, 0.5)]),
            ("planar_d1", hj.NearHoverPlanar4D("x", d_row=1), [hj.Interval(-0.3, 0.7)]),
            ("twin", hj.TwinDoubleIntegrator(), [hj.Interval(-0.2, 0.2), hj.Interval(-0.1, 0.3)])]


@pytest.mark.parametrize("diss", [hj.PER_NODE, hj.GLOBAL], ids=["per_node", "global"])
@pytest.mark.parametrize("dims", [(13, 8, 11, 6), (7, 9, 5, 12), (17, 21, 19, 23)])
@pytest.mark.parametrize("which", [0, 1, 2], ids=["planar_d0", "planar_d1", "twin"])
def test_fast4d_lax_friedrichs(gpu_ctx, oracle, diss, dims, which):
    """The Lax-Friedrichs variants of the specialised 4D kernel (per-node and
    global dissipation, every row shape) against the oracle, bitwise."""
    name, model, ivs = _lf_models()[which]
    n0, n1, n2, n3 = dims
    if name == "twin":
        g = hj.Grid([(-1.0, 1.0, n0), (-1.0, 1.0, n1), (-1.0, 1.0, n2), (-1.0, 1.0, n3)])
    else:
        g = hj.Grid([(-5.0, 5.0, n0), (-2.0, 2.0, n1), (-0.35, 0.35, n2), (-1.5, 1.5, n3)])
    db = hj.IntervalField.constant(g, ivs)
    c = hj.ScalarField(g, band_np(g, 0, -0.6 * g.dims()[0].max, 0.6 * g.dims()[0].max))
    cfg = hj.SolveConfig(tolerance=1e-6, max_iters=40, scheme=hj.LAX_FRIEDRICHS, dissipation=diss)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.dt == want.dt
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


@pytest.mark.parametrize("diss", [hj.PER_NODE, hj.GLOBAL], ids=["per_node", "global"])
def test_fast4d_lax_friedrichs_matches_generic(gpu_ctx, monkeypatch, diss):
    """Config-2 model on 31^4 with the LF scheme: specialised kernel == generic kernel."""
    case = with_iters(workload_case(configs.config2(31)), 60)
    case.cfg.scheme = hj.LAX_FRIEDRICHS
    case.cfg.dissipation = diss
    init, c = case.init_field(), case.c_field()
    fast = hj.solve(init, c, case.model, case.db, case.cfg, ctx=gpu_ctx)
    monkeypatch.setenv("HJB_FAST", "0")
    gen = hj.solve(init, c, case.model, case.db, case.cfg, ctx=gpu_ctx)
    assert fast.iterations == gen.iterations == 60
    assert same(fast.value.values(), gen.value.values())
    assert same(fast.residual_history, gen.residual_history)


def _axis0_bounds(g, specs, seed=7, break_node=None):
    """Per-node IntervalField varying along axis 0 only (GP bounds over x):
    one (center, half-width) profile per channel."""
    rng = np.random.default_rng(seed)
    n0 = g.dim(0).n
    s0 = g.size() // n0
    lo, hi = [], []
    for (c, w) in specs:
        mid = c + 0.3 * np.sin(np.linspace(0.0, 3.0, n0)) + 0.05 * rng.standard_normal(n0)
        half = w * (1.0 + 0.5 * rng.random(n0))
        lo.append(np.repeat(mid - half, s0))
        hi.append(np.repeat(mid + half, s0))
    if break_node is not None:
        lo[0][break_node] -= 1e-3
    return hj.IntervalField(g, len(specs), lo=lo, hi=hi)


PV_CASES = [
    ("planar_d0", lambda: configs.planar_model(), [(0.0, 0.5)],
     [(-5.0, 5.0, 15), (-2.0, 2.0, 9), (-0.35, 0.35, 7), (-1.5, 1.5, 11)]),
    ("planar_d1", lambda: hj.NearHoverPlanar4D("x", d_row=1), [(0.1, 0.4)],
     [(-5.0, 5.0, 13), (-2.0, 2.0, 8), (-0.35, 0.35, 9), (-1.5, 1.5, 6)]),
    ("twin", lambda: hj.TwinDoubleIntegrator(), [(0.0, 0.15), (0.05, 0.1)],
     [(-2.5, 2.5, 11), (-3.0, 3.0, 9), (-2.5, 2.5, 7), (-3.0, 3.0, 13)]),
]


@pytest.mark.parametrize("case", PV_CASES, ids=[c[0] for c in PV_CASES])
@pytest.mark.parametrize("broken", [False, True], ids=["axis0", "not_axis0"])
def test_fast4d_axis0_varying_bounds(gpu_ctx, oracle, monkeypatch, case, broken):
    """Per-node bounds varying along axis 0 only (the sim's GP bounds) run the
    specialised kernel's plane-varying variant; a field that is not a
    function of x0 alone falls back to the generic kernel.  Both bitwise equal
    to the oracle and to HJB_FAST=0."""
    _, mk, specs, dims = case
    g = hj.Grid(dims)
    model = mk()
    db = _axis0_bounds(g, specs, break_node=(g.size() // 2) if broken else None)
    c = hj.ScalarField(g, band_np(g, 0, -0.6 * g.dims()[0].max, 0.6 * g.dims()[0].max))
    cfg = hj.SolveConfig(tolerance=1e-6, max_iters=40)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())
    monkeypatch.setenv("HJB_FAST", "0")
    gen = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert same(gen.value.values(), got.value.values())


@pytest.mark.parametrize("balance", ["0", "1"], ids=["dynamic_items", "static_balanced"])
@pytest.mark.parametrize("dims", [(17, 21, 19, 23), (31, 9, 7, 12)])
def test_fast4d_schedules(gpu_ctx, oracle, monkeypatch, balance, dims):
    """Both CTA schedules of k_fast4d (dynamic tile x chunk items; static
    balanced tile-plane ranges, pieces spanning tiles) against the oracle."""
    monkeypatch.setenv("HJB_BALANCE", balance)
    n0, n1, n2, n3 = dims
    g = hj.Grid([(-5.0, 5.0, n0), (-2.0, 2.0, n1), (-0.35, 0.35, n2), (-1.5, 1.5, n3)])
    model = configs.planar_model()
    db = hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    cfg = hj.SolveConfig(tolerance=1e-5, max_iters=30)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


@pytest.mark.parametrize("case", PV_CASES, ids=[c[0] for c in PV_CASES])
@pytest.mark.parametrize("spread", [0.05, 1.0], ids=["narrow", "sign_mixing"])
def test_fast4d_per_node_bounds(gpu_ctx, oracle, monkeypatch, case, spread):
    """Per-node bounds varying in every axis (e.g. a resampled constant field
    with rounding noise, or GP bounds over several axes) run k_fast4d's
    per-node variant (slopes and slope shapes of the disturbance rows formed
    per cell and plane); bitwise equal to the oracle and to HJB_PN=0 (the
    generic kernel).  `sign_mixing` makes the row shapes differ cell to cell."""
    _, mk, specs, dims = case
    g = hj.Grid(dims)
    model = mk()
    rng = np.random.default_rng(11)
    lo, hi = [], []
    for (cen, w) in specs:
        a = cen + spread * (rng.random(g.size()) - 0.5)
        b = a + w * rng.random(g.size())
        lo.append(a)
        hi.append(b)
    db = hj.IntervalField(g, len(specs), lo=lo, hi=hi)
    c = hj.ScalarField(g, band_np(g, 0, -0.6 * g.dims()[0].max, 0.6 * g.dims()[0].max))
    cfg = hj.SolveConfig(tolerance=1e-6, max_iters=40)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())
    monkeypatch.setenv("HJB_PN", "0")
    gen = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert same(gen.value.values(), got.value.values())


@pytest.mark.parametrize("order,rk", [(1, 1), (3, 3)])
def test_constraint_plane_table_matches_field(gpu_ctx, oracle, monkeypatch, order, rk):
    """A constraint that varies along axis 0 only (every BASELINE 4D config)
    is read from a per-plane table; the result equals the per-node path
    (HJB_CPLANE=0) and the oracle bitwise."""
    case = with_iters(workload_case(configs.config2(23)), 12)
    cfg = hj.SolveConfig(**case.cfg.__dict__)
    cfg.spatial_order, cfg.time_order = order, rk
    init, c = case.init_field(), case.c_field()
    monkeypatch.setenv("HJB_CPLANE", "1")
    got = hj.solve(init, c, case.model, case.db, cfg, ctx=gpu_ctx)
    want = oracle.solve(init, c, case.model, case.db, cfg)
    assert same(got.value.values(), want.value.values())
    assert same(got.residual_history, want.residual_history)
    monkeypatch.setenv("HJB_CPLANE", "0")
    per_node = hj.solve(init, c, case.model, case.db, cfg, ctx=gpu_ctx)
    assert same(per_node.value.values(), got.value.values())


def test_concurrent_first_launches_in_fresh_process():
    """Several host threads (one context each, the reference's concurrent
    subsystem jobs, sim.cpp:340-363) launching the TMA kernels for the first
    time in a fresh process: the per-device kernel attributes must be set
    before any of them launches."""
    import subprocess
    import sys
    from pathlib import Path
    code = r'''
import sys, threading
sys.path.insert(0, sys.argv[1])
from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj
w = configs.config2(21)
ctxs = [hj.Context(0) for _ in range(4)]
errs = []
gate = threading.Barrier(4)
def job(k):
    try:
        cfg = hj.SolveConfig(**w.cfg.__dict__)
        cfg.max_iters = 5
        if k % 2:
            cfg.spatial_order, cfg.time_order = 3, 3
        c = hj.signed_distance_band(w.grid, 0, -4.0, 4.0, ctx=ctxs[k])
        gate.wait()  # every thread reaches its first TMA-kernel launch together
        hj.solve(c, c, w.model, w.dbounds(), cfg, ctx=ctxs[k])
    except Exception as e:
        errs.append(repr(e))
th = [threading.Thread(target=job, args=(k,)) for k in range(4)]
[t.start() for t in th]
[t.join() for t in th]
assert not errs, errs
print("ok")
'''
    root = str(Path(__file__).resolve().parent.parent)
    for _ in range(3):  # a fresh process each time: the attributes start unset
        r = subprocess.run([sys.executable, "-c", code, root], capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_result_reports_the_kernel_family(gpu_ctx):
    """A solve says which kernel family ran it (a model outside the 4D fast
    path's shapes falls to the generic kernel: reported, not silent)."""
    from paper_2101_05916_b200 import configs
    w = configs.config2(21)
    c = hj.signed_distance_band(w.grid, 0, -4.0, 4.0, ctx=gpu_ctx)
    cfg = hj.SolveConfig(max_iters=3)
    assert hj.solve(c, c, w.model, w.dbounds(), cfg, ctx=gpu_ctx).kernel == "fast4d_multisweep"
    w5 = configs.config2(61)
    c5 = hj.signed_distance_band(w5.grid, 0, -4.0, 4.0, ctx=gpu_ctx)
    assert hj.solve(c5, c5, w5.model, w5.dbounds(), cfg, ctx=gpu_ctx).kernel == "fast4d"
    w1 = configs.config1()
    c1 = hj.signed_distance_band(w1.grid, 0, 0.0, 3.0, ctx=gpu_ctx)
    assert hj.solve(c1, c1, w1.model, w1.dbounds(), cfg, ctx=gpu_ctx).kernel == "small2d"
    g3 = hj.Grid([(0.0, 1.0, 9), (0.0, 1.0, 9), (0.0, 1.0, 9)])
    adv = hj.ConstantAdvection([1.0, 0.5, -0.25])
    c3 = hj.ScalarField(g3, np.zeros(g3.size()))
    db3 = hj.IntervalField.constant(g3, [])
    assert hj.solve(c3, c3, adv, db3, cfg, ctx=gpu_ctx).kernel == "generic"
    cfg.spatial_order, cfg.time_order = 3, 3
    assert hj.solve(c, c, w.model, w.dbounds(), cfg, ctx=gpu_ctx).kernel == "ho4d"
