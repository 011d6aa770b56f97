"""Pin the C restatement (oracle/hj_oracle.c) to the reference itself.

oracle/_ref/libhjref.so is the UNMODIFIED reference sources compiled in place;
every case must agree bitwise (IEEE ==), including iteration counts and
residual histories.  Runs on CPU (`-m "not gpu"`).
"""
import math

import numpy as np
import pytest

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj

from cases import (band_np, quad_setup, same, solve_cases, with_iters, workload_case)


@pytest.mark.parametrize("case,iters", solve_cases(), ids=lambda x: getattr(x, "name", str(x)))
def test_solve_matches_reference(oracle, ref, case, iters):
    case = with_iters(case, iters)
    init, c = case.init_field(), case.c_field()
    a = oracle.solve(init, c, case.model, case.db, case.cfg)
    b = ref.solve(init, c, case.model, case.db, case.cfg)
    assert a.iterations == b.iterations
    assert a.converged == b.converged
    assert a.dt == b.dt
    assert same(a.value.values(), b.value.values())
    assert same(a.residual_history, b.residual_history)


def test_config1_known_answer(oracle):
    """SURVEY.md §6 [probe]: config 1 converges in 146 iterations, dt 4.0912e-3."""
    case = workload_case(configs.config1())
    r = oracle.solve(case.init_field(), case.c_field(), case.model, case.db, case.cfg)
    assert r.converged and r.iterations == 146
    assert abs(r.dt - 4.0912e-3) < 1e-7
    assert int(np.sum(r.value.values() <= 0)) == 4544


@pytest.mark.parametrize("speeds,dims,want", [
    ([10.1], [(0.0, 1.0, 21)], 0.8 / (10.1 / 0.05)),
    ([2.0, 10.1], [(0.0, 1.0, 21), (0.0, 1.4, 21)], 0.8 / (2.0 / 0.05 + 10.1 / 0.07)),
])
def test_cfl_dt_formula(oracle, ref, speeds, dims, want):
    """test_solver.cpp:48-78."""
    g = hj.Grid(dims)
    m = hj.ConstantAdvection(speeds)
    db = hj.IntervalField.constant(g, [])
    a = oracle.cfl_dt(g, m, db, 0.8)
    assert a == ref.cfl_dt(g, m, db, 0.8)
    assert a == pytest.approx(want, rel=1e-12)


def test_cfl_zero_flow_and_halving(oracle, ref):
    from oracle.oracle import OracleError
    m = hj.ConstantAdvection([0.0])
    g = hj.Grid([(0.0, 1.0, 11)])
    with pytest.raises(OracleError) as e1:
        oracle.cfl_dt(g, m, hj.IntervalField.constant(g, []), 0.8)
    with pytest.raises(OracleError) as e2:
        ref.cfl_dt(g, m, hj.IntervalField.constant(g, []), 0.8)
    assert e1.value.code == e2.value.code == 2
    m = hj.ConstantAdvection([1.0])
    g21, g41 = hj.Grid([(0.0, 1.0, 21)]), hj.Grid([(0.0, 1.0, 41)])
    d1 = oracle.cfl_dt(g21, m, hj.IntervalField.constant(g21, []), 0.8)
    d2 = oracle.cfl_dt(g41, m, hj.IntervalField.constant(g41, []), 0.8)
    assert d2 == pytest.approx(d1 / 2, rel=1e-12)


@pytest.mark.parametrize("scheme", [hj.GODUNOV, hj.LAX_FRIEDRICHS])
def test_vi_step_matches_reference(oracle, ref, scheme):
    case = quad_setup(31)
    case.cfg.scheme = scheme
    rng = np.random.default_rng(3)
    v = hj.ScalarField(case.grid, case.c + 0.3 * rng.random(case.grid.size()))
    dt = oracle.cfl_dt(case.grid, case.model, case.db, 0.8)
    a = oracle.vi_step(v, case.c_field(), case.model, case.db, dt, case.cfg)
    b = ref.vi_step(v, case.c_field(), case.model, case.db, dt, case.cfg)
    assert same(a, b)


def test_vi_step_linear_transport_and_clamp(oracle):
    """test_solver.cpp:80-111 known answers."""
    from oracle.oracle import OracleError
    m = hj.ConstantAdvection([1.0])
    g = hj.Grid([(0.0, 1.0, 11)])
    db = hj.IntervalField.constant(g, [])
    dt = oracle.cfl_dt(g, m, db, 0.8)
    v = hj.ScalarField(g, g.coords(0))
    c = hj.ScalarField(g, fill=-100.0)
    lf = hj.SolveConfig(scheme=hj.LAX_FRIEDRICHS)
    nxt = oracle.vi_step(v, c, m, db, dt, lf)
    assert np.allclose(nxt, v.values() + dt, rtol=1e-12, atol=0)
    nxt_g = oracle.vi_step(v, c, m, db, dt)
    assert np.allclose(nxt_g[1:-1], v.values()[1:-1] + dt, rtol=1e-12, atol=0)
    cc = hj.ScalarField(g, -g.coords(0))
    assert same(oracle.vi_step(cc, cc, m, db, dt), cc.values())
    with pytest.raises(OracleError) as e:
        oracle.vi_step(v, c, m, db, 10 * dt)
    assert e.value.code == 1


def test_resample_seed_jump_match_reference(oracle, ref):
    rng = np.random.default_rng(11)
    src_g = configs.planar_grid(7)
    dst_g = configs.planar_grid(13)
    f = hj.ScalarField(src_g, rng.standard_normal(src_g.size()))
    assert same(oracle.resample(f, dst_g), ref.resample(f, dst_g))
    back = hj.ScalarField(dst_g, oracle.resample(f, dst_g))
    assert same(oracle.resample(back, src_g), ref.resample(back, src_g))
    assert oracle.max_adjacent_jump(f) == ref.max_adjacent_jump(f)
    g2 = hj.Grid([(0.1, 0.9, 6), (0.2, 0.8, 12)])
    f2 = hj.ScalarField(hj.Grid([(0, 1, 9), (0, 1, 9)]), rng.random(81))
    assert same(oracle.resample(f2, g2), ref.resample(f2, g2))


def test_levelset_matches_reference(oracle, ref):
    g = configs.planar_grid(9)
    assert same(oracle.signed_distance_band(g, 0, -4.0, 4.0), ref.signed_distance_band(g, 0, -4.0, 4.0))
    assert same(oracle.signed_distance_band(g, 0, -4.0, 4.0), band_np(g, 0, -4.0, 4.0))
    g2 = hj.Grid([(-2, 2, 41), (-2, 2, 41)])
    lo, hi = [-0.8, -1.2], [1.1, 0.4]
    assert same(oracle.signed_distance_box(g2, lo, hi), ref.signed_distance_box(g2, lo, hi))


def test_coarse_to_fine_matches_reference(oracle, ref):
    case = quad_setup(41)
    coarse = hj.Grid([(0.0, 3.2, 21), (-5.0, 5.0, 21)])
    a = oracle.solve_coarse_to_fine(case.c_field(), case.model, case.db, coarse, case.cfg)
    b = ref.solve_coarse_to_fine(case.c_field(), case.model, case.db, coarse, case.cfg)
    for x, y in ((a.coarse, b.coarse), (a.fine, b.fine)):
        assert x.iterations == y.iterations
        assert same(x.value.values(), y.value.values())
    warm = a.fine.value
    case2 = quad_setup(41, dbar=0.4)
    a = oracle.solve_coarse_to_fine(case2.c_field(), case2.model, case2.db, coarse, case2.cfg, warm)
    b = ref.solve_coarse_to_fine(case2.c_field(), case2.model, case2.db, coarse, case2.cfg, warm)
    assert a.fine.iterations == b.fine.iterations
    assert same(a.fine.value.values(), b.fine.value.values())


def test_hamiltonian_and_flow_bounds_probes(oracle, ref):
    """test_dynamics.cpp:124-199 restated: oracle == reference on random probes."""
    rng = np.random.default_rng(3)
    db1 = [hj.Interval(-0.4, 0.25)]
    db2 = [hj.Interval(-0.4, 0.25), hj.Interval(-0.1, 0.5)]
    models = [(hj.Quad2DVert(), db1), (hj.NearHoverPlanar4D("x"), db1),
              (hj.NearHoverPlanar4D("x", d_row=0), db1), (hj.TwinDoubleIntegrator(), db2),
              (hj.NearHoverVertical2D(), db1), (hj.DoubleIntegrator(), db1)]
    for m, db in models:
        for _ in range(100):
            x = rng.uniform(-1, 1, m.state_dim())
            p = rng.uniform(-1, 1, m.state_dim())
            assert oracle.hamiltonian(m, x, p, db) == ref.hamiltonian(m, x, p, db)
            assert same(oracle.flow_bounds(m, x, db), ref.flow_bounds(m, x, db))
    # known answers (test_dynamics.cpp:124-134, 168-181)
    q = hj.Quad2DVert()
    db = [hj.Interval(-0.3, 0.3)]
    assert oracle.hamiltonian(q, [1.0, 2.0], [0.0, 1.0], db) == pytest.approx(-9.8 + 0.3)
    assert oracle.hamiltonian(q, [1.0, 2.0], [1.0, 0.0], db) == pytest.approx(2.0)
    a = oracle.flow_bounds(q, [1.0, 2.0], db)
    assert a[1] == pytest.approx(10.1) and a[0] == pytest.approx(2.0)
    a = oracle.flow_bounds(hj.NearHoverPlanar4D("x"), [0, 0, 0, 0], db)
    assert a[3] == pytest.approx(10.0 * 0.2443)


def test_multilevel_two_levels_is_coarse_to_fine(oracle, ref):
    """hjo_solve_multilevel with 2 levels == the reference's solve_coarse_to_fine."""
    q = quad_setup(41)
    coarse = hj.Grid([(0.0, 3.2, 21), (-5.0, 5.0, 21)])
    a = oracle.solve_multilevel(q.c_field(), q.model, q.db, [coarse], q.cfg)
    b = ref.solve_coarse_to_fine(q.c_field(), q.model, q.db, coarse, q.cfg)
    for x, y in zip(a.levels, (b.coarse, b.fine)):
        assert x.iterations == y.iterations
        assert same(x.value.values(), y.value.values())
