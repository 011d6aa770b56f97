"""ENO2/ENO3 + TVD-RK2/RK3 restatement (oracle/hj_oracle.c).  PARITY UNPINNED:
the reference has no high-order scheme, so the restatement is
validated by (i) exact reduction to the reference update at order 1 / Euler,
(ii) convergence order on smooth advection, (iii) sign agreement with the
first-order reference solution away from the zero level set."""
import math

import numpy as np
import pytest

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj

from cases import quad_setup, same, with_iters, workload_case

FORCE_HO = 1


@pytest.mark.parametrize("scheme,diss", [(hj.GODUNOV, hj.PER_NODE), (hj.LAX_FRIEDRICHS, hj.PER_NODE),
                                         (hj.LAX_FRIEDRICHS, hj.GLOBAL)])
def test_stage_machinery_reduces_to_reference(oracle, ref, scheme, diss):
    for case in (with_iters(quad_setup(21), 120), with_iters(workload_case(configs.config2(9)), 30)):
        case.cfg.scheme, case.cfg.dissipation = scheme, diss
        want = ref.solve(case.init_field(), case.c_field(), case.model, case.db, case.cfg)
        cfg = hj.SolveConfig(**case.cfg.__dict__)
        cfg.flags = FORCE_HO
        got = oracle.solve(case.init_field(), case.c_field(), case.model, case.db, cfg)
        assert got.iterations == want.iterations
        assert same(got.value.values(), want.value.values())
        assert same(got.residual_history, want.residual_history)


def _advection_error(oracle, n, order, rk, scheme=hj.GODUNOV):
    g = hj.Grid([(0.0, 2.0, n)])
    x = g.coords(0)
    v0 = np.sin(math.pi * x) + 0.5 * np.cos(2 * math.pi * x)
    m = hj.ConstantAdvection([1.0])
    db = hj.IntervalField.constant(g, [])
    cfg = hj.SolveConfig(cfl_factor=0.5, tolerance=1e-300, max_iters=100000, spatial_order=order,
                         time_order=rk, time_horizon=0.25, scheme=scheme)
    r = oracle.solve(hj.ScalarField(g, v0), hj.ScalarField(g, fill=-100.0), m, db, cfg)
    t = r.iterations * r.dt
    exact = np.sin(math.pi * (x + t)) + 0.5 * np.cos(2 * math.pi * (x + t))
    mask = (x > 0.3) & (x < 1.2)
    return float(np.max(np.abs(r.value.values() - exact)[mask]))


@pytest.mark.parametrize("order,rk,min_rate", [(1, 1, 0.8), (2, 2, 1.7), (3, 3, 2.5)])
def test_convergence_order_on_smooth_advection(oracle, order, rk, min_rate):
    errs = [_advection_error(oracle, n, order, rk) for n in (41, 81, 161)]
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert min(rates) >= min_rate, (errs, rates)


def test_lf_high_order_converges_too(oracle):
    errs = [_advection_error(oracle, n, 2, 2, hj.LAX_FRIEDRICHS) for n in (41, 81, 161)]
    assert math.log2(errs[1] / errs[2]) >= 1.5, errs


def test_eno2_rk2_config1_safe_set_agrees_with_reference(oracle):
    """BASELINE config 1 names ENO2 + TVD-RK2: its safe set agrees with the
    first-order reference solution except within a cell of the boundary."""
    case = workload_case(configs.config1())
    first = oracle.solve(case.init_field(), case.c_field(), case.model, case.db, case.cfg)
    cfg = hj.SolveConfig(**case.cfg.__dict__)
    cfg.spatial_order, cfg.time_order = 2, 2
    ho = oracle.solve(case.init_field(), case.c_field(), case.model, case.db, cfg)
    assert ho.converged
    a = first.value.array() <= 0
    b = ho.value.array() <= 0
    diff = a != b
    # every disagreement touches the first-order zero level set
    near = np.zeros_like(diff)
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            near |= np.roll(np.roll(a, di, 0), dj, 1) != a
    assert not np.any(diff & ~near)
    assert np.all(ho.value.values() >= case.c)
