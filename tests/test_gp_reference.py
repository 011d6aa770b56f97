"""GP bounds pinned to the REFERENCE: the reference's own
GpModel::predict and bounds_on_grid (proj/src/gp.cpp:188-249, compiled in
place into oracle/_ref/libhjref_gp.so) against the C restatement the device
kernels are tested on (oracle/hj_oracle.c hjo_gp_*), bitwise, on the same
fitted factors.  The reference's fit needs Eigen (absent), so the factors
come from the product's own host fit (hjb_gp_fit) or numpy; both sides read
the same factor.  CPU only; the device comparison is in test_gpu_gp.py."""
import numpy as np
import pytest

from paper_2101_05916_b200 import hjsafe as hj

from cases import same
from gp_cases import GRID_CASES, bump_samples, fitted


@pytest.mark.parametrize("case", GRID_CASES, ids=[c[0] for c in GRID_CASES])
def test_restatement_bounds_match_reference(oracle, ref_gp, case):
    _, dims, mk, idims = case
    g = hj.Grid(dims)
    models = mk()
    for conf in (3.0, 1.5):
        want_lo, want_hi = ref_gp.gp_bounds_on_grid(models, idims, g, confidence=conf)
        got_lo, got_hi = oracle.gp_bounds_on_grid(models, idims, g, confidence=conf)
        for ch in range(len(models)):
            assert same(got_lo[ch], want_lo[ch]) and same(got_hi[ch], want_hi[ch])


@pytest.mark.parametrize("n,dims", [(0, 1), (1, 1), (60, 1), (300, 1), (80, 2), (45, 3)])
def test_restatement_predict_matches_reference(oracle, ref_gp, n, dims):
    if n == 0:
        m = hj.GpModel.prior(hj.GpHyperparams(0.02, [0.7] * dims, 0.001))
    else:
        m = fitted(n, 7 + n, dims=dims)
    X = np.random.default_rng(n).uniform(-2.5, 2.5, size=(97, dims))
    X[0] = m._inputs[0] if n else 0.0  # on a training point
    want = ref_gp.gp_predict(m, X)
    got = oracle.gp_predict(m, X)
    assert same(got[0], want[0]) and same(got[1], want[1])


@pytest.mark.parametrize("policy", ["search", "fixed"])
def test_product_fit_through_reference_bounds(oracle, ref_gp, policy):
    """The product's host fit (hjb_gp_fit) on the reference test's bump data
    (test_gp.cpp:20-33 shape), bounds by the reference's own loops vs the
    restatement; and the reference's coverage expectation on that data."""
    X, y = bump_samples(200, 0.05, 21)
    data = [hj.DisturbanceMeasurement([float(x)], float(v)) for x, v in zip(X[:, 0], y)]
    cfg = hj.GpConfig(policy=policy, prior=hj.GpHyperparams(0.09, [0.4], 0.002))
    m = hj.GpModel.fit(data, cfg)
    g = hj.Grid([(-2.0, 2.0, 41), (-1.0, 1.0, 3)])
    want_lo, want_hi = ref_gp.gp_bounds_on_grid([m], [[0]], g, 3.0)
    got_lo, got_hi = oracle.gp_bounds_on_grid([m], [[0]], g, 3.0)
    assert same(got_lo[0], want_lo[0]) and same(got_hi[0], want_hi[0])
    xs = g.coords(0)
    truth = np.repeat(0.5 * np.exp(-xs * xs), 3)
    assert np.all((want_lo[0] <= truth) & (truth <= want_hi[0]))


def test_reference_errors_match_restatement(oracle, ref_gp):
    from oracle.oracle import OracleError
    g = hj.Grid([(-2.0, 2.0, 9), (-1.0, 1.0, 5)])
    m = fitted(20, 3)
    for models, idims, msg in (
            ([m], [[0, 1]], "bounds_on_grid: input-dim map does not match GP"),
            ([m], [[2]], "bounds_on_grid: input dim out of grid range")):
        with pytest.raises(OracleError, match=msg):
            ref_gp.gp_bounds_on_grid(models, idims, g)
        with pytest.raises(Exception, match=msg):
            oracle.gp_bounds_on_grid(models, idims, g)
    bad = hj.GpModel.prior(hj.GpHyperparams(1.0, [1.0], 0.0))
    bad._hp = hj.GpHyperparams(-1.0, [1.0], 0.0)
    with pytest.raises(OracleError, match="GP: signal variance must be > 0"):
        ref_gp.gp_bounds_on_grid([bad], [[0]], g)  # the product's message: test_gpu_gp.py
