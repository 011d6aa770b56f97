"""GP bounds, CPU side: the oracle restatement of
GpModel::predict / bounds_on_grid (oracle/hj_oracle.c) against the
reference's own known-answer tests (proj/tests/test_gp.cpp, restated), and
the library's host GpModel::fit (hjb_gp_fit) against a numpy restatement of
gp.cpp:43-186.

Parity status: gp.cpp needs Eigen, which is absent from this image, so the
reference GP cannot be compiled here — the restatement is
pinned by the reference's known-answer tests below, not by the reference
binary.
"""
import math

import numpy as np
import pytest

from paper_2101_05916_b200 import hjsafe as hj

from gp_cases import bump_samples, factor_model, numpy_fit


def test_prior_only_bounds_are_3_sigma_exactly(oracle):
    """test_gp.cpp:111-121."""
    m = hj.GpModel.prior(hj.GpHyperparams(0.01, [1.0], 0.0))
    g = hj.Grid([(0.0, 3.0, 11)])
    lo, hi = oracle.gp_bounds_on_grid([m], [[0]], g)
    assert np.all(np.abs(lo[0] + 0.3) <= 1e-12 * 0.3)
    assert np.all(np.abs(hi[0] - 0.3) <= 1e-12 * 0.3)


def test_noise_free_single_point_is_interpolated(oracle):
    """test_gp.cpp:37-44."""
    m = factor_model(hj.GpHyperparams(1.0, [0.5], 0.0), [[0.3]], [1.0])
    mean, var = oracle.gp_predict(m, [[0.3]])
    assert mean[0] == pytest.approx(1.0, rel=1e-6)
    assert var[0] == pytest.approx(0.0, abs=1e-6)


def test_far_from_data_reverts_to_prior(oracle):
    """test_gp.cpp:46-53."""
    m = factor_model(hj.GpHyperparams(0.04, [0.5], 1e-4), [[0.0]], [1.0])
    mean, var = oracle.gp_predict(m, [[40.0]])
    assert mean[0] == pytest.approx(0.0, abs=1e-9)
    assert var[0] == pytest.approx(0.04, rel=1e-9)


def test_zero_noise_point_collapses_band(oracle):
    """test_gp.cpp:123-133."""
    m = factor_model(hj.GpHyperparams(0.04, [0.5], 0.0), [[1.0]], [1.0])
    g = hj.Grid([(0.0, 2.0, 5)])
    lo, hi = oracle.gp_bounds_on_grid([m], [[0]], g)
    assert lo[0][2] == pytest.approx(1.0, rel=1e-4)
    assert hi[0][2] == pytest.approx(1.0, rel=1e-4)


def test_symmetric_data_even_mean(oracle):
    """test_gp.cpp:69-79."""
    xs, ys = [], []
    for x in (0.4, 1.0, 1.7):
        xs += [[x], [-x]]
        ys += [0.8, 0.8]
    m = factor_model(hj.GpHyperparams(0.5, [0.7], 1e-3), xs, ys)
    for x in (0.2, 0.9, 1.5, 2.5):
        a, _ = oracle.gp_predict(m, [[x]])
        b, _ = oracle.gp_predict(m, [[-x]])
        assert a[0] == pytest.approx(b[0], rel=1e-9)


def test_variance_bounds(oracle):
    """test_gp.cpp:81-99: latent variance at training points <= noise,
    posterior variance <= prior variance everywhere."""
    X, y = bump_samples(60, 0.1, 3)
    hp = hj.GpHyperparams(0.25, [0.6], 0.01)
    m = factor_model(hp, X, y)
    _, v = oracle.gp_predict(m, X[:10])
    assert np.all(v <= hp.noise_var + 1e-9)
    X2, y2 = bump_samples(120, 0.05, 7)
    hp2 = hj.GpHyperparams(0.09, [0.4], 0.002)
    m2 = factor_model(hp2, X2, y2)
    q = np.random.default_rng(23).uniform(-4.0, 4.0, size=(1000, 1))
    _, v2 = oracle.gp_predict(m2, q)
    assert np.all(v2 <= hp2.signal_var + 1e-12)


def test_datum_shrinks_band(oracle):
    """test_gp.cpp:101-109."""
    hp = hj.GpHyperparams(0.09, [0.5], 0.004)
    base_x, base_y = [[0.0], [-0.5]], [0.1, 0.2]
    a = factor_model(hp, base_x, base_y)
    b = factor_model(hp, base_x + [[1.0]], base_y + [0.15])
    _, va = oracle.gp_predict(a, [[1.0]])
    _, vb = oracle.gp_predict(b, [[1.0]])
    assert vb[0] <= va[0] + 1e-12


def test_bounds_are_per_node_predict(oracle):
    """bounds_on_grid == predict at each node's input coordinates."""
    X, y = bump_samples(40, 0.05, 11)
    X2 = np.hstack([X, np.random.default_rng(4).uniform(-1, 1, size=(40, 1))])
    m = factor_model(hj.GpHyperparams(0.2, [0.5, 0.7], 0.003), X2, y)
    g = hj.Grid([(-2.0, 2.0, 5), (-1.0, 1.0, 4), (0.0, 1.0, 3)])
    lo, hi = oracle.gp_bounds_on_grid([m], [[0, 2]], g, confidence=2.5)
    for lin in range(g.size()):
        idx = g.unravel(lin)
        x = [g.coord(0, idx[0]), g.coord(2, idx[2])]
        mu, var = oracle.gp_predict(m, [x])
        band = 2.5 * math.sqrt(var[0] + 0.003)
        assert lo[0][lin] == mu[0] - band and hi[0][lin] == mu[0] + band


def test_oracle_errors(oracle):
    from oracle.oracle import OracleError
    m = hj.GpModel.prior(hj.GpHyperparams(0.01, [1.0], 0.0))
    g = hj.Grid([(0.0, 1.0, 3)])
    with pytest.raises(OracleError, match="input dim out of grid range"):
        oracle.gp_bounds_on_grid([m], [[1]], g)
    with pytest.raises(OracleError, match="does not match GP"):
        oracle.gp_bounds_on_grid([m], [[0, 0]], g)


# ----------------------------------------------------------- host fit
@pytest.mark.parametrize("policy", [hj.gp_module.SEARCH, hj.gp_module.FIXED])
def test_fit_matches_numpy_restatement(policy):
    X, y = bump_samples(200, 0.05, 17)
    cfg = hj.GpConfig(policy=policy, prior=hj.GpHyperparams(0.09, [0.4], 0.002))
    m = hj.GpModel.fit([hj.DisturbanceMeasurement(list(x), v) for x, v in zip(X, y)], cfg)
    want = numpy_fit(X, y, cfg)
    hp = m.hyperparams()
    # same candidate chosen (y_sd sums in a different order in numpy)
    assert hp.signal_var == pytest.approx(want["hp"].signal_var, rel=1e-12)
    assert hp.noise_var == pytest.approx(want["hp"].noise_var, rel=1e-12)
    assert hp.lengthscales == pytest.approx(want["hp"].lengthscales, rel=1e-12)
    np.testing.assert_allclose(m._chol, want["L"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(m._alpha, want["alpha"], rtol=1e-9, atol=1e-9)
    assert m.log_marginal_likelihood() == pytest.approx(want["lml"], rel=1e-10)


def test_fit_subsamples_to_max_training():
    X, y = bump_samples(700, 0.05, 5)
    cfg = hj.GpConfig(policy=hj.gp_module.FIXED, prior=hj.GpHyperparams(0.09, [0.4], 0.002),
                      max_training=300)
    m = hj.GpModel.fit([hj.DisturbanceMeasurement(list(x), v) for x, v in zip(X, y)], cfg)
    assert m.training_count() == 300
    idx = [(i * 699) // 299 for i in range(300)]  # gp.cpp:52-53
    assert np.array_equal(m._inputs[:, 0], X[idx, 0])


def test_fit_errors():
    with pytest.raises(hj.InvalidArgument, match="need at least one measurement"):
        hj.GpModel.fit([])
    with pytest.raises(hj.InvalidArgument, match="non-finite value"):
        hj.GpModel.fit([hj.DisturbanceMeasurement([0.0], float("nan"))])
    with pytest.raises(hj.InvalidArgument, match="lengthscale count"):
        hj.GpModel.fit([hj.DisturbanceMeasurement([0.0, 1.0], 1.0)],
                       hj.GpConfig(policy=hj.gp_module.FIXED))
    with pytest.raises(hj.InvalidArgument, match="signal variance"):
        hj.GpModel.prior(hj.GpHyperparams(0.0, [1.0], 0.0))
