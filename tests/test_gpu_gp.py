"""GP bounds on the device against the oracle restatement,
bitwise: hjb_gp_bounds_on_grid[_dev] / hjb_gp_predict_batch, the reference's
GP known-answer tests through the product API, and the GP -> solve chain of
run_update_job (sim.cpp:339-363)."""
import numpy as np
import pytest
import torch

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj

from cases import band_np, same
from gp_cases import GRID_CASES as CASES, bump_samples, factor_model, fitted as _fitted

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_bounds_on_grid_matches_oracle(gpu_ctx, oracle, case):
    _, dims, mk, idims = case
    g = hj.Grid(dims)
    models = mk()
    want_lo, want_hi = oracle.gp_bounds_on_grid(models, idims, g, confidence=3.0)
    got = hj.bounds_on_grid(models, idims, g, 3.0, ctx=gpu_ctx)
    for ch in range(len(models)):
        assert same(got.lo(ch).values(), want_lo[ch])
        assert same(got.hi(ch).values(), want_hi[ch])


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_bounds_on_grid_matches_reference(gpu_ctx, ref_gp, case):
    """The device kernels against the REFERENCE's own bounds_on_grid
    (gp.cpp:211-249 via oracle/_ref/libhjref_gp.so), bitwise."""
    _, dims, mk, idims = case
    g = hj.Grid(dims)
    models = mk()
    want_lo, want_hi = ref_gp.gp_bounds_on_grid(models, idims, g, confidence=3.0)
    got = hj.bounds_on_grid(models, idims, g, 3.0, ctx=gpu_ctx)
    for ch in range(len(models)):
        assert same(got.lo(ch).values(), want_lo[ch])
        assert same(got.hi(ch).values(), want_hi[ch])


def test_predict_and_fit_through_reference(gpu_ctx, ref_gp):
    """Product host fit -> device predict_batch / bounds vs the reference's
    predict and bounds_on_grid on the same factor; hyperparameter errors
    carry the reference's messages."""
    X, y = bump_samples(250, 0.05, 33)
    data = [hj.DisturbanceMeasurement([float(a)], float(b)) for a, b in zip(X[:, 0], y)]
    m = hj.GpModel.fit(data, hj.GpConfig())
    Q = np.random.default_rng(4).uniform(-3, 3, size=(300, 1))
    want = ref_gp.gp_predict(m, Q)
    got = m.predict_batch(Q, ctx=gpu_ctx)
    assert same(np.asarray(got[0]), want[0]) and same(np.asarray(got[1]), want[1])
    g = configs.planar_grid(21)
    want_lo, want_hi = ref_gp.gp_bounds_on_grid([m], [[0]], g, 3.0)
    b = hj.bounds_on_grid([m], [[0]], g, 3.0, ctx=gpu_ctx)
    assert same(b.lo(0).values(), want_lo[0]) and same(b.hi(0).values(), want_hi[0])
    from oracle.oracle import OracleError
    for hp, msg in ((hj.GpHyperparams(-1.0, [1.0], 0.0), "GP: signal variance must be > 0"),
                    (hj.GpHyperparams(1.0, [1.0], -1.0), "GP: noise variance must be >= 0"),
                    (hj.GpHyperparams(1.0, [0.0], 0.0), "GP: lengthscales must be > 0")):
        bad = hj.GpModel.prior(hj.GpHyperparams(1.0, [1.0], 0.0))
        bad._hp = hp
        with pytest.raises(OracleError, match=msg):
            ref_gp.gp_bounds_on_grid([bad], [[0]], g)
        with pytest.raises(hj.InvalidArgument, match=msg):
            hj.bounds_on_grid([bad], [[0]], g, ctx=gpu_ctx)


def test_bounds_on_grid_dev_into_torch(gpu_ctx, oracle):
    g = configs.planar_grid(21)
    m = _fitted(300, 101)
    lo = torch.empty(g.size(), dtype=torch.float64, device="cuda")
    hi = torch.empty_like(lo)
    torch.cuda.synchronize()
    hj.bounds_on_grid_dev([m], [[0]], g, [lo.data_ptr()], [hi.data_ptr()], 3.0, ctx=gpu_ctx)
    gpu_ctx.synchronize()
    wl, wh = oracle.gp_bounds_on_grid([m], [[0]], g)
    assert same(lo.cpu().numpy(), wl[0]) and same(hi.cpu().numpy(), wh[0])


@pytest.mark.parametrize("n", [1, 32, 37, 300, 500, 1024, 2100])
def test_predict_batch_matches_oracle(gpu_ctx, oracle, n):
    m = _fitted(n, 40 + n) if n > 1 else factor_model(hj.GpHyperparams(0.04, [0.5], 1e-4),
                                                      [[0.0]], [1.0])
    q = np.random.default_rng(n).uniform(-3.0, 3.0, size=(257, 1))
    mean, var = m.predict_batch(q, ctx=gpu_ctx)
    wm, wv = oracle.gp_predict(m, q)
    assert same(mean, wm) and same(var, wv)


def test_reference_known_answers_through_product(gpu_ctx):
    """test_gp.cpp:55-67 (bump tracked within 0.1 after a hyper search) and
    :135-147 (the 3-sigma band covers >= 99 % of held-out samples, through
    violation_check)."""
    X, y = bump_samples(200, 0.05, 17)
    m = hj.GpModel.fit([hj.DisturbanceMeasurement(list(x), v) for x, v in zip(X, y)])
    xs = np.arange(-2.0, 2.0 + 1e-9, 0.1)
    mean, _ = m.predict_batch(xs.reshape(-1, 1), ctx=gpu_ctx)
    assert np.all(np.abs(mean - 0.5 * np.exp(-xs * xs)) < 0.1)
    assert m.predict([0.0], ctx=gpu_ctx).mean == pytest.approx(0.5, rel=0.2)

    Xt, yt = bump_samples(300, 0.05, 101)
    mt = hj.GpModel.fit([hj.DisturbanceMeasurement(list(x), v) for x, v in zip(Xt, yt)])
    g = hj.Grid([(-2.0, 2.0, 81)])
    b = hj.bounds_on_grid([mt], [[0]], g, ctx=gpu_ctx)
    Xh, yh = bump_samples(1000, 0.05, 202)
    lo = np.interp(Xh[:, 0], g.coords(0), b.lo(0).values())
    hi = np.interp(Xh[:, 0], g.coords(0), b.hi(0).values())
    assert np.mean((yh >= lo) & (yh <= hi)) >= 0.99
    vc = hj.violation_check(b, 0, [float(Xh[0, 0])], float(yh[0]), ctx=gpu_ctx)
    assert vc.inside == bool(yh[0] >= lo[0] and yh[0] <= hi[0])
    assert vc.margin == pytest.approx(min(yh[0] - lo[0], hi[0] - yh[0]), abs=1e-12)


def test_gp_bounds_feed_solve(gpu_ctx, oracle):
    """run_update_job (sim.cpp:339-363): GP bounds on the subsystem grid, then
    a warm solve with the per-node IntervalField, against the oracle chain."""
    g = hj.Grid([(-5.0, 5.0, 15), (-2.0, 2.0, 9), (-0.35, 0.35, 7), (-1.5, 1.5, 11)])
    X = np.random.default_rng(3).uniform(-5.0, 5.0, size=(120, 1))
    y = 0.3 * np.sin(X[:, 0]) + np.random.default_rng(4).normal(0.0, 0.05, size=120)
    m = hj.GpModel.fit([hj.DisturbanceMeasurement(list(x), v) for x, v in zip(X, y)])
    db = hj.bounds_on_grid([m], [[0]], g, 3.0, ctx=gpu_ctx)
    wl, wh = oracle.gp_bounds_on_grid([m], [[0]], g, 3.0)
    assert same(db.lo(0).values(), wl[0]) and same(db.hi(0).values(), wh[0])
    model = configs.planar_model()
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=30)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


def test_errors(gpu_ctx):
    g = hj.Grid([(0.0, 1.0, 3)])
    m = hj.GpModel.prior(hj.GpHyperparams(0.01, [1.0], 0.0))
    with pytest.raises(hj.InvalidArgument, match="input dim out of grid range"):
        hj.bounds_on_grid([m], [[1]], g, ctx=gpu_ctx)
    with pytest.raises(hj.InvalidArgument, match="does not match GP"):
        hj.bounds_on_grid([m], [[0, 0]], g, ctx=gpu_ctx)
    with pytest.raises(hj.InvalidArgument, match="one input-dim map per channel"):
        hj.bounds_on_grid([m], [[0], [0]], g, ctx=gpu_ctx)
