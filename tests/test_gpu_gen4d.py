"""GPU parity of the run-time-shape 4D sweep (k_fast4d<ShapeGen>) against the
CPU oracle: user models whose rows fit the fast path's structure (one-axis
rows with any inputs, input-free two-term rows, nothing on x0) but none of
the compiled shapes.  Before this variant such models ran the generic
one-thread-per-node kernel (~3.5x slower per cell).

Bitwise (IEEE ==) values, identical iteration counts and residual histories
(the update is update_chunk, proj/src/solver.cpp:106-190, term by term).
"""
import numpy as np
import pytest

from paper_2101_05916_b200 import abi
from paper_2101_05916_b200 import hjsafe as hj

from cases import band_np, same

pytestmark = pytest.mark.gpu

C_, T_, K_ = abi.TERM_COORD, abi.TERM_TAN, abi.TERM_CONST


def mixed_model():
    """Rows: x3 + d | -2 x2 + 0.5 x3 | 9.8 tan x2 | -1.5 x1 + 4 u (a one-axis
    row with a disturbance, a two-term linear row, a linear tan row and a
    control row; row axes 3, (2, 3), 2, 1)."""
    B = np.zeros((4, 1))
    B[3, 0] = 4.0
    Cm = np.zeros((4, 1))
    Cm[0, 0] = 1.0
    return hj.SeparableAffineModel(
        [[(C_, 3, 1.0)], [(C_, 2, -2.0), (C_, 3, 0.5)], [(T_, 2, 9.8)], [(C_, 1, -1.5)]],
        B, Cm, [hj.Interval(-0.4, 0.4)])


def inputs_model():
    """Two controls and two disturbances on rows 1 and 3, drifts over axes
    2, 3, 1 and a constant row: x2 | x3 + u0 + d0 | -0.7 x1 | -9.8 + u1 - d1."""
    B = np.zeros((4, 2))
    B[1, 0] = 1.0
    B[3, 1] = 2.5
    Cm = np.zeros((4, 2))
    Cm[1, 0] = 1.0
    Cm[3, 1] = -0.5
    return hj.SeparableAffineModel(
        [[(C_, 2, 1.0)], [(C_, 3, 1.0)], [(C_, 1, -0.7)], [(K_, 0, -9.8)]],
        B, Cm, [hj.Interval(-1.0, 1.0), hj.Interval(0.0, 8.0)])


def advection_model():
    """Constant drifts only (every row a table of length one)."""
    return hj.ConstantAdvection([1.0, -0.5, 0.25, 0.75])


def x0_model():
    """Rows on the march axis x0 (re-formed every plane): 2 x1 + 0.05 u |
    x0 + 0.3 x3 | -0.4 x0 + d | x1  (a two-term row on (x0, x3), a one-axis
    x0 row with a disturbance; no row depends on its own axis, as Godunov
    requires, solver.cpp:293-295)."""
    B = np.zeros((4, 1))
    B[0, 0] = 0.05
    Cm = np.zeros((4, 1))
    Cm[2, 0] = 1.0
    return hj.SeparableAffineModel(
        [[(C_, 1, 2.0)], [(C_, 0, 1.0), (C_, 3, 0.3)], [(C_, 0, -0.4)], [(C_, 1, 1.0)]],
        B, Cm, [hj.Interval(-1.0, 1.0)])


MODELS = {"mixed": (mixed_model, 1), "inputs": (inputs_model, 2), "advection": (advection_model, 0),
          "x0rows": (x0_model, 1)}


def _setup(name, dims):
    make, nd = MODELS[name]
    n0, n1, n2, n3 = dims
    g = hj.Grid([(-5.0, 5.0, n0), (-2.0, 2.0, n1), (-0.35, 0.35, n2), (-1.5, 1.5, n3)])
    db = hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)] * nd)
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    return g, make(), db, c


def _check(got, want):
    assert got.dt == want.dt
    assert got.iterations == want.iterations
    assert got.converged == want.converged
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


@pytest.mark.parametrize("ms", ["0", "1"])
@pytest.mark.parametrize("dims", [(13, 8, 11, 6), (9, 21, 19, 23), (17, 12, 10, 40),
                                  (33, 5, 6, 101)])
@pytest.mark.parametrize("name", sorted(MODELS))
def test_gen4d_matches_oracle(gpu_ctx, oracle, monkeypatch, name, dims, ms):
    """Irregular grids (odd / even contiguous extents, partial tiles, chunked
    marches), per-sweep launches (HJB_MS=0) and the multi-sweep persistent
    launch, against the oracle."""
    monkeypatch.setenv("HJB_MS", ms)
    g, model, db, c = _setup(name, dims)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=40)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.kernel == ("fast4d_multisweep" if ms == "1" else "fast4d_gen")
    _check(got, want)


@pytest.mark.parametrize("diss", ["per_node", "global"])
@pytest.mark.parametrize("dims", [(13, 8, 11, 6), (9, 21, 19, 23), (33, 5, 6, 101)])
@pytest.mark.parametrize("name", sorted(MODELS))
def test_gen4d_lax_friedrichs_matches_oracle(gpu_ctx, oracle, name, dims, diss):
    """Lax-Friedrichs on the run-time-shape variant (per-node / global alpha,
    the rows' input channels read at run time) against the oracle."""
    g, model, db, c = _setup(name, dims)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=30, scheme=hj.LAX_FRIEDRICHS,
                         dissipation=hj.GLOBAL if diss == "global" else hj.PER_NODE)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.kernel == "fast4d_gen"
    _check(got, want)


def test_gen4d_lax_friedrichs_shared_channel(gpu_ctx, oracle):
    """One disturbance channel entering two rows (LfParams::single = 0): the
    channel's coefficient is summed over its rows in row order."""
    B = np.zeros((4, 1))
    B[3, 0] = 2.0
    Cm = np.zeros((4, 1))
    Cm[0, 0] = 1.0
    Cm[2, 0] = -0.5
    model = hj.SeparableAffineModel(
        [[(C_, 1, 1.0)], [(C_, 3, -0.7)], [(C_, 3, 1.0)], [(C_, 1, -1.0)]], B, Cm,
        [hj.Interval(-1.0, 1.0)])
    g = hj.Grid([(-5.0, 5.0, 13), (-2.0, 2.0, 11), (-0.35, 0.35, 9), (-1.5, 1.5, 14)])
    db = hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    for diss in (hj.PER_NODE, hj.GLOBAL):
        cfg = hj.SolveConfig(tolerance=1e-4, max_iters=30, scheme=hj.LAX_FRIEDRICHS,
                             dissipation=diss)
        got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
        assert got.kernel == "fast4d_gen"
        _check(got, oracle.solve(c, c, model, db, cfg))


@pytest.mark.parametrize("P", [2, 3])
def test_gen4d_lax_friedrichs_sharded(gpu_ctx, P):
    """The slab-partitioned LF solve (in-process ranks) on the run-time-shape
    variant equals the single-GPU solve bit for bit."""
    import torch
    from paper_2101_05916_b200 import sharded
    g, model, db, c = _setup("inputs", (21, 13, 11, 17))
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=40, scheme=hj.LAX_FRIEDRICHS)
    ref = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert ref.kernel == "fast4d_gen"
    ct = torch.tensor(c.values(), device="cuda")
    out = torch.full_like(ct, float("nan"))
    torch.cuda.synchronize()
    r = sharded.solve_sharded_local_dev(P, g, model, db, ct.data_ptr(), ct.data_ptr(),
                                        out.data_ptr(), cfg, gpu_ctx, history_capacity=40)
    assert r.iterations == ref.iterations and r.dt == ref.dt
    assert same(out.cpu().numpy(), ref.value.values())


@pytest.mark.parametrize("name", sorted(MODELS))
def test_gen4d_to_convergence(gpu_ctx, oracle, monkeypatch, name):
    """A whole solve to convergence: identical iteration count (north_star)."""
    monkeypatch.setenv("HJB_MS", "0")
    g, model, db, c = _setup(name, (15, 13, 11, 17))
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=6000)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert want.converged
    _check(got, want)


@pytest.mark.parametrize("name", sorted(MODELS))
def test_gen4d_matches_generic_kernel(gpu_ctx, monkeypatch, name):
    """Run-time-shape variant == generic kernel (HJB_FAST=0), bit for bit, on
    a grid large enough for the autotuned per-sweep path."""
    monkeypatch.setenv("HJB_MS", "0")
    g, model, db, c = _setup(name, (41, 41, 41, 41))
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=25)
    fast = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert fast.kernel == "fast4d_gen"
    monkeypatch.setenv("HJB_FAST", "0")
    gen = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert gen.kernel == "generic"
    assert same(fast.value.values(), gen.value.values())
    assert same(fast.residual_history, gen.residual_history)


def test_gen4d_outside_scope_falls_back(gpu_ctx, oracle):
    """ENO/TVD-RK with rows on x0 stays on the generic stage kernel, and so
    does LF for a row with two input terms (still bitwise against the
    oracle)."""
    g = hj.Grid([(-5.0, 5.0, 11), (-2.0, 2.0, 9), (-0.35, 0.35, 7), (-1.5, 1.5, 8)])
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=20)
    model, db = mixed_model(), hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    B2 = np.zeros((4, 2))
    B2[3, 0], B2[3, 1] = 1.0, 0.5
    two = hj.SeparableAffineModel(
        [[(C_, 1, 1.0)], [(C_, 3, -0.7)], [(C_, 3, 1.0)], [(C_, 1, -1.0)]], B2, None,
        [hj.Interval(-1.0, 1.0), hj.Interval(-0.5, 0.5)])
    db0 = hj.IntervalField.constant(g, [])
    lf = hj.SolveConfig(tolerance=1e-4, max_iters=20, scheme=hj.LAX_FRIEDRICHS)
    got = hj.solve(c, c, two, db0, lf, ctx=gpu_ctx)
    assert got.kernel == "generic"
    _check(got, oracle.solve(c, c, two, db0, lf))
    ho = hj.SolveConfig(tolerance=1e-4, max_iters=10, spatial_order=3, time_order=3)
    xm, xdb = x0_model(), hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    got = hj.solve(c, c, xm, xdb, ho, ctx=gpu_ctx)
    assert got.kernel == "ho_generic"  # rows on x0: the stage kernels march x0
    _check(got, oracle.solve(c, c, xm, xdb, ho))



@pytest.mark.parametrize("P", [2, 3])
def test_gen4d_sharded_local_ranks_equal_solve(gpu_ctx, monkeypatch, P):
    """The slab-partitioned solve (in-process ranks: the NCCL path's per-rank
    plans, halo offsets and boundary-first launches) with the run-time-shape
    variant equals the single-GPU solve bit for bit."""
    import torch
    from paper_2101_05916_b200 import sharded
    monkeypatch.setenv("HJB_MS", "0")
    g, model, db, c = _setup("mixed", (21, 13, 11, 17))
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=60)
    ref = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert ref.kernel == "fast4d_gen"
    ct = torch.tensor(c.values(), device="cuda")
    out = torch.full_like(ct, float("nan"))
    torch.cuda.synchronize()
    r = sharded.solve_sharded_local_dev(P, g, model, db, ct.data_ptr(), ct.data_ptr(),
                                        out.data_ptr(), cfg, gpu_ctx, history_capacity=60)
    assert r.iterations == ref.iterations and r.dt == ref.dt
    assert same(r.residual_history, ref.residual_history)
    assert same(out.cpu().numpy(), ref.value.values())


def test_gen4d_x0_rows_not_sharded(gpu_ctx):
    """A row on the slab axis x0 is rejected by the slab-partitioned solve
    (local plane numbers would index the x0 tables) with Unsupported."""
    import torch
    from paper_2101_05916_b200 import sharded
    g, model, db, c = _setup("x0rows", (12, 7, 6, 8))
    ct = torch.tensor(c.values(), device="cuda")
    out = torch.empty_like(ct)
    with pytest.raises(hj.Unsupported):
        sharded.solve_sharded_local_dev(2, g, model, db, ct.data_ptr(), ct.data_ptr(),
                                        out.data_ptr(), hj.SolveConfig(max_iters=5), gpu_ctx)


@pytest.mark.parametrize("name", sorted(MODELS))
def test_gen4d_target_set(gpu_ctx, oracle, name):
    """Reach-avoid update max(c, min(l, stepped)) on the run-time-shape
    variant (the target-set instantiation) against the restatement."""
    g, model, db, c = _setup(name, (13, 11, 9, 14))
    tl = hj.ScalarField(g, band_np(g, 1, -1.0, 1.0))
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=30)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx, target=tl)
    assert got.kernel == "fast4d_gen"
    _check(got, oracle.solve(c, c, model, db, cfg, target=tl))


def _per_node_db(g, nd, kind, seed=5):
    """Per-node bounds for nd channels: 'axis0' varies along x0 only (the
    plane-varying variant), 'mixed' varies at every node with lo / hi of
    both signs (slopes whose shapes change cell to cell)."""
    rng = np.random.default_rng(seed)
    lo, hi = [], []
    shape = g.shape
    for _ in range(nd):
        if kind == "axis0":
            base = -0.5 + 0.2 * rng.random(shape[0])
            a = np.broadcast_to(base.reshape(-1, 1, 1, 1), shape).reshape(-1).copy()
            b = a + 0.3 + 0.4 * np.broadcast_to(rng.random(shape[0]).reshape(-1, 1, 1, 1),
                                                shape).reshape(-1)
        else:
            a = -0.4 + 0.8 * (rng.random(g.size()) - 0.5)
            b = a + 0.6 * rng.random(g.size())
        lo.append(a)
        hi.append(b)
    return hj.IntervalField(g, nd, lo=lo, hi=hi)


@pytest.mark.parametrize("kind", ["axis0", "mixed"])
@pytest.mark.parametrize("dims", [(13, 8, 11, 6), (9, 21, 19, 23)])
@pytest.mark.parametrize("name", ["mixed", "inputs", "x0rows"])
def test_gen4d_per_node_bounds(gpu_ctx, oracle, monkeypatch, name, dims, kind):
    """Per-node disturbance bounds (plane-varying and every-node) on the
    run-time-shape variant: a disturbance row's slopes are (drift + controls)
    + max / min of its products per cell and plane; bitwise vs the oracle and
    vs the generic kernel (HJB_PN=0)."""
    make, nd = MODELS[name]
    n0, n1, n2, n3 = dims
    g = hj.Grid([(-5.0, 5.0, n0), (-2.0, 2.0, n1), (-0.35, 0.35, n2), (-1.5, 1.5, n3)])
    model = make()
    db = _per_node_db(g, nd, kind)
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    cfg = hj.SolveConfig(tolerance=1e-6, max_iters=30)
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.kernel == "fast4d_gen"
    _check(got, want)
    monkeypatch.setenv("HJB_PN", "0")
    gen = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert same(gen.value.values(), got.value.values())


@pytest.mark.parametrize("scheme", ["gd", "lf"])
@pytest.mark.parametrize("order,rk", [(1, 2), (2, 2), (3, 3)])
@pytest.mark.parametrize("dims", [(9, 21, 19, 23), (17, 12, 10, 40)])
@pytest.mark.parametrize("name", ["mixed", "inputs", "advection"])
def test_gen4d_high_order_matches_oracle(gpu_ctx, oracle, name, dims, order, rk, scheme):
    """ENO1-3 + TVD-RK2/3 stages on the run-time-shape k_ho4t (Godunov: the
    reference flux per axis from hhat = 0.0; LF: run-time channels) against
    the CPU restatement, bitwise."""
    g, model, db, c = _setup(name, dims)
    cfg = hj.SolveConfig(tolerance=1e-4, max_iters=12, spatial_order=order, time_order=rk)
    if scheme == "lf":
        cfg.scheme = hj.LAX_FRIEDRICHS
    want = oracle.solve(c, c, model, db, cfg)
    got = hj.solve(c, c, model, db, cfg, ctx=gpu_ctx)
    assert got.kernel == "ho4d"
    _check(got, want)
