"""Target set (reach-avoid) — B200 extension named by BASELINE.json's
north_star ("min/max against the target and avoid sets").  The reference
has no target set: its update clamps against the avoid set only,
V' = max(c, stepped) (proj/src/solver.cpp:178-179), so parity is UNPINNED by
construction.  The extension's update is

    V' = max(c, min(l, stepped))      (std::min(stepped, l), then the clamp)

applied after every Euler step and every TVD-RK stage.  These tests pin the
C restatement (oracle/hj_oracle.c) to that formula with numpy, and to the
reference where the target is inactive; the GPU tests pin the device kernels
(k_fast4d TG variant, generic k_step / k_ho_stage) to the restatement bit
for bit.
"""
import numpy as np
import pytest
import torch

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj

from cases import band_np, fmax_np, same


def _cfg2(n=11):
    w = configs.config2(n)
    g = w.grid
    c = band_np(g, 0, -4.0, 4.0)
    # target: the box x in [2.5, 3.5], |vx| <= 1 as a signed distance (< 0
    # inside), next to the avoid set's edge where the avoid-only V* > 0
    l = fmax_np(band_np(g, 0, 2.5, 3.5), band_np(g, 1, -1.0, 1.0))
    return w, g, c, l


def test_restatement_update_formula(oracle):
    """One step with a target = numpy max(c, min(l, stepped)) where stepped
    is the same step without any clamp (c = -1e300)."""
    w, g, c, l = _cfg2(9)
    rng = np.random.default_rng(3)
    v = c + 4.0 * rng.random(g.size())  # above l inside the target box
    dt = oracle.cfl_dt(g, w.model, w.dbounds(), 0.8)
    vf = hj.ScalarField(g, v)
    stepped = oracle.vi_step(vf, hj.ScalarField(g, np.full(g.size(), -1e300)), w.model, w.dbounds(),
                             dt)
    want = np.where(l < stepped, l, stepped)
    want = np.where(want > c, want, c)
    got = oracle.vi_step(vf, hj.ScalarField(g, c), w.model, w.dbounds(), dt,
                         target=hj.ScalarField(g, l))
    assert same(got, want)
    assert not same(got, oracle.vi_step(vf, hj.ScalarField(g, c), w.model, w.dbounds(), dt))


@pytest.mark.parametrize("order,rk", [(1, 1), (2, 2), (3, 3)])
def test_inactive_target_reproduces_reference_path(oracle, ref, order, rk):
    """l >= every value: the update is the reference's (bitwise, same
    iteration count); at first order checked against the reference itself."""
    w, g, c, _ = _cfg2(11)
    cf = hj.ScalarField(g, c)
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=200, spatial_order=order, time_order=rk)
    big = hj.ScalarField(g, np.full(g.size(), 1e300))
    a = oracle.solve(cf, cf, w.model, w.dbounds(), cfg, target=big)
    b = oracle.solve(cf, cf, w.model, w.dbounds(), cfg)
    assert a.iterations == b.iterations and same(a.value.values(), b.value.values())
    assert same(a.residual_history, b.residual_history)
    if order == 1 and rk == 1:
        r = ref.solve(cf, cf, w.model, w.dbounds(), cfg)
        assert r.iterations == a.iterations and same(r.value.values(), a.value.values())


def test_reach_avoid_invariants(oracle):
    """V* >= c, V* <= max(c, l), V* <= the avoid-only V* (a target can only
    lower the value), and lowering l lowers V* pointwise."""
    w, g, c, l = _cfg2(11)
    cf = hj.ScalarField(g, c)
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=2000)
    avoid = oracle.solve(cf, cf, w.model, w.dbounds(), cfg).value.values()
    ra = oracle.solve(cf, cf, w.model, w.dbounds(), cfg, target=hj.ScalarField(g, l)).value.values()
    lower = oracle.solve(cf, cf, w.model, w.dbounds(), cfg,
                         target=hj.ScalarField(g, l - 0.5)).value.values()
    assert np.all(ra >= c) and np.all(ra <= np.maximum(c, l))
    assert np.all(ra <= avoid) and np.all(lower <= ra)
    assert np.any(ra < avoid)


def test_reference_shim_rejects_target(ref):
    w, g, c, l = _cfg2(5)
    cf = hj.ScalarField(g, c)
    cfg = hj.SolveConfig(max_iters=2)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        k = cfg.to_c()
        k.target = hj.ScalarField(g, l).ptr()
        # the shim's make_cfg refuses: the reference has no target set
        ref._call(ref.lib.hjr_solve, *ref_solve_args(ref, g, w, cf, k))


def ref_solve_args(ref, g, w, cf, k):
    import ctypes as C
    from oracle.oracle import RefResult, model_spec, _arr, _vals
    r = RefResult()
    out = np.empty(g.size())
    return (C.byref(g.to_c()), C.byref(model_spec(w.model)), C.byref(w.dbounds().to_c()),
            _arr(_vals(cf)), _arr(_vals(cf)), C.byref(k), _arr(out), C.byref(r))


# ------------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("n,iters", [(21, 300), (11, 3000)])
def test_gpu_4d_fast_path_target_matches_restatement(gpu_ctx, oracle, n, iters):
    """k_fast4d's TG variant (config-2 model, Godunov, constant bounds)."""
    w, g, c, l = _cfg2(n)
    cf, lf = hj.ScalarField(g, c), hj.ScalarField(g, l)
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=iters)
    got = hj.solve(cf, cf, w.model, w.dbounds(), cfg, ctx=gpu_ctx, target=lf)
    want = oracle.solve(cf, cf, w.model, w.dbounds(), cfg, target=lf)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,order,rk", [(hj.LAX_FRIEDRICHS, 1, 1), (hj.GODUNOV, 3, 3),
                                             (hj.LAX_FRIEDRICHS, 2, 2)])
def test_gpu_generic_target_matches_restatement(gpu_ctx, oracle, scheme, order, rk):
    w, g, c, l = _cfg2(11)
    cf, lf = hj.ScalarField(g, c), hj.ScalarField(g, l)
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=150, scheme=scheme, spatial_order=order,
                         time_order=rk)
    got = hj.solve(cf, cf, w.model, w.dbounds(), cfg, ctx=gpu_ctx, target=lf)
    want = oracle.solve(cf, cf, w.model, w.dbounds(), cfg, target=lf)
    assert got.iterations == want.iterations
    assert same(got.residual_history, want.residual_history)
    assert same(got.value.values(), want.value.values())


@pytest.mark.gpu
def test_gpu_2d_target_and_vi_step(gpu_ctx, oracle):
    """Config-1 model (2D, generic sweep instead of the cluster kernel) with a
    target band z in [1, 2]; and vi_step with a target."""
    w = configs.config1()
    g = w.grid
    c = band_np(g, 0, 0.0, 3.0)
    l = band_np(g, 0, 1.0, 2.0)
    cf, lf = hj.ScalarField(g, c), hj.ScalarField(g, l)
    got = hj.solve(cf, cf, w.model, w.dbounds(), w.cfg, ctx=gpu_ctx, target=lf)
    want = oracle.solve(cf, cf, w.model, w.dbounds(), w.cfg, target=lf)
    assert got.iterations == want.iterations and got.converged == want.converged
    assert same(got.value.values(), want.value.values())
    dt = oracle.cfl_dt(g, w.model, w.dbounds(), 0.8)
    rng = np.random.default_rng(9)
    v = hj.ScalarField(g, c + rng.random(g.size()))
    assert same(hj.vi_step(v, cf, w.model, w.dbounds(), dt, ctx=gpu_ctx, target=lf).values(),
                oracle.vi_step(v, cf, w.model, w.dbounds(), dt, target=lf))


@pytest.mark.gpu
def test_gpu_target_device_pointer_and_inactive(gpu_ctx):
    """solve_dev with a device target; an inactive target (l = 1e300) gives
    the avoid-only solve bit for bit (the TG kernel variant vs the default)."""
    w, g, c, l = _cfg2(21)
    ct = torch.tensor(c, device="cuda")
    big = torch.full_like(ct, 1e300)
    out_a = torch.empty_like(ct)
    out_b = torch.empty_like(ct)
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=200)
    torch.cuda.synchronize()
    ra = hj.solve_dev(g, w.model, w.dbounds(), ct.data_ptr(), ct.data_ptr(), out_a.data_ptr(), cfg,
                      ctx=gpu_ctx, history_capacity=200, target_ptr=big.data_ptr())
    rb = hj.solve_dev(g, w.model, w.dbounds(), ct.data_ptr(), ct.data_ptr(), out_b.data_ptr(), cfg,
                      ctx=gpu_ctx, history_capacity=200)
    assert ra.iterations == rb.iterations and same(ra.residual_history, rb.residual_history)
    assert same(out_a.cpu().numpy(), out_b.cpu().numpy())


@pytest.mark.gpu
def test_gpu_target_rejected_by_chain_and_shards(gpu_ctx):
    from paper_2101_05916_b200 import sharded
    w, g, c, l = _cfg2(11)
    ct = torch.tensor(c, device="cuda")
    lt = torch.tensor(l, device="cuda")
    out = torch.empty_like(ct)
    cfg = hj.SolveConfig(max_iters=5)
    lib_cfg = cfg.to_c()
    lib_cfg.target = lt.data_ptr()
    import ctypes as C
    from paper_2101_05916_b200 import abi
    r = abi.HjbSolveResult()
    rc = abi.load().hjb_solve_sharded_local_dev(
        gpu_ctx.handle, 2, C.byref(g.to_c()), C.byref(w.model.to_c()), C.byref(w.dbounds().to_c()),
        C.c_void_p(ct.data_ptr()), C.c_void_p(ct.data_ptr()), C.byref(lib_cfg),
        C.c_void_p(out.data_ptr()), C.byref(r))
    assert rc == abi.HJB_ERR_UNSUPPORTED
