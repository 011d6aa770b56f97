"""Exercise every kernel family of libhjb.so on small grids, for
compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_kernels.py

Covers k_fast4d (Godunov / Lax-Friedrichs / per-node bounds / target set /
multi-sweep persistent / run-time row shapes), k_ho4t (ENO2), k_eno3g (ENO3 Godunov and LF),
the generic k_step / k_ho_stage, k_small2d / k_small2d_ho (2D cluster
kernels), the sharded in-process protocol, the resample / seed chain,
k_gp_ring (GP bounds) and the safety-filter batch.  Every result is also
checked against the CPU restatement, so a sanitizer run is a parity run.
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle.oracle import Restatement  # noqa: E402
from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import gp as gpm  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402
from paper_2101_05916_b200 import sharded  # noqa: E402
from cases import band_np, fmax_np  # noqa: E402


def check(name, got, want):
    ok = np.array_equal(np.asarray(got), np.asarray(want))
    print(f"{'ok  ' if ok else 'FAIL'} {name}", flush=True)
    if not ok:
        sys.exit(1)


def main():
    ora = Restatement()
    ctx = hj.Context(0)
    n = int(os.environ.get("SAN_N", "9"))
    w = configs.config2(n)
    g = w.grid
    c = hj.ScalarField(g, band_np(g, 0, -4.0, 4.0))
    base = dict(tolerance=1e-12, max_iters=6)
    # first order: Godunov (k_fast4d), multi-sweep, LF per-node / global
    for label, extra, env in (("k_fast4d godunov", {}, {"HJB_MS": "0"}),
                              ("k_fast4d multi-sweep", {}, {"HJB_MS": "1"}),
                              ("k_fast4d lf per-node", {"scheme": hj.LAX_FRIEDRICHS}, {}),
                              ("k_fast4d lf global", {"scheme": hj.LAX_FRIEDRICHS,
                                                      "dissipation": hj.GLOBAL}, {})):
        os.environ.update(env)
        cfg = hj.SolveConfig(**base, **extra)
        r = hj.solve(c, c, w.model, w.dbounds(), cfg, ctx=ctx)
        check(label, r.value.values(), ora.solve(c, c, w.model, w.dbounds(), cfg).value.values())
        for k in env:
            os.environ.pop(k)
    # run-time row shapes (k_fast4d<ShapeGen>): a user model outside the
    # compiled shapes, per-sweep and multi-sweep launches
    from test_gpu_gen4d import mixed_model  # noqa: E402
    mm, mdb = mixed_model(), hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    for label, env, extra in (("k_fast4d run-time shape", {"HJB_MS": "0"}, {}),
                              ("k_fast4d run-time shape multi-sweep", {"HJB_MS": "1"}, {}),
                              ("k_fast4d run-time shape lf", {}, {"scheme": hj.LAX_FRIEDRICHS})):
        os.environ.update(env)
        cfg = hj.SolveConfig(**base, **extra)
        r = hj.solve(c, c, mm, mdb, cfg, ctx=ctx)
        check(label, r.value.values(), ora.solve(c, c, mm, mdb, cfg).value.values())
        for k in env:
            os.environ.pop(k)
    # per-node bounds (k_fast4d PV=2), target set (TG)
    rng = np.random.default_rng(2)
    lo = -0.5 - 0.1 * rng.random(g.size())
    hi = 0.5 + 0.1 * rng.random(g.size())
    pn = hj.IntervalField(g, 1, lo=[lo], hi=[hi])
    cfg = hj.SolveConfig(**base)
    check("k_fast4d per-node bounds", hj.solve(c, c, w.model, pn, cfg, ctx=ctx).value.values(),
          ora.solve(c, c, w.model, pn, cfg).value.values())
    tg = hj.ScalarField(g, fmax_np(band_np(g, 0, 2.5, 3.5), band_np(g, 1, -1.0, 1.0)))
    check("k_fast4d target", hj.solve(c, c, w.model, w.dbounds(), cfg, ctx=ctx, target=tg).value.values(),
          ora.solve(c, c, w.model, w.dbounds(), cfg, target=tg).value.values())
    # high order: ENO2 (k_ho4t), ENO3 (k_eno3g) Godunov + LF, generic (HJB_FAST=0)
    for label, order, rk, extra, env in (("k_ho4t eno2/rk2", 2, 2, {}, {}),
                                         ("k_eno3g eno3/rk3", 3, 3, {}, {}),
                                         ("k_eno3g lf", 3, 3, {"scheme": hj.LAX_FRIEDRICHS}, {}),
                                         ("k_ho_stage generic", 3, 3, {}, {"HJB_FAST": "0"}),
                                         ("k_step generic", 1, 1, {}, {"HJB_FAST": "0"})):
        os.environ.update(env)
        cfg = hj.SolveConfig(**base, spatial_order=order, time_order=rk, **extra)
        cfg.max_iters = 3
        r = hj.solve(c, c, w.model, w.dbounds(), cfg, ctx=ctx)
        check(label, r.value.values(), ora.solve(c, c, w.model, w.dbounds(), cfg).value.values())
        for k in env:
            os.environ.pop(k)
    # 2D cluster kernels (config 1 model, 41^2)
    w1 = configs.config1()
    g1 = hj.Grid([(-2.0, 4.0, 41), (-4.0, 4.0, 41)])
    c1 = hj.ScalarField(g1, band_np(g1, 0, 0.0, 3.0))
    db1 = hj.IntervalField.constant(g1, [hj.Interval(-0.5, 0.5)])
    for label, order, rk in (("k_small2d", 1, 1), ("k_small2d_ho", 2, 2)):
        cfg = hj.SolveConfig(tolerance=1e-4, max_iters=40, spatial_order=order, time_order=rk)
        check(label, hj.solve(c1, c1, w1.model, db1, cfg, ctx=ctx).value.values(),
              ora.solve(c1, c1, w1.model, db1, cfg).value.values())
    # sharded in-process protocol (boundary/interior launches, copies, reduce)
    import torch
    ct = torch.tensor(c.values(), device="cuda")
    out = torch.empty_like(ct)
    torch.cuda.synchronize()
    for order, rk in ((1, 1), (3, 3)):
        cfg = hj.SolveConfig(**base, spatial_order=order, time_order=rk)
        cfg.max_iters = 4
        sharded.solve_sharded_local_dev(3, g, w.model, w.dbounds(), ct.data_ptr(), ct.data_ptr(),
                                        out.data_ptr(), cfg, ctx)
        check(f"sharded local x3 order {order}", out.cpu().numpy(),
              ora.solve(c, c, w.model, w.dbounds(), cfg).value.values())
    # adaptive chain (resample + seed + per-node coarse bounds)
    ws = configs.config5(levels=(5, 9))
    cf = hj.ScalarField(ws[-1].grid, ws[-1].constraint(band_np, fmax_np))
    cfg = hj.SolveConfig(tolerance=1e-12, max_iters=5)
    a = hj.solve_multilevel(cf, ws[-1].model, ws[-1].dbounds(), [ws[0].grid], cfg, ctx=ctx)
    b = ora.solve_multilevel(cf, ws[-1].model, ws[-1].dbounds(), [ws[0].grid], cfg)
    check("multilevel chain", a.levels[-1].value.values(), b.levels[-1].value.values())
    # GP bounds on the grid (k_gp_ring)
    rng = np.random.default_rng(5)
    X = rng.uniform(-5, 5, size=(40, 1))
    y = np.sin(X[:, 0]) * 0.3
    hp = gpm.GpHyperparams(0.2, [1.5], 1e-3)
    from gp_cases import factor_model
    m = factor_model(hp, X, y)
    bd = gpm.bounds_on_grid([m], [[0]], g, ctx=ctx)
    want = ora.gp_bounds_on_grid([m], [[0]], g)
    check("k_gp_ring bounds", bd.lo(0).values(), want[0][0])
    print("all kernels exercised", flush=True)


if __name__ == "__main__":
    main()
