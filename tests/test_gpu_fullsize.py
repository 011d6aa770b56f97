"""Parity at the BASELINE grid sizes (SURVEY §8c config-level protocol).

The full-grid solve / stage runs on the device; the CPU oracle recomputes a
handful of axis-0 planes of the same update (first planes, middle, last
planes: every grid edge, tile seam and axis-3 segment of those planes) from
the same inputs, which keeps the CPU side to seconds at 101^4.
"""
import numpy as np
import pytest
import torch

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj
from paper_2101_05916_b200 import sharded

from cases import band_np, same

pytestmark = pytest.mark.gpu


def _planes(n0):
    return [(0, 4), (n0 // 2 - 2, n0 // 2 + 2), (n0 - 4, n0)]


@pytest.mark.parametrize("n", [71, 101])
def test_first_order_sweep_full_grid(gpu_ctx, oracle, n):
    """One first-order Godunov sweep of config 2/3/4's 4D model on the full
    n^4 grid from V = c (k_fast4d) against the oracle's sweep of those planes."""
    w = configs.config2(n)
    g = w.grid
    c = band_np(g, 0, -4.0, 4.0)
    cf = hj.ScalarField(g, c)
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.max_iters = 1
    got = hj.solve(cf, cf, w.model, w.dbounds(), cfg, ctx=gpu_ctx)
    dt = oracle.cfl_dt(g, w.model, w.dbounds(), cfg.cfl_factor)
    assert got.dt == dt
    gv = got.value.values()
    s0 = g.size() // n
    want = np.empty(g.size())
    mx = 0.0
    for b, e in _planes(n):
        mx = max(mx, oracle.sweep_planes(g, w.model, w.dbounds(), cf, cf, dt, b, e, want))
        assert same(gv[b * s0:e * s0], want[b * s0:e * s0]), (b, e)
    assert got.residual_history[0] >= mx / dt


def test_config3_eno3_stage_full_grid(gpu_ctx, oracle):
    """One ENO3 / TVD-RK3 final stage (k_eno3g, ghost-layout buffers) on the
    full 101^4 grid from random stage inputs, against the oracle's stage of
    the first, middle and last planes."""
    n = 101
    w = configs.config3(n)
    g = w.grid
    rng = np.random.default_rng(101)
    c = band_np(g, 0, -4.0, 4.0)
    vn = c + 0.2 * rng.random(g.size())
    vs = vn + 0.05 * rng.random(g.size())
    dt = oracle.cfl_dt(g, w.model, w.dbounds(), 0.8)
    vst, vnt, ct = (torch.tensor(x, device="cuda") for x in (vs, vn, c))
    out = torch.empty_like(vst)
    torch.cuda.synchronize()
    dv = sharded.ho_stage_planes_dev(g, w.model, w.dbounds(), vst.data_ptr(), vnt.data_ptr(),
                                     ct.data_ptr(), dt, 3, 3, 0, n, out.data_ptr(), ctx=gpu_ctx)
    gv = out.cpu().numpy()
    del vst, vnt, ct, out
    s0 = g.size() // n
    want = np.empty(g.size())
    mx = 0.0
    for b, e in _planes(n):
        mx = max(mx, oracle.ho_stage_planes(g, w.model, w.dbounds(), vs, vn, hj.ScalarField(g, c),
                                            dt, 3, 3, b, e, want))
        assert same(gv[b * s0:e * s0], want[b * s0:e * s0]), (b, e)
    assert dv >= mx
