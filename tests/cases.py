"""Parity cases shared by the CPU (oracle vs reference / golden) and GPU tests.

Each case is a small, seeded instance of the reference's hot path.  Grids
are sized so the CPU oracle finishes in seconds.  Cases restate the
reference's own test setups (proj/tests/test_solver.cpp) and BASELINE.json
configs at reduced resolution.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj


def band_np(grid: hj.Grid, dim: int, lo: float, hi: float) -> np.ndarray:
    """signed_distance_band (levelset.cpp:54-66) in numpy, same arithmetic."""
    x = grid.coords(dim)
    v = np.where((lo - x) < (x - hi), x - hi, lo - x)  # std::max(lo - x, x - hi)
    shape = [1] * grid.ndims()
    shape[dim] = grid.dim(dim).n
    return np.broadcast_to(v.reshape(shape), grid.shape).reshape(-1).copy()


def fmax_np(a, b):
    return np.where(a < b, b, a)


@dataclass
class Case:
    name: str
    grid: hj.Grid
    model: hj.DynamicsModel
    db: hj.IntervalField
    c: np.ndarray
    cfg: hj.SolveConfig
    init: np.ndarray | None = None
    per_node: bool = False

    def init_field(self):
        return hj.ScalarField(self.grid, self.c if self.init is None else self.init)

    def c_field(self):
        return hj.ScalarField(self.grid, self.c)


def quad_setup(n, dbar=0.3, **cfg):
    """QuadSetup of test_solver.cpp:33-44."""
    g = hj.Grid([(0.0, 3.2, n), (-5.0, 5.0, n)])
    c = band_np(g, 0, 0.35, 2.8)
    db = hj.IntervalField.constant(g, [hj.Interval(-dbar, dbar)])
    return Case(f"quad{n}_d{dbar}", g, hj.Quad2DVert(), db, c, hj.SolveConfig(**cfg))


def workload_case(w: configs.Workload, **cfg_over):
    c = w.constraint(band_np, fmax_np)
    cfg = hj.SolveConfig(**{**w.cfg.__dict__, **cfg_over})
    return Case(w.name, w.grid, w.model, w.dbounds(), c, cfg)


def per_node_case(n=21, seed=7):
    """Quad2DVert with a per-node disturbance field (GP-style bounds)."""
    rng = np.random.default_rng(seed)
    g = hj.Grid([(0.0, 3.2, n), (-5.0, 5.0, n)])
    c = band_np(g, 0, 0.35, 2.8)
    lo = -0.2 - 0.3 * rng.random(g.size())
    hi = 0.2 + 0.3 * rng.random(g.size())
    db = hj.IntervalField(g, 1, lo=[lo], hi=[hi])
    return Case(f"quad{n}_pernode", g, hj.Quad2DVert(), db, c, hj.SolveConfig(), per_node=True)


def twin_case(n=11):
    """Decomposition test setup, test_decomposition.cpp:116-144, coarser."""
    g = hj.Grid([(-2.5, 2.5, n), (-3.0, 3.0, n), (-2.5, 2.5, n), (-3.0, 3.0, n)])
    c = band_np(g, 0, -1.8, 1.8)
    for dim, lo, hi in ((1, -2.4, 2.4), (2, -1.8, 1.8), (3, -2.4, 2.4)):
        c = fmax_np(c, band_np(g, dim, lo, hi))
    db = hj.IntervalField.constant(g, [hj.Interval(-0.15, 0.15)] * 2)
    return Case(f"twin{n}", g, hj.TwinDoubleIntegrator(), db, c, hj.SolveConfig())


def stock_planar_case(n=11):
    """Stock reference NearHoverPlanar4D (wind on the velocity row)."""
    g = configs.planar_grid(n)
    c = band_np(g, 0, -4.0, 4.0)
    db = hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)])
    return Case(f"stock_planar{n}", g, hj.NearHoverPlanar4D("x"), db, c, hj.SolveConfig())


def solve_cases():
    """(case, max_iters) pairs solved to convergence or to the budget."""
    out = []
    c1 = workload_case(configs.config1())
    out.append((c1, 20000))
    out.append((quad_setup(41), 20000))
    q = quad_setup(21)
    q.cfg.scheme = hj.LAX_FRIEDRICHS
    q.name = "quad21_lf_pernode"
    out.append((q, 300))
    q = quad_setup(21)
    q.cfg.scheme = hj.LAX_FRIEDRICHS
    q.cfg.dissipation = hj.GLOBAL
    q.name = "quad21_lf_global"
    out.append((q, 300))
    out.append((per_node_case(), 20000))
    b = workload_case(configs.config2(11))
    out.append((b, 60))
    b = workload_case(configs.config2(13))
    b.cfg.scheme = hj.LAX_FRIEDRICHS
    b.name = "cfg2_13_lf"
    out.append((b, 40))
    out.append((twin_case(9), 20000))
    out.append((stock_planar_case(9), 50))
    d = quad_setup(15)
    d.model = hj.DoubleIntegrator()
    d.name = "double_int15"
    out.append((d, 20000))
    v = workload_case(configs.config5(levels=(11,))[0])
    out.append((v, 50))
    return out


def with_iters(case: Case, k: int) -> Case:
    cfg = hj.SolveConfig(**case.cfg.__dict__)
    cfg.max_iters = k
    return Case(case.name, case.grid, case.model, case.db, case.c, cfg, case.init, case.per_node)


def same(a, b) -> bool:
    """IEEE == equality (+0 == -0), the parity contract."""
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and bool(np.all(a == b))


def hash_field(v) -> str:
    import hashlib
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64) + 0.0)  # -0 -> +0
    return hashlib.sha256(v.tobytes()).hexdigest()
