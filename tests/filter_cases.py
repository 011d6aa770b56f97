"""Shared cases for the safety-filter / decomposition tests."""
import numpy as np

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj

from cases import band_np


def queries(grid, n, seed, spread=0.1):
    """Uniform states over the grid box widened by `spread` (some land
    outside: out-of-domain), plus node-aligned and cell-face-aligned states."""
    rng = np.random.default_rng(seed)
    lo = np.array([d.min for d in grid.dims()])
    hi = np.array([d.max for d in grid.dims()])
    X = lo + (hi - lo) * rng.uniform(-spread, 1 + spread, size=(n, grid.ndims()))
    k = max(1, n // 10)
    idx = rng.integers(0, [d.n for d in grid.dims()], size=(k, grid.ndims()))
    X[:k] = np.array([[grid.coord(d, int(i[d])) for d in range(grid.ndims())] for i in idx])
    X[k:2 * k, 0] = lo[0] + (hi[0] - lo[0]) * rng.integers(0, 5, size=k) / 4
    return X


def vertical_case(oracle):
    """Config 1 (2D), converged by the restatement."""
    w = configs.config1()
    c = hj.ScalarField(w.grid, band_np(w.grid, 0, 0.0, 3.0))
    res = oracle.solve(c, c, w.model, w.dbounds(), w.cfg)
    return w.grid, w.model, w.dbounds(), res.value


def planar_case(n=9, seed=4, per_node=False):
    """4D planar model, a random smooth-ish V (the query math is defined for
    any finite field) and constant or per-node wind bounds."""
    w = configs.config2(n)
    g = w.grid
    rng = np.random.default_rng(seed)
    idx = np.indices(g.shape).reshape(g.ndims(), -1).T.astype(float)
    V = np.sin(idx @ rng.uniform(0.2, 0.9, g.ndims())) + 0.3 * rng.standard_normal(g.size())
    if per_node:
        lo = -0.5 + 0.2 * rng.random(g.size())
        hi = lo + 0.4 + 0.3 * rng.random(g.size())
        db = hj.IntervalField(g, 1, lo=[lo], hi=[hi])
    else:
        db = w.dbounds()
    return g, w.model, db, hj.ScalarField(g, V)


def converged(value):
    return hj.SolveResult(value=value, converged=True)


def decomposition_10d(n4=7, n2=11, seed=9):
    """NearHover10D split into x / y (4D planar) and z (2D vertical)
    subsystems, as sim.cpp builds it, with random finite V per subsystem."""
    rng = np.random.default_rng(seed)
    x, y = configs.config2(n4), configs.config2(n4)
    y.model = hj.NearHoverPlanar4D("y", configs.planar_model().p, d_row=0)
    z = configs.config1()
    z.grid = configs.vertical_grid(n2)
    subs, values, dbs = [], [], []
    maps = [([0, 1, 2, 3], [0], [0]), ([4, 5, 6, 7], [1], [1]), ([8, 9], [2], [2])]
    for w, (sm, cm, dm), name in zip((x, y, z), maps, ("x", "y", "z")):
        subs.append(hj.Subsystem(name, w.model, sm, cm, dm))
        g = w.grid
        idx = np.indices(g.shape).reshape(g.ndims(), -1).T.astype(float)
        V = np.cos(idx @ rng.uniform(0.3, 1.1, g.ndims())) - 0.4 + 0.2 * rng.standard_normal(g.size())
        values.append(hj.ScalarField(g, V))
        dbs.append(w.dbounds())
    full = []
    for k in range(400):
        xf = np.zeros(10)
        for s, v in zip(subs, values):
            g = v.grid()
            lo = np.array([d.min for d in g.dims()])
            hi = np.array([d.max for d in g.dims()])
            xf[s.state_map] = lo + (hi - lo) * rng.uniform(-0.03, 1.03, g.ndims())
        full.append(xf)
    X = np.array(full)
    U = rng.uniform(-0.5, 0.5, size=(len(X), 3))
    return subs, values, dbs, (10, 3, 3), X, U
