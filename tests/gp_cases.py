"""Shared GP fixtures: synthetic disturbance samples (the reference test's
bump d(x) = 0.5 exp(-x^2) + noise, test_gp.cpp:20-33, with numpy's seeded
generator), factor construction and a numpy restatement of GpModel::fit
(gp.cpp:43-186) to check the library's host fit."""
import math

import numpy as np

from paper_2101_05916_b200 import hjsafe as hj


def bump_samples(n, noise_sd, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-2.0, 2.0, size=n)
    y = 0.5 * np.exp(-x * x) + (rng.normal(0.0, noise_sd, size=n) if noise_sd > 0 else 0.0)
    return x.reshape(-1, 1), np.asarray(y, dtype=np.float64)


def kmat(hp, A, B):
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    q = np.zeros((A.shape[0], B.shape[0]))
    for d in range(A.shape[1]):
        r = (A[:, d][:, None] - B[:, d][None, :]) / hp.lengthscales[d]
        q += r * r
    return hp.signal_var * np.exp(-0.5 * q)


def factor(hp, X, y):
    X = np.asarray(X, dtype=np.float64).reshape(len(y), -1)
    K = kmat(hp, X, X) + (hp.noise_var + 1e-8 * hp.signal_var) * np.eye(len(y))
    L = np.linalg.cholesky(K)
    z = np.linalg.solve(L, np.asarray(y, dtype=np.float64))
    alpha = np.linalg.solve(L.T, z)
    lml = (-0.5 * float(np.dot(y, alpha)) - float(np.sum(np.log(np.diag(L))))
           - 0.5 * len(y) * math.log(2.0 * math.pi))
    return L, alpha, lml


def factor_model(hp, X, y):
    """A GpModel from the exact posterior factor of (X, y) under hp."""
    X = np.asarray(X, dtype=np.float64).reshape(len(y), -1)
    L, alpha, lml = factor(hp, X, y)
    return hj.GpModel.from_factor(hp, X, alpha, L, lml)


def uniform_subsample(n, cap):
    if n <= cap:
        return list(range(n))
    idx = [(i * (n - 1)) // (cap - 1) for i in range(cap)]
    out = []
    for i in idx:
        if not out or out[-1] != i:
            out.append(i)
    return out


def candidates(X, y):
    y_sd = max(math.sqrt(float(np.dot(y, y)) / len(y) + 1e-12), 1e-3)
    rng_ = [max(float(X[:, d].max() - X[:, d].min()), 1e-3) for d in range(X.shape[1])]
    out = []
    for sf in (0.5, 1.0, 2.0):
        for ls in (0.08, 0.2, 0.5, 1.0):
            for sn in (0.03, 0.08, 0.2, 0.5):
                out.append(hj.GpHyperparams((sf * y_sd) * (sf * y_sd),
                                            [ls * r for r in rng_], (sn * y_sd) * (sn * y_sd)))
    return out


def numpy_fit(X, y, cfg):
    X = np.asarray(X, dtype=np.float64)
    tr = uniform_subsample(len(y), cfg.max_training)
    xs, ys = X[tr], y[tr]
    chosen = cfg.prior
    if cfg.policy == "search":
        s = uniform_subsample(len(ys), cfg.search_subsample)
        sx, sy = xs[s], ys[s]
        best = -math.inf
        for hp in candidates(sx, sy):
            try:
                _, _, lml = factor(hp, sx, sy)
            except np.linalg.LinAlgError:
                continue
            if lml > best:
                best, chosen = lml, hp
    L, alpha, lml = factor(chosen, xs, ys)
    return {"hp": chosen, "L": L, "alpha": alpha, "lml": lml}


def fitted(n, seed, hp=None, dims=1):
    X, y = bump_samples(n, 0.05, seed)
    if dims > 1:
        X = np.hstack([X] + [np.random.default_rng(seed + k).uniform(-1, 1, size=(n, 1))
                             for k in range(dims - 1)])
    hp = hp or hj.GpHyperparams(0.09, [0.4] * dims, 0.002)
    return factor_model(hp, X, y)


GRID_CASES = [
    # (name, grid, models, input dims)
    ("prior_1d", [(0.0, 3.0, 11)], lambda: [hj.GpModel.prior(hj.GpHyperparams(0.01, [1.0], 0.0))],
     [[0]]),
    ("one_point", [(0.0, 2.0, 5)],
     lambda: [factor_model(hj.GpHyperparams(0.04, [0.5], 0.0), [[1.0]], [1.0])], [[0]]),
    ("bump60_2d", [(-2.0, 2.0, 41), (-1.0, 1.0, 9)], lambda: [fitted(60, 3)], [[0]]),
    ("bump300_4d_x", [(-2.0, 2.0, 13), (-2.0, 2.0, 7), (-0.35, 0.35, 5), (-1.5, 1.5, 6)],
     lambda: [fitted(300, 101)], [[0]]),
    ("two_dims", [(-2.0, 2.0, 9), (-1.0, 1.0, 5), (-1.0, 1.0, 7)], lambda: [fitted(80, 9, dims=2)],
     [[0, 2]]),
    ("repeated_axis", [(-2.0, 2.0, 9), (-1.0, 1.0, 5)], lambda: [fitted(50, 5, dims=2)], [[1, 1]]),
    ("two_channels", [(-2.0, 2.0, 11), (-1.0, 1.0, 6)],
     lambda: [fitted(40, 1), fitted(70, 2)], [[0], [1]]),
    ("n1100_R2", [(-2.0, 2.0, 17), (-1.0, 1.0, 3)], lambda: [fitted(1100, 8)], [[0]]),
]
