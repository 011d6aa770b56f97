"""GP disturbance bounds (reference proj/include/hjsafe/gp.hpp, proj/src/gp.cpp).

SURVEY §8f-2: the step before the solve path.  `bounds_on_grid` produces the
per-node `IntervalField` the solver consumes; here it runs on the device
(`hjb_gp_bounds_on_grid[_dev]`, csrc/hjb_gp.cu): the GP posterior is
evaluated once per DISTINCT input point (the grid nodes' coordinates along
the channel's input dims) and broadcast to the nodes, bit for bit what the
reference's per-node `GpModel::predict` computes.  `GpModel.fit` runs on the
host inside libhjb.so (`hjb_gp_fit`, O(n^3) once per model update).

Reference map:
  DisturbanceMeasurement, GpHyperparams, GpConfig .. gp.hpp:14-37
  GpModel (prior / fit / predict) .................. gp.hpp:41-75, gp.cpp:32-208
  bounds_on_grid ................................... gp.hpp:83-87, gp.cpp:211-249
  ViolationCheck / violation_check ................. gp.hpp:89-97, gp.cpp:251-258
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import abi
from . import hjsafe as hj

__all__ = ["DisturbanceMeasurement", "GpHyperparams", "GpConfig", "GpModel", "Prediction",
           "bounds_on_grid", "bounds_on_grid_dev", "ViolationCheck", "violation_check"]


@dataclass
class DisturbanceMeasurement:
    """gp.hpp:14-18."""
    x: list
    value: float = 0.0
    time: float = 0.0


@dataclass
class GpHyperparams:
    """gp.hpp:22-29 (squared-exponential kernel, per-dimension lengthscales)."""
    signal_var: float = 0.01
    lengthscales: list = field(default_factory=lambda: [1.0])
    noise_var: float = 0.0

    def validate(self, input_dim: int):
        """gp.cpp:14-21."""
        if not (self.signal_var > 0.0):
            raise hj.InvalidArgument("GP: signal variance must be > 0")
        if not (self.noise_var >= 0.0):
            raise hj.InvalidArgument("GP: noise variance must be >= 0")
        if len(self.lengthscales) != input_dim:
            raise hj.InvalidArgument("GP: lengthscale count does not match input dim")
        for v in self.lengthscales:
            if not (v > 0.0):
                raise hj.InvalidArgument("GP: lengthscales must be > 0")


FIXED, SEARCH = "fixed", "search"


@dataclass
class GpConfig:
    """gp.hpp:31-37."""
    policy: str = SEARCH
    prior: GpHyperparams = field(default_factory=GpHyperparams)
    max_training: int = 500
    search_subsample: int = 250


@dataclass
class Prediction:
    """GpModel::Prediction, gp.hpp:55-58."""
    mean: float = 0.0
    variance: float = 0.0


class GpModel:
    """Gaussian-process posterior over one scalar disturbance channel
    (gp.hpp:41-75).  Fit once, then predictions are read-only."""

    def __init__(self):
        self._hp = GpHyperparams()
        self._dim = 1
        self._inputs = np.zeros((0, 1))
        self._alpha = np.zeros(0)
        self._chol = np.zeros((0, 0))
        self._lml = 0.0

    @staticmethod
    def prior(hp: GpHyperparams) -> "GpModel":
        """gp.cpp:32-38."""
        m = GpModel()
        m._dim = len(hp.lengthscales)
        hp.validate(m._dim)
        m._hp = GpHyperparams(hp.signal_var, list(hp.lengthscales), hp.noise_var)
        m._inputs = np.zeros((0, m._dim))
        return m

    @staticmethod
    def from_factor(hp: GpHyperparams, inputs, alpha, chol, lml: float = 0.0) -> "GpModel":
        """A fitted model from its stored factor (inputs, alpha, lower chol)."""
        m = GpModel()
        X = np.ascontiguousarray(np.asarray(inputs, dtype=np.float64))
        if X.ndim == 1:
            X = X.reshape(-1, 1)
        m._dim = X.shape[1]
        hp.validate(m._dim)
        m._hp = GpHyperparams(hp.signal_var, list(hp.lengthscales), hp.noise_var)
        m._inputs = X
        m._alpha = np.ascontiguousarray(np.asarray(alpha, dtype=np.float64))
        m._chol = np.ascontiguousarray(np.asarray(chol, dtype=np.float64))
        if m._alpha.shape != (X.shape[0],) or m._chol.shape != (X.shape[0], X.shape[0]):
            raise hj.InvalidArgument("GP: factor shapes do not match the training inputs")
        m._lml = float(lml)
        return m

    @staticmethod
    def fit(data: Sequence[DisturbanceMeasurement], cfg: GpConfig | None = None) -> "GpModel":
        """gp.cpp:124-186 (hjb_gp_fit on the host)."""
        cfg = cfg or GpConfig()
        if len(data) == 0:
            raise hj.InvalidArgument("GP fit: need at least one measurement")
        dim = len(data[0].x)
        for d in data:
            if len(d.x) != dim:
                raise hj.InvalidArgument("GP fit: inconsistent input dims")
        X = np.ascontiguousarray(np.array([d.x for d in data], dtype=np.float64).reshape(-1, dim))
        y = np.ascontiguousarray(np.array([d.value for d in data], dtype=np.float64))
        fc = abi.HjbGpFitConfig()
        fc.policy = abi.GP_SEARCH if cfg.policy == SEARCH else abi.GP_FIXED
        fc.max_training = int(cfg.max_training)
        fc.search_subsample = int(cfg.search_subsample)
        fc.prior_signal_var = cfg.prior.signal_var
        fc.prior_noise_var = cfg.prior.noise_var
        ls = list(cfg.prior.lengthscales)
        fc.prior_n_lengthscales = len(ls)
        for i, v in enumerate(ls[:abi.HJB_MAX_DIMS]):
            fc.prior_lengthscales[i] = v
        cap = min(len(data), int(cfg.max_training))
        inputs = np.zeros((cap, dim))
        alpha = np.zeros(cap)
        chol = np.zeros((cap, cap))
        out = abi.HjbGpModel()
        lml = C.c_double()
        hj._check(abi.load().hjb_gp_fit(len(data), dim, X.ctypes.data, y.ctypes.data,
                                        C.byref(fc), inputs.ctypes.data, alpha.ctypes.data,
                                        chol.ctypes.data, C.byref(out), C.byref(lml)))
        n = int(out.n_train)
        hp = GpHyperparams(out.signal_var, [out.lengthscales[d] for d in range(dim)],
                           out.noise_var)
        return GpModel.from_factor(hp, inputs[:n].copy(), alpha[:n].copy(),
                                   chol[:n, :n].copy(), lml.value)

    # ---------------------------------------------------------- accessors
    def hyperparams(self) -> GpHyperparams:
        return self._hp

    def training_count(self) -> int:
        return int(self._inputs.shape[0])

    def input_dim(self) -> int:
        return self._dim

    def log_marginal_likelihood(self) -> float:
        return self._lml

    def to_c(self, input_dims: Sequence[int] | None = None) -> abi.HjbGpModel:
        m = abi.HjbGpModel()
        m.input_dim = self._dim
        dims = list(range(self._dim)) if input_dims is None else list(input_dims)
        m.n_dims = len(dims)
        for i, d in enumerate(dims[:abi.HJB_MAX_DIMS]):
            m.input_dims[i] = int(d)
        m.n_train = self.training_count()
        m.signal_var = self._hp.signal_var
        m.noise_var = self._hp.noise_var
        for i, v in enumerate(self._hp.lengthscales[:abi.HJB_MAX_DIMS]):
            m.lengthscales[i] = v
        dp = C.POINTER(C.c_double)
        m.inputs = self._inputs.ctypes.data_as(dp)
        m.alpha = self._alpha.ctypes.data_as(dp)
        m.chol = self._chol.ctypes.data_as(dp)
        return m

    # -------------------------------------------------------- prediction
    def predict_batch(self, X, ctx: hj.Context | None = None):
        """GpModel::predict at many points on the device: (mean, variance)."""
        Xa = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        if Xa.ndim == 1:
            Xa = Xa.reshape(-1, self._dim) if self._dim > 1 else Xa.reshape(-1, 1)
        if Xa.shape[1] != self._dim:
            raise hj.InvalidArgument("GP predict: input dim mismatch")
        nq = Xa.shape[0]
        mean = np.empty(nq)
        var = np.empty(nq)
        cm = self.to_c()
        hj._check(abi.load().hjb_gp_predict_batch(hj._ctx(ctx), C.byref(cm), nq, Xa.ctypes.data,
                                                  mean.ctypes.data, var.ctypes.data))
        return mean, var

    def predict(self, x, ctx: hj.Context | None = None) -> Prediction:
        """gp.cpp:188-208."""
        xa = np.asarray(x, dtype=np.float64).reshape(-1)
        if xa.size != self._dim:
            raise hj.InvalidArgument("GP predict: input dim mismatch")
        mean, var = self.predict_batch(xa.reshape(1, -1), ctx)
        return Prediction(float(mean[0]), float(var[0]))


def _models_c(channel_models, input_dims):
    if len(channel_models) != len(input_dims):
        raise hj.InvalidArgument("bounds_on_grid: one input-dim map per channel")
    if len(channel_models) > abi.HJB_MAX_INPUT:
        raise hj.Unsupported("bounds_on_grid: too many channels")
    arr = (abi.HjbGpModel * max(1, len(channel_models)))()
    for ch, (m, dims) in enumerate(zip(channel_models, input_dims)):
        if len(dims) > abi.HJB_MAX_DIMS:
            raise hj.InvalidArgument("bounds_on_grid: input-dim map does not match GP")
        arr[ch] = m.to_c(dims)
    return arr


def bounds_on_grid(channel_models: Sequence[GpModel], input_dims: Sequence[Sequence[int]],
                   grid: hj.Grid, confidence: float = 3.0, threads: int = 0,
                   ctx: hj.Context | None = None) -> hj.IntervalField:
    """gp.cpp:211-249 on the device; returns a per-node IntervalField.
    `threads` is accepted for signature parity (the device decides)."""
    models = _models_c(channel_models, input_dims)
    nch = len(channel_models)
    n = grid.size()
    lo = [np.empty(n) for _ in range(nch)]
    hi = [np.empty(n) for _ in range(nch)]
    plo = (C.c_void_p * max(1, nch))(*[a.ctypes.data for a in lo])
    phi = (C.c_void_p * max(1, nch))(*[a.ctypes.data for a in hi])
    g = grid.to_c()
    hj._check(abi.load().hjb_gp_bounds_on_grid(hj._ctx(ctx), C.byref(g), nch, models,
                                               float(confidence), plo, phi))
    return hj.IntervalField(grid, nch, lo=lo, hi=hi)


def bounds_on_grid_dev(channel_models: Sequence[GpModel], input_dims: Sequence[Sequence[int]],
                       grid: hj.Grid, lo_ptrs: Sequence[int], hi_ptrs: Sequence[int],
                       confidence: float = 3.0, ctx: hj.Context | None = None):
    """bounds_on_grid into device buffers (grid.size() doubles per channel):
    the per-node bounds stay in HBM for hjb_solve_dev."""
    models = _models_c(channel_models, input_dims)
    nch = len(channel_models)
    plo = (C.c_void_p * max(1, nch))(*[int(p) for p in lo_ptrs])
    phi = (C.c_void_p * max(1, nch))(*[int(p) for p in hi_ptrs])
    g = grid.to_c()
    hj._check(abi.load().hjb_gp_bounds_on_grid_dev(hj._ctx(ctx), C.byref(g), nch, models,
                                                   float(confidence), plo, phi))


@dataclass
class ViolationCheck:
    """gp.hpp:89-92."""
    inside: bool = False
    margin: float = 0.0


def violation_check(field_: hj.IntervalField, channel: int, x, measured: float,
                    ctx: hj.Context | None = None) -> ViolationCheck:
    """gp.cpp:251-258: IntervalField::at (multilinear, interval_field.cpp:
    29-31) of the channel at x, closed-interval membership and margin."""
    from .safety import DeviceBuffer, interp_batch
    ctx = ctx or hj.default_context()
    g = field_.grid()
    vals = []
    for f in (field_.lo(channel), field_.hi(channel)):
        buf = DeviceBuffer(ctx, f.values().nbytes)
        buf.upload(f.values())
        v, _ = interp_batch(g, buf.ptr, np.asarray(x, dtype=np.float64).reshape(1, -1), ctx)
        buf.free()
        vals.append(float(v[0]))
    lo, hi = vals
    margin = min(measured - lo, hi - measured)
    return ViolationCheck(bool(measured >= lo and measured <= hi), margin)
