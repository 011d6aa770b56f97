"""Safety filter and decomposition over device-resident value functions.

Mirrors the reference's `SafetyFilter` (proj/include/hjsafe/safety.hpp:35-107,
proj/src/safety.cpp) and `Decomposition` (proj/include/hjsafe/decomposition.hpp,
proj/src/decomposition.cpp) — SURVEY §8(f) items 1 and 4: the caller side of
the solve path.  The value function V* stays in HBM; every query (single or
batched) runs the `hjb_filter_batch_dev` / `hjb_interp_batch_dev` kernels of
libhjb.so, which restate the reference's per-query arithmetic bit for bit.
The host side keeps only the filter's small state (lambda, emergency flag,
min V*) and the decomposition's recombination (max over subsystems, control
scatter), in the reference's order.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import abi
from . import hjsafe as hj

__all__ = ["FilterDecision", "Violation", "FilterBatch", "SafetyFilter", "Subsystem",
           "CombinedDecision", "CombinedBatch", "Decomposition", "project", "scatter",
           "DeviceBuffer", "DeviceSolve", "interp_batch"]


# ------------------------------------------------------------- device memory
class DeviceBuffer:
    """Device allocation owned through the library (hjb_malloc_dev)."""

    def __init__(self, ctx: hj.Context, nbytes: int):
        self._lib = abi.load()
        self._ctx = ctx
        p = C.c_void_p()
        hj._check(self._lib.hjb_malloc_dev(ctx.handle, int(nbytes), C.byref(p)))
        self.ptr = p.value
        self.nbytes = int(nbytes)

    def upload(self, arr: np.ndarray):
        a = np.ascontiguousarray(arr)
        if a.nbytes > self.nbytes:
            raise hj.InvalidArgument("DeviceBuffer: upload larger than the buffer")
        hj._check(self._lib.hjb_copy_h2d(self._ctx.handle, self.ptr, a.ctypes.data, a.nbytes))

    def download(self, out: np.ndarray):
        hj._check(self._lib.hjb_copy_d2h(self._ctx.handle, out.ctypes.data, self.ptr, out.nbytes))
        return out

    def free(self):
        if self.ptr:
            try:
                self._lib.hjb_free_dev(self._ctx.handle, self.ptr)
            finally:
                self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class _Workspace:
    """Grow-only device buffers for batched queries."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.bufs: dict[str, DeviceBuffer] = {}

    def get(self, name: str, nbytes: int) -> DeviceBuffer:
        b = self.bufs.get(name)
        if b is None or b.nbytes < nbytes:
            if b is not None:
                b.free()
            b = DeviceBuffer(self.ctx, max(nbytes, 64))
            self.bufs[name] = b
        return b


def _queries(x, nd: int) -> np.ndarray:
    X = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if X.ndim == 1:
        X = X.reshape(1, -1)
    if X.ndim != 2 or X.shape[1] != nd:
        raise hj.InvalidArgument("interp: query rank mismatch")
    return X


def interp_batch(grid: hj.Grid, field_ptr: int, x, ctx: hj.Context | None = None,
                 workspace: _Workspace | None = None):
    """interp_ex (grid.cpp:113-131) of a device field at many states:
    (values, out_of_domain)."""
    ctx = ctx or hj.default_context()
    ws = workspace or _Workspace(ctx)
    X = _queries(x, grid.ndims())
    nq = X.shape[0]
    dx = ws.get("ix", X.nbytes)
    dx.upload(X)
    dv = ws.get("iv", nq * 8)
    do = ws.get("io", nq)
    g = grid.to_c()
    hj._check(abi.load().hjb_interp_batch_dev(ctx.handle, C.byref(g), field_ptr, nq, dx.ptr,
                                              dv.ptr, do.ptr))
    v = dv.download(np.empty(nq))
    o = do.download(np.empty(nq, dtype=np.uint8))
    return v, o.astype(bool)


# ------------------------------------------------------------ decisions
@dataclass
class FilterDecision:
    """safety.hpp:14-22."""
    control: list = field(default_factory=list)
    worst_disturbance: list = field(default_factory=list)
    override_active: bool = False
    degenerate: bool = False
    out_of_domain: bool = False
    value: float = 0.0
    band: float = 0.0


@dataclass
class Violation:
    """safety.hpp:24-27."""
    x: list
    margin: float = 0.0


@dataclass
class FilterBatch:
    """Column form of many FilterDecisions (one row per query)."""
    value: np.ndarray
    band: np.ndarray
    control: np.ndarray            # (nq, control_dim)
    worst_disturbance: np.ndarray  # (nq, disturbance_dim); 0 where passed through
    flags: np.ndarray              # uint8 HJB_FILTER_* bits

    @property
    def override_active(self) -> np.ndarray:
        return (self.flags & abi.FILTER_OVERRIDE) != 0

    @property
    def degenerate(self) -> np.ndarray:
        return (self.flags & abi.FILTER_DEGENERATE) != 0

    @property
    def out_of_domain(self) -> np.ndarray:
        return (self.flags & abi.FILTER_OOD) != 0

    def decision(self, q: int) -> FilterDecision:
        ov = bool(self.flags[q] & abi.FILTER_OVERRIDE)
        return FilterDecision(control=[float(u) for u in self.control[q]],
                              worst_disturbance=[float(d) for d in self.worst_disturbance[q]]
                              if ov else [],
                              override_active=ov,
                              degenerate=bool(self.flags[q] & abi.FILTER_DEGENERATE),
                              out_of_domain=bool(self.flags[q] & abi.FILTER_OOD),
                              value=float(self.value[q]), band=float(self.band[q]))


def _grid_of(solved) -> hj.Grid:
    return solved.grid if isinstance(solved, DeviceSolve) else solved.value.grid()


def _std_max(a, b):
    """std::max(a, b) = (a < b) ? b : a, elementwise."""
    return np.where(np.asarray(a) < np.asarray(b), b, a)


# ---------------------------------------------------------------- filter
@dataclass
class _State:
    """SafetyFilter::State, safety.hpp:75-82, with V* resident on the device
    (the host copy `value` is filled on demand for a device-adopted V*)."""
    grid: hj.Grid
    value: hj.ScalarField | None
    dbounds: hj.IntervalField
    dev_value: DeviceBuffer
    dev_db: list
    eta_floor: float
    min_value: float
    lam: float = 0.0
    emergency: bool = False


@dataclass
class DeviceSolve:
    """A solve whose V* stayed in HBM (hjb_solve_dev): the metadata of
    SolveResult (solver.hpp:27-36) plus the device buffer of V*."""
    grid: hj.Grid
    value: DeviceBuffer
    iterations: int = 0
    dt: float = 0.0
    wall_seconds: float = 0.0
    converged: bool = False
    final_residual: float = 0.0

    def to_host(self) -> hj.SolveResult:
        v = self.value.download(np.empty(self.grid.size()))
        return hj.SolveResult(value=hj.ScalarField(self.grid, v, check=False),
                              iterations=self.iterations, dt=self.dt,
                              wall_seconds=self.wall_seconds, converged=self.converged,
                              final_residual=self.final_residual)


class SafetyFilter:
    """Least-restrictive safety filter around a converged value function
    (safety.hpp:28-107).  filter / optimal_control / value_at / dbound_at /
    contract run on the GPU; the *_batch forms answer many states per call."""

    @dataclass
    class Config:
        eta_floor: float = 1e-5
        contract_base: float = 0.05
        contract_ratio: float = 1.5
        cap_fraction: float = 0.8

    def __init__(self, model: hj.DynamicsModel, solved: hj.SolveResult,
                 dbounds: hj.IntervalField, cfg: "SafetyFilter.Config | None" = None,
                 ctx: hj.Context | None = None):
        if model is None:
            raise hj.InvalidArgument("SafetyFilter: null model")
        if _grid_of(solved).ndims() != model.state_dim():
            raise hj.InvalidArgument("SafetyFilter: grid rank does not match model")
        self._model = model
        self._cfg = cfg or SafetyFilter.Config()
        self._ctx = ctx or hj.default_context()
        self._lock = threading.Lock()
        self._ws = _Workspace(self._ctx)
        self._state = self._make_state(solved, dbounds)

    # safety.cpp:53-66
    def _make_state(self, solved, dbounds: hj.IntervalField) -> _State:
        if not solved.converged:
            raise hj.InvalidArgument("SafetyFilter: value function is not converged")
        dbounds.validate()
        if isinstance(solved, DeviceSolve):  # V* already in HBM: no host round trip
            grid, v, dev = solved.grid, None, solved.value
            mn = C.c_double()
            hj._check(abi.load().hjb_field_reduce_dev(self._ctx.handle, grid.size(), dev.ptr,
                                                      C.byref(mn), None))
            mn = mn.value
        else:
            v = solved.value
            grid = v.grid()
            dev = DeviceBuffer(self._ctx, v.size() * 8)
            dev.upload(v.values())
            mn = float(np.min(v.values()))
        dev_db = []
        if not dbounds.is_constant():
            for ch in range(dbounds.channels()):
                lo = DeviceBuffer(self._ctx, grid.size() * 8)
                lo.upload(dbounds.lo(ch).values())
                hi = DeviceBuffer(self._ctx, grid.size() * 8)
                hi.upload(dbounds.hi(ch).values())
                dev_db.append((lo, hi))
        return _State(grid=grid, value=v, dbounds=dbounds, dev_value=dev, dev_db=dev_db,
                      eta_floor=self._cfg.eta_floor, min_value=mn, lam=0.0,
                      emergency=mn >= 0.0)

    def _snapshot(self) -> _State:
        with self._lock:
            return self._state

    def _dbounds_c(self, s: _State) -> abi.HjbDbounds:
        d = abi.HjbDbounds()
        d.channels = s.dbounds.channels()
        if s.dbounds.is_constant():
            d.per_node = 0
            for ch in range(d.channels):
                b = s.dbounds.at_node(ch, 0)
                d.constant[ch].lo = b.lo
                d.constant[ch].hi = b.hi
        else:
            d.per_node = 1
            for ch, (lo, hi) in enumerate(s.dev_db):
                d.lo[ch] = C.cast(C.c_void_p(lo.ptr), C.POINTER(C.c_double))
                d.hi[ch] = C.cast(C.c_void_p(hi.ptr), C.POINTER(C.c_double))
        return d

    def _run(self, s: _State, X: np.ndarray, U: np.ndarray | None, mode: int) -> FilterBatch:
        nq = X.shape[0]
        m, p = self._model.control_dim(), self._model.disturbance_dim()
        ws = self._ws
        dx = ws.get("x", X.nbytes)
        dx.upload(X)
        du_ptr = None
        if U is not None and m > 0:
            du = ws.get("u", U.nbytes)
            du.upload(U)
            du_ptr = du.ptr
        dval, dband = ws.get("val", nq * 8), ws.get("band", nq * 8)
        dctl, dwst = ws.get("ctl", nq * m * 8), ws.get("wst", nq * p * 8)
        dflg = ws.get("flg", nq)
        out = abi.HjbFilterOut(dval.ptr, dband.ptr, dctl.ptr, dwst.ptr, dflg.ptr)
        cfg = abi.HjbFilterConfig(mode, 0, s.eta_floor, s.lam)
        g, mm, d = s.grid.to_c(), self._model.to_c(), self._dbounds_c(s)
        hj._check(abi.load().hjb_filter_batch_dev(self._ctx.handle, C.byref(g), C.byref(mm),
                                                  C.byref(d), s.dev_value.ptr, nq, dx.ptr, du_ptr,
                                                  C.byref(cfg), C.byref(out)))
        return FilterBatch(value=dval.download(np.empty(nq)), band=dband.download(np.empty(nq)),
                           control=dctl.download(np.empty((nq, m))),
                           worst_disturbance=dwst.download(np.empty((nq, p))),
                           flags=dflg.download(np.empty(nq, dtype=np.uint8)))

    # ---- queries
    def filter_batch(self, x, u_perf) -> FilterBatch:
        """SafetyFilter::filter (safety.cpp:108-127) for every row of x."""
        s = self._snapshot()
        X = _queries(x, s.grid.ndims())
        m = self._model.control_dim()
        U = np.ascontiguousarray(np.asarray(u_perf, dtype=np.float64)).reshape(X.shape[0], -1) \
            if m > 0 else np.zeros((X.shape[0], 0))
        if U.shape != (X.shape[0], m):
            raise hj.InvalidArgument("filter: control dim mismatch")
        return self._run(s, X, U, abi.FILTER_FILTER)

    def optimal_control_batch(self, x) -> FilterBatch:
        """SafetyFilter::optimal_control (safety.cpp:86-106) for every row of x."""
        s = self._snapshot()
        return self._run(s, _queries(x, s.grid.ndims()), None, abi.FILTER_OPTIMAL)

    def filter(self, x: Sequence[float], u_perf: Sequence[float]) -> FilterDecision:
        if len(u_perf) != self._model.control_dim():
            raise hj.InvalidArgument("filter: control dim mismatch")
        return self.filter_batch([list(x)], [list(u_perf)]).decision(0)

    def optimal_control(self, x: Sequence[float]) -> FilterDecision:
        return self.optimal_control_batch([list(x)]).decision(0)

    def value_at_batch(self, x) -> np.ndarray:
        s = self._snapshot()
        v, _ = interp_batch(s.grid, s.dev_value.ptr, x, self._ctx, self._ws)
        return v

    def value_at(self, x: Sequence[float]) -> float:
        return float(self.value_at_batch([list(x)])[0])

    def dbound_at(self, channel: int, x: Sequence[float]) -> hj.Interval:
        """IntervalField::at (interval_field.cpp:29-31): multilinear interpolation
        of the lo / hi fields (a constant field is interpolated node by node)."""
        s = self._snapshot()
        if not (0 <= channel < s.dbounds.channels()):
            raise hj.InvalidArgument("dbound_at: channel out of range")
        if s.dbounds.is_constant():
            key = f"const_db_{channel}"
            if key not in self._ws.bufs:
                n = s.grid.size()
                lo = DeviceBuffer(self._ctx, n * 8)
                lo.upload(s.dbounds.lo(channel).values())
                hi = DeviceBuffer(self._ctx, n * 8)
                hi.upload(s.dbounds.hi(channel).values())
                self._ws.bufs[key] = lo
                self._ws.bufs[key + "_hi"] = hi
            lo_ptr, hi_ptr = self._ws.bufs[key].ptr, self._ws.bufs[key + "_hi"].ptr
        else:
            lo_ptr, hi_ptr = s.dev_db[channel][0].ptr, s.dev_db[channel][1].ptr
        g = s.grid
        lo, _ = interp_batch(g, lo_ptr, [list(x)], self._ctx)
        hi, _ = interp_batch(g, hi_ptr, [list(x)], self._ctx)
        return hj.Interval(float(lo[0]), float(hi[0]))

    # ---- state
    def contract(self, violations: Sequence[Violation]) -> float:
        """safety.cpp:128-153: raise lambda to the smallest schedule value that
        excludes every violation site; never decreases it."""
        with self._lock:
            s = self._state
            if not violations:
                return s.lam
            v, _ = interp_batch(s.grid, s.dev_value.ptr, [list(x.x) for x in violations],
                                self._ctx, self._ws)
            deepest = -math.inf
            for val in v:
                t = -float(val)
                deepest = t if deepest < t else deepest  # std::max(deepest, -interp)
            cap = self._cfg.cap_fraction * abs(s.min_value)
            lam = self._cfg.contract_base
            emergency = False
            while lam <= deepest:
                lam *= self._cfg.contract_ratio
                if lam > cap:
                    lam = cap
                    emergency = True
                    break
            lam = s.lam if lam < s.lam else lam  # std::max(lambda, state.lambda)
            self._state = _State(grid=s.grid, value=s.value, dbounds=s.dbounds, dev_value=s.dev_value,
                                 dev_db=s.dev_db, eta_floor=s.eta_floor, min_value=s.min_value,
                                 lam=lam, emergency=s.emergency or emergency)
            return lam

    def adopt(self, solved: hj.SolveResult, dbounds: hj.IntervalField):
        """safety.cpp:155-161: install a new converged V* and bounds, reset lambda."""
        if _grid_of(solved).ndims() != self._model.state_dim():
            raise hj.InvalidArgument("adopt: grid rank does not match model")
        nxt = self._make_state(solved, dbounds)
        with self._lock:
            self._state = nxt
            for k in [k for k in self._ws.bufs if k.startswith("const_db_")]:
                self._ws.bufs.pop(k).free()

    def lambda_(self) -> float:
        return self._snapshot().lam

    def emergency(self) -> bool:
        return self._snapshot().emergency

    def dbounds_snapshot(self) -> hj.IntervalField:
        return self._snapshot().dbounds

    def value_snapshot(self) -> hj.ScalarField:
        s = self._snapshot()
        if s.value is None:  # device-adopted V*: copy out once
            v = s.dev_value.download(np.empty(s.grid.size()))
            s.value = hj.ScalarField(s.grid, v, check=False)
        return s.value

    def value_device(self) -> DeviceBuffer:
        """V* of the current state, resident in HBM (warm-start source)."""
        return self._snapshot().dev_value

    def grid(self) -> hj.Grid:
        return self._snapshot().grid

    def model(self) -> hj.DynamicsModel:
        return self._model

    def min_value(self) -> float:
        return self._snapshot().min_value


# ----------------------------------------------------------- decomposition
@dataclass
class Subsystem:
    """decomposition.hpp:14-20."""
    name: str
    model: hj.DynamicsModel
    state_map: list
    control_map: list
    disturbance_map: list


def project(x_full: Sequence[float], sub: Subsystem) -> list:
    """decomposition.cpp:10-14."""
    return [x_full[i] for i in sub.state_map]


def scatter(x_sub: Sequence[float], sub: Subsystem, x_full: list) -> None:
    """decomposition.cpp:16-20."""
    for i, j in enumerate(sub.state_map):
        x_full[j] = x_sub[i]


@dataclass
class CombinedDecision:
    """decomposition.hpp:25-31."""
    control: list = field(default_factory=list)
    override_active: bool = False
    out_of_domain: bool = False
    value: float = 0.0
    band: float = 0.0


@dataclass
class CombinedBatch:
    value: np.ndarray
    band: np.ndarray
    control: np.ndarray
    override_active: np.ndarray
    out_of_domain: np.ndarray

    def decision(self, q: int) -> CombinedDecision:
        return CombinedDecision(control=[float(u) for u in self.control[q]],
                                override_active=bool(self.override_active[q]),
                                out_of_domain=bool(self.out_of_domain[q]),
                                value=float(self.value[q]), band=float(self.band[q]))


def _check_cover(subs, dim, attr, what):
    seen = [False] * dim
    for s in subs:
        for i in getattr(s, attr):
            if i >= dim or i < 0:
                raise hj.InvalidArgument(f"{what}: index out of range")
            if seen[i]:
                raise hj.InvalidArgument(f"{what}: index maps overlap")
            seen[i] = True
    if not all(seen):
        raise hj.InvalidArgument(f"{what}: index maps do not cover all entries")


class Decomposition:
    """Split filter over self-contained subsystems (decomposition.hpp:33-80):
    membership is the max of the subsystem values; one shared contraction
    level on the combined value.  Batched queries run one device batch per
    subsystem and recombine in the reference's order."""

    def __init__(self, subsystems: Sequence[Subsystem], full_state_dim: int,
                 full_control_dim: int, full_disturbance_dim: int):
        self._subs = list(subsystems)
        if not self._subs:
            raise hj.InvalidArgument("Decomposition: no subsystems")
        for s in self._subs:
            if s.model is None:
                raise hj.InvalidArgument("Decomposition: null model")
            if (len(s.state_map) != s.model.state_dim() or len(s.control_map) != s.model.control_dim()
                    or len(s.disturbance_map) != s.model.disturbance_dim()):
                raise hj.InvalidArgument("Decomposition: index map sizes do not match model")
        _check_cover(self._subs, full_state_dim, "state_map", "state_map")
        _check_cover(self._subs, full_control_dim, "control_map", "control_map")
        _check_cover(self._subs, full_disturbance_dim, "disturbance_map", "disturbance_map")
        self._n, self._m, self._p = full_state_dim, full_control_dim, full_disturbance_dim
        self._filters: list[SafetyFilter] = []
        self._schedule = SafetyFilter.Config()
        self._lock = threading.Lock()
        self._lam = 0.0
        self._emergency = False

    def attach(self, filters: Sequence[SafetyFilter]):
        if len(filters) != len(self._subs):
            raise hj.InvalidArgument("Decomposition: one filter per subsystem")
        for f in filters:
            if f is None:
                raise hj.InvalidArgument("Decomposition: null filter")
        with self._lock:
            self._filters = list(filters)

    def count(self) -> int:
        return len(self._subs)

    def subsystem(self, i: int) -> Subsystem:
        return self._subs[i]

    def filter(self, i: int) -> SafetyFilter:
        return self._filters[i]

    def _need_filters(self):
        if not self._filters:
            raise RuntimeError("Decomposition: filters not attached")

    def _full(self, x):
        X = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        if X.ndim == 1:
            X = X.reshape(1, -1)
        return X

    def _combined_value_rows(self, X: np.ndarray) -> np.ndarray:
        """decomposition.cpp:72-81 per row: +inf when any subsystem query
        leaves its grid, else the max of the subsystem values."""
        value = np.full(X.shape[0], -np.inf)
        ood = np.zeros(X.shape[0], dtype=bool)
        for s, f in zip(self._subs, self._filters):
            b = f.optimal_control_batch(X[:, s.state_map])
            value = np.where(ood, value, _std_max(value, b.value))
            ood |= b.out_of_domain
        return np.where(ood, np.inf, value)

    def combined_value_batch(self, x) -> np.ndarray:
        with self._lock:
            self._need_filters()
            return self._combined_value_rows(self._full(x))

    def combined_value(self, x_full: Sequence[float]) -> float:
        return float(self.combined_value_batch([list(x_full)])[0])

    def combined_control_batch(self, x, u_perf) -> CombinedBatch:
        """decomposition.cpp:88-126 for every row."""
        X = self._full(x)
        U = np.ascontiguousarray(np.asarray(u_perf, dtype=np.float64)).reshape(X.shape[0], -1)
        if X.shape[1] != self._n or U.shape[1] != self._m:
            raise hj.InvalidArgument("combined_control: dimension mismatch")
        with self._lock:
            self._need_filters()
            nq = X.shape[0]
            value = np.full(nq, -np.inf)
            band = np.zeros(nq)
            ood = np.zeros(nq, dtype=bool)
            opt = []
            for s, f in zip(self._subs, self._filters):
                xs = X[:, s.state_map]
                d = f.filter_batch(xs, np.zeros((nq, len(s.control_map))))
                o = d.out_of_domain
                ood |= o
                value = np.where(o, np.inf, _std_max(value, d.value))
                band = _std_max(band, d.band)
                opt.append(f.optimal_control_batch(xs))
            passthru = (~ood) & (value <= -self._lam - band)
            control = np.zeros((nq, self._m))
            for s, o in zip(self._subs, opt):
                for j, cj in enumerate(s.control_map):
                    control[:, cj] = o.control[:, j]
            control = np.where(passthru[:, None], U, control)
            return CombinedBatch(value=value, band=band, control=control,
                                 override_active=~passthru, out_of_domain=ood)

    def combined_control(self, x_full: Sequence[float], u_perf: Sequence[float]) -> CombinedDecision:
        if len(x_full) != self._n or len(u_perf) != self._m:
            raise hj.InvalidArgument("combined_control: dimension mismatch")
        return self.combined_control_batch([list(x_full)], [list(u_perf)]).decision(0)

    def contract(self, violations_full: Sequence[Violation]) -> float:
        """decomposition.cpp:128-160."""
        with self._lock:
            self._need_filters()
            if not violations_full:
                return self._lam
            vals = self._combined_value_rows(self._full([list(v.x) for v in violations_full]))
            deepest = -math.inf
            for v in vals:
                t = -float(v)
                deepest = t if deepest < t else deepest
            min_combined = -math.inf
            for f in self._filters:
                m = f.min_value()
                min_combined = m if min_combined < m else min_combined
            cap = self._schedule.cap_fraction * abs(min_combined if min_combined < 0.0 else 0.0)
            lam = self._schedule.contract_base
            emergency = min_combined >= 0.0
            while lam <= deepest:
                lam *= self._schedule.contract_ratio
                if lam > cap:
                    lam = cap
                    emergency = True
                    break
            self._lam = lam if self._lam < lam else self._lam
            self._emergency = self._emergency or emergency
            return self._lam

    def lambda_(self) -> float:
        with self._lock:
            return self._lam

    def emergency(self) -> bool:
        with self._lock:
            return self._emergency

    def warm_update(self, constraints: Sequence[DeviceBuffer], dbounds: Sequence[hj.IntervalField],
                    cfg: hj.SolveConfig, contexts: Sequence[hj.Context] | None = None
                    ) -> list:
        """The solve half of the reference's background update job
        (sim.cpp:339-363, "warm subsystem solves, one thread each"): every
        subsystem re-solves from its filter's current V* under new bounds,
        concurrently, with V* never leaving HBM.  `constraints[i]` is the
        subsystem's constraint on the device.  Returns DeviceSolve results
        for adopt()."""
        if len(constraints) != len(self._subs) or len(dbounds) != len(self._subs):
            raise hj.InvalidArgument("warm_update: one constraint and bound field per subsystem")
        self._need_filters()
        ctxs = list(contexts) if contexts else [hj.Context(0) for _ in self._subs]
        out: list = [None] * len(self._subs)
        errors: list = [None] * len(self._subs)

        def job(i):
            try:
                f, s = self._filters[i], self._subs[i]
                g = f.grid()
                dst = DeviceBuffer(ctxs[i], g.size() * 8)
                r = hj.solve_dev(g, s.model, dbounds[i], f.value_device().ptr, constraints[i].ptr,
                                 dst.ptr, cfg, ctx=ctxs[i])
                out[i] = DeviceSolve(grid=g, value=dst, iterations=r.iterations, dt=r.dt,
                                     wall_seconds=r.wall_seconds, converged=r.converged,
                                     final_residual=r.final_residual)
            except Exception as e:  # reported like the reference's job->error
                errors[i] = e

        threads = [threading.Thread(target=job, args=(i,)) for i in range(len(self._subs))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for e in errors:
            if e is not None:
                raise e
        return out

    def adopt(self, solved: Sequence, dbounds: Sequence[hj.IntervalField]):
        """decomposition.cpp:172-182 (host SolveResults or device DeviceSolves)."""
        if len(solved) != len(self._subs) or len(dbounds) != len(self._subs):
            raise hj.InvalidArgument("adopt: one result per subsystem")
        with self._lock:
            self._need_filters()
            for f, r, d in zip(self._filters, solved, dbounds):
                f.adopt(r, d)
            self._lam = 0.0
