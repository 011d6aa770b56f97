"""Python mirror of the reference solver API (hjsafe, ``proj/include/hjsafe``).

Same names, argument meaning and error behaviour as the reference's C++ API,
implemented over the C ABI of ``libhjb.so`` (include/hjb.h).  Every compute
call runs on the GPU; there is no CPU path.  Reference ``std::invalid_argument``
surfaces as :class:`InvalidArgument` (a ``ValueError``), ``std::runtime_error``
as :class:`SolverRuntimeError`, the divergence guard as :class:`DivergenceError`.

Reference map:
  Grid / GridDim / ScalarField ........ grid.hpp:11-69
  IntervalField ....................... interval_field.hpp:11-42
  models .............................. dynamics.hpp:96-271
  SolveConfig / SolveResult ........... solver.hpp:12-43
  cfl_dt / vi_step / solve ............ solver.hpp:48-65
  solve_coarse_to_fine / resample ..... solver.hpp:70-77, grid.hpp:108-109
  signed_distance_band, field_max/min . levelset.hpp:31-39
  GpModel / bounds_on_grid ........... gp.hpp:41-97 (gp.py)
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import abi

# ----------------------------------------------------------------- errors


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class SolverRuntimeError(RuntimeError):
    """std::runtime_error in the reference."""


class DivergenceError(SolverRuntimeError):
    """solve: diverging (residual grew 10x above its minimum)."""


class CudaError(RuntimeError):
    pass


class Unsupported(RuntimeError):
    pass


def _check(rc: int):
    if rc == abi.HJB_OK:
        return
    msg = abi.load().hjb_last_error().decode()
    if rc == abi.HJB_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == abi.HJB_ERR_RUNTIME:
        raise SolverRuntimeError(msg)
    if rc == abi.HJB_ERR_DIVERGED:
        raise DivergenceError(msg)
    if rc == abi.HJB_ERR_UNSUPPORTED:
        raise Unsupported(msg)
    raise CudaError(msg)


# ------------------------------------------------------------------ context
_tls = threading.local()


class Context:
    """Owns a CUDA stream and device workspaces (hjb_context)."""

    def __init__(self, device: int = 0):
        self._lib = abi.load()
        h = C.c_void_p()
        _check(self._lib.hjb_context_create(device, C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            self._lib.hjb_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self._lib.hjb_context_launch_count(self.handle))

    @property
    def stream(self) -> int:
        return int(self._lib.hjb_context_stream(self.handle) or 0)

    def synchronize(self):
        _check(self._lib.hjb_context_synchronize(self.handle))


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(0)
        _tls.ctx = ctx
    return ctx


# --------------------------------------------------------------------- grid
@dataclass(frozen=True)
class Interval:
    lo: float = 0.0
    hi: float = 0.0


@dataclass(frozen=True)
class GridDim:
    min: float = 0.0
    max: float = 1.0
    n: int = 2


class Grid:
    """Uniform Cartesian grid, row-major with the last dim fastest (grid.hpp:23-48)."""

    def __init__(self, dims: Sequence):
        self._dims = tuple(d if isinstance(d, GridDim) else GridDim(float(d[0]), float(d[1]), int(d[2]))
                           for d in dims)
        if len(self._dims) < 1:
            raise InvalidArgument("Grid: ndims must be >= 1")
        if len(self._dims) > 32:
            raise InvalidArgument("Grid: ndims must be <= 32")
        for i, d in enumerate(self._dims):
            if not (d.min < d.max):
                raise InvalidArgument(f"Grid: min must be < max in dim {i}")
            if d.n < 2:
                raise InvalidArgument(f"Grid: need at least 2 nodes in dim {i}")
            if not (math.isfinite(d.min) and math.isfinite(d.max)):
                raise InvalidArgument(f"Grid: non-finite bounds in dim {i}")
        self._spacing = tuple((d.max - d.min) / float(d.n - 1) for d in self._dims)
        strides = [1] * len(self._dims)
        for i in range(len(self._dims) - 2, -1, -1):
            strides[i] = strides[i + 1] * self._dims[i + 1].n
        self._strides = tuple(strides)

    def ndims(self) -> int:
        return len(self._dims)

    def size(self) -> int:
        return int(np.prod([d.n for d in self._dims], dtype=np.int64))

    def dim(self, i: int) -> GridDim:
        return self._dims[i]

    def dims(self):
        return self._dims

    @property
    def shape(self):
        return tuple(d.n for d in self._dims)

    def spacing(self, i: int) -> float:
        return self._spacing[i]

    def stride(self, i: int) -> int:
        return self._strides[i]

    def coord(self, d: int, k: int) -> float:
        """Grid::coord, grid.cpp:33-38 (endpoint exact)."""
        dim = self._dims[d]
        if k >= dim.n:
            raise IndexError("Grid::coord: index out of range")
        if k == dim.n - 1:
            return dim.max
        return dim.min + float(k) * self._spacing[d]

    def coords(self, d: int) -> np.ndarray:
        dim = self._dims[d]
        x = dim.min + np.arange(dim.n, dtype=np.float64) * self._spacing[d]
        x[-1] = dim.max
        return x

    def linear_index(self, index) -> int:
        return int(sum(int(i) * s for i, s in zip(index, self._strides)))

    def unravel(self, lin: int):
        out = []
        for s in self._strides:
            out.append(lin // s)
            lin -= out[-1] * s
        return out

    def __eq__(self, other):
        return isinstance(other, Grid) and self._dims == other._dims

    def __hash__(self):
        return hash(self._dims)

    def __repr__(self):
        return "Grid(" + ", ".join(f"({d.min}, {d.max}, {d.n})" for d in self._dims) + ")"

    def to_c(self) -> abi.HjbGrid:
        if len(self._dims) > abi.HJB_MAX_DIMS:
            raise Unsupported(f"device kernels support grids up to {abi.HJB_MAX_DIMS} dims")
        g = abi.HjbGrid()
        g.ndims = len(self._dims)
        for i, d in enumerate(self._dims):
            g.dims[i].min = d.min
            g.dims[i].max = d.max
            g.dims[i].n = d.n
        return g


class ScalarField:
    """One fp64 value per grid node (grid.hpp:50-69); rejects non-finite values."""

    def __init__(self, grid: Grid, values=None, fill: float = 0.0, check: bool = True):
        self._grid = grid
        if values is None:
            self._v = np.full(grid.size(), fill, dtype=np.float64)
        else:
            v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))
            if v.size != grid.size():
                raise InvalidArgument("ScalarField: value count does not match grid")
            if check and not np.all(np.isfinite(v)):
                raise InvalidArgument("ScalarField: non-finite value")
            self._v = v

    def grid(self) -> Grid:
        return self._grid

    def values(self) -> np.ndarray:
        return self._v

    def size(self) -> int:
        return self._v.size

    def __getitem__(self, i):
        return self._v[i]

    def __setitem__(self, i, x):
        self._v[i] = x

    def array(self) -> np.ndarray:
        return self._v.reshape(self._grid.shape)

    def ptr(self):
        return self._v.ctypes.data_as(C.c_void_p)


class IntervalField:
    """Per-node [lo, hi] per disturbance channel (interval_field.hpp:11-42)."""

    def __init__(self, grid: Grid, channels: int = 0, lo=None, hi=None, constant=None):
        self._grid = grid
        self._constant = list(constant) if constant is not None else None
        if constant is not None:
            self._lo = self._hi = None
        else:
            self._lo = [ScalarField(grid, None if lo is None else lo[c]) for c in range(channels)]
            self._hi = [ScalarField(grid, None if hi is None else hi[c]) for c in range(channels)]

    @staticmethod
    def constant(grid: Grid, bounds: Sequence[Interval]) -> "IntervalField":
        b = [x if isinstance(x, Interval) else Interval(*x) for x in bounds]
        for x in b:
            if not (x.lo <= x.hi):
                raise InvalidArgument("IntervalField: lo > hi")
        return IntervalField(grid, constant=b)

    def grid(self) -> Grid:
        return self._grid

    def channels(self) -> int:
        return len(self._constant) if self._constant is not None else len(self._lo)

    def is_constant(self) -> bool:
        return self._constant is not None

    def lo(self, ch: int) -> ScalarField:
        if self._constant is not None:
            return ScalarField(self._grid, fill=self._constant[ch].lo)
        return self._lo[ch]

    def hi(self, ch: int) -> ScalarField:
        if self._constant is not None:
            return ScalarField(self._grid, fill=self._constant[ch].hi)
        return self._hi[ch]

    def at_node(self, ch: int, lin: int) -> Interval:
        if self._constant is not None:
            return self._constant[ch]
        return Interval(float(self._lo[ch][lin]), float(self._hi[ch][lin]))

    def validate(self):
        for c in range(self.channels()):
            if not np.all(self.lo(c).values() <= self.hi(c).values()):
                raise SolverRuntimeError("IntervalField: lo > hi at a node")

    def to_c(self) -> abi.HjbDbounds:
        d = abi.HjbDbounds()
        d.channels = self.channels()
        if self._constant is not None:
            d.per_node = 0
            for c, b in enumerate(self._constant):
                d.constant[c].lo = b.lo
                d.constant[c].hi = b.hi
        else:
            d.per_node = 1
            for c in range(d.channels):
                d.lo[c] = self._lo[c].values().ctypes.data_as(C.POINTER(C.c_double))
                d.hi[c] = self._hi[c].values().ctypes.data_as(C.POINTER(C.c_double))
        return d


# ------------------------------------------------------------------ models
def _term(kind=abi.TERM_NONE, axis=0, scale=0.0):
    return (kind, axis, scale)


class DynamicsModel:
    """Control-affine model with box inputs (dynamics.hpp:37-59).

    Subclasses describe drift as up to two single-coordinate terms per row
    (the separable form every reference model has) plus constant B, C.
    """

    name_ = "model"

    def state_dim(self) -> int:
        raise NotImplementedError

    def control_dim(self) -> int:
        raise NotImplementedError

    def disturbance_dim(self) -> int:
        raise NotImplementedError

    def name(self) -> str:
        return self.name_

    def control_bounds(self) -> list[Interval]:
        raise NotImplementedError

    def drift_terms(self) -> list[list[tuple]]:
        raise NotImplementedError

    def control_matrix(self) -> np.ndarray:
        return np.zeros((self.state_dim(), self.control_dim()))

    def disturbance_matrix(self) -> np.ndarray:
        return np.zeros((self.state_dim(), self.disturbance_dim()))

    def disturbance_rows(self) -> list[int]:
        return []

    def to_c(self) -> abi.HjbModel:
        m = abi.HjbModel()
        m.state_dim, m.control_dim, m.disturbance_dim = (
            self.state_dim(), self.control_dim(), self.disturbance_dim())
        for i, terms in enumerate(self.drift_terms()):
            for t, (kind, axis, scale) in enumerate(terms):
                m.drift[i][t].kind = kind
                m.drift[i][t].axis = axis
                m.drift[i][t].scale = scale
        B, Cm = self.control_matrix(), self.disturbance_matrix()
        for i in range(self.state_dim()):
            for j in range(self.control_dim()):
                m.control[i][j] = float(B[i, j])
            for k in range(self.disturbance_dim()):
                m.disturbance[i][k] = float(Cm[i, k])
        for j, b in enumerate(self.control_bounds()):
            m.ubounds[j].lo = b.lo
            m.ubounds[j].hi = b.hi
        return m

    # point evaluations in the reference's own arithmetic (used by tests)
    def drift_at(self, x) -> np.ndarray:
        out = np.zeros(self.state_dim())
        for i, terms in enumerate(self.drift_terms()):
            v = 0.0
            for t, (kind, axis, scale) in enumerate(terms):
                if kind == abi.TERM_NONE:
                    continue
                tv = {abi.TERM_COORD: lambda: scale * x[axis],
                      abi.TERM_TAN: lambda: scale * math.tan(x[axis]),
                      abi.TERM_CONST: lambda: scale}[kind]()
                v = tv if t == 0 else v + tv
            out[i] = v
        return out


@dataclass
class Quad2DParams:
    k_thrust: float = 19.6
    k_offset: float = 0.0
    gravity: float = -9.8


class Quad2DVert(DynamicsModel):
    """x1' = x2, x2' = k_T u + g + k_0 + d (dynamics.hpp:102-125, dynamics.cpp:126-132)."""

    name_ = "quad2d_vert"
    Params = Quad2DParams

    def __init__(self, p: Quad2DParams | None = None):
        self.p = p or Quad2DParams()

    def state_dim(self):
        return 2

    def control_dim(self):
        return 1

    def disturbance_dim(self):
        return 1

    def control_bounds(self):
        return [Interval(0.0, 1.0)]

    def disturbance_rows(self):
        return [1]

    def drift_terms(self):
        return [[_term(abi.TERM_COORD, 1, 1.0)],
                [_term(abi.TERM_CONST, 0, self.p.gravity + self.p.k_offset)]]

    def control_matrix(self):
        B = np.zeros((2, 1))
        B[1, 0] = self.p.k_thrust
        return B

    def disturbance_matrix(self):
        Cm = np.zeros((2, 1))
        Cm[1, 0] = 1.0
        return Cm


@dataclass
class Planar4DParams:
    d0: float = 10.0
    d1: float = 8.0
    n0: float = 10.0
    gravity: float = 9.8
    max_angle_cmd: float = 0.2443


class NearHoverPlanar4D(DynamicsModel):
    """(p, v, theta, omega) planar subsystem (dynamics.hpp:133-162, dynamics.cpp:134-143).

    ``d_row`` selects the state row the wind enters: 1 (reference default,
    v' = g tan(theta) + d) or 0 (BASELINE.json configs 2-5, p' = v + d).
    """

    Params = Planar4DParams

    def __init__(self, axis: str = "x", p: Planar4DParams | None = None, d_row: int = 1):
        if d_row not in (0, 1):
            raise InvalidArgument("NearHoverPlanar4D: d_row must be 0 or 1")
        self.axis = axis
        self.p = p or Planar4DParams()
        self.d_row = d_row

    def name(self):
        return f"near_hover_{self.axis}4d"

    def state_dim(self):
        return 4

    def control_dim(self):
        return 1

    def disturbance_dim(self):
        return 1

    def control_bounds(self):
        return [Interval(-self.p.max_angle_cmd, self.p.max_angle_cmd)]

    def disturbance_rows(self):
        return [self.d_row]

    def drift_terms(self):
        p = self.p
        return [[_term(abi.TERM_COORD, 1, 1.0)],
                [_term(abi.TERM_TAN, 2, p.gravity)],
                [_term(abi.TERM_COORD, 2, -p.d1), _term(abi.TERM_COORD, 3, 1.0)],
                [_term(abi.TERM_COORD, 2, -p.d0)]]

    def control_matrix(self):
        B = np.zeros((4, 1))
        B[3, 0] = self.p.n0
        return B

    def disturbance_matrix(self):
        Cm = np.zeros((4, 1))
        Cm[self.d_row, 0] = 1.0
        return Cm


@dataclass
class Vertical2DParams:
    gravity: float = 9.8
    thrust_gain: float = 1.0
    thrust_frac_lo: float = 0.6
    thrust_frac_hi: float = 1.4


class NearHoverVertical2D(DynamicsModel):
    """p_z' = v_z, v_z' = k_T T - g + d (dynamics.hpp:170-197, dynamics.cpp:145-151)."""

    name_ = "near_hover_z2d"
    Params = Vertical2DParams

    def __init__(self, p: Vertical2DParams | None = None):
        self.p = p or Vertical2DParams()

    def state_dim(self):
        return 2

    def control_dim(self):
        return 1

    def disturbance_dim(self):
        return 1

    def control_bounds(self):
        w = self.p.gravity / self.p.thrust_gain
        return [Interval(self.p.thrust_frac_lo * w, self.p.thrust_frac_hi * w)]

    def disturbance_rows(self):
        return [1]

    def drift_terms(self):
        return [[_term(abi.TERM_COORD, 1, 1.0)], [_term(abi.TERM_CONST, 0, -self.p.gravity)]]

    def control_matrix(self):
        B = np.zeros((2, 1))
        B[1, 0] = self.p.thrust_gain
        return B

    def disturbance_matrix(self):
        Cm = np.zeros((2, 1))
        Cm[1, 0] = 1.0
        return Cm


@dataclass
class DoubleIntegratorParams:
    a_min: float = -1.0
    a_max: float = 1.0


class DoubleIntegrator(DynamicsModel):
    """(p, v), v' = a + d (dynamics.hpp:201-223, dynamics.cpp:153-158)."""

    name_ = "double_integrator"
    Params = DoubleIntegratorParams

    def __init__(self, p: DoubleIntegratorParams | None = None):
        self.p = p or DoubleIntegratorParams()

    def state_dim(self):
        return 2

    def control_dim(self):
        return 1

    def disturbance_dim(self):
        return 1

    def control_bounds(self):
        return [Interval(self.p.a_min, self.p.a_max)]

    def disturbance_rows(self):
        return [1]

    def drift_terms(self):
        return [[_term(abi.TERM_COORD, 1, 1.0)], []]

    def control_matrix(self):
        B = np.zeros((2, 1))
        B[1, 0] = 1.0
        return B

    def disturbance_matrix(self):
        Cm = np.zeros((2, 1))
        Cm[1, 0] = 1.0
        return Cm


class TwinDoubleIntegrator(DynamicsModel):
    """Two stacked double integrators (dynamics.hpp:227-244, dynamics.cpp:160-168)."""

    name_ = "twin_double_integrator"

    def __init__(self, p: DoubleIntegratorParams | None = None):
        self.p = p or DoubleIntegratorParams()

    def state_dim(self):
        return 4

    def control_dim(self):
        return 2

    def disturbance_dim(self):
        return 2

    def control_bounds(self):
        return [Interval(self.p.a_min, self.p.a_max), Interval(self.p.a_min, self.p.a_max)]

    def disturbance_rows(self):
        return [1, 3]

    def drift_terms(self):
        return [[_term(abi.TERM_COORD, 1, 1.0)], [], [_term(abi.TERM_COORD, 3, 1.0)], []]

    def control_matrix(self):
        B = np.zeros((4, 2))
        B[1, 0] = 1.0
        B[3, 1] = 1.0
        return B

    def disturbance_matrix(self):
        Cm = np.zeros((4, 2))
        Cm[1, 0] = 1.0
        Cm[3, 1] = 1.0
        return Cm


class ConstantAdvection(DynamicsModel):
    """Drift-only model xdot_i = speed_i (the reference's test model,
    proj/tests/test_solver.cpp:14-29)."""

    name_ = "advection"

    def __init__(self, speed: Sequence[float]):
        self.speed = [float(s) for s in speed]

    def state_dim(self):
        return len(self.speed)

    def control_dim(self):
        return 0

    def disturbance_dim(self):
        return 0

    def control_bounds(self):
        return []

    def drift_terms(self):
        return [[_term(abi.TERM_CONST, 0, s)] for s in self.speed]


class SeparableAffineModel(DynamicsModel):
    """A user-defined control-affine model in the separable form the C ABI
    takes (``hjb_model``, include/hjb.h): per row up to two drift terms
    ``(kind, axis, scale)`` with kind one of ``abi.TERM_COORD`` (scale*x[axis]),
    ``abi.TERM_TAN`` (scale*tan(x[axis])) or ``abi.TERM_CONST`` (scale), and
    constant control / disturbance matrices B, C — the structure every
    reference model has (dynamics.cpp:126-198).  4D models whose rows do not
    depend on x0 run the fast 4D kernel (compiled shapes or the run-time-shape
    variant); the rest run the generic kernel."""

    name_ = "separable_affine"

    def __init__(self, drift: Sequence[Sequence[tuple]], control=None, disturbance=None,
                 control_bounds: Sequence[Interval] = ()):
        self.drift = [[_term(*t) for t in row] for row in drift]
        n = len(self.drift)
        self.B = np.zeros((n, 0)) if control is None else np.asarray(control, dtype=np.float64)
        self.C = (np.zeros((n, 0)) if disturbance is None
                  else np.asarray(disturbance, dtype=np.float64))
        self.ub = list(control_bounds)
        if self.B.shape[0] != n or self.C.shape[0] != n or len(self.ub) != self.B.shape[1]:
            raise ValueError("SeparableAffineModel: inconsistent row / input counts")
        if any(len(row) > 2 for row in self.drift):
            raise ValueError("SeparableAffineModel: at most two drift terms per row")

    def state_dim(self):
        return len(self.drift)

    def control_dim(self):
        return self.B.shape[1]

    def disturbance_dim(self):
        return self.C.shape[1]

    def control_bounds(self):
        return list(self.ub)

    def disturbance_rows(self):
        return [i for i in range(self.state_dim()) if np.any(self.C[i] != 0.0)]

    def drift_terms(self):
        return [list(row) for row in self.drift]

    def control_matrix(self):
        return self.B.copy()

    def disturbance_matrix(self):
        return self.C.copy()


class NearHover10D(DynamicsModel):
    """Stacked x/y planar + z vertical model (dynamics.hpp:250-271).  Grids of
    rank 10 exceed the device kernels; it exists for decomposition (the solver
    runs its 4D/4D/2D subsystems)."""

    name_ = "near_hover_10d"

    def __init__(self, planar: Planar4DParams | None = None, vert: Vertical2DParams | None = None):
        self.x = NearHoverPlanar4D("x", planar)
        self.y = NearHoverPlanar4D("y", planar)
        self.z = NearHoverVertical2D(vert)

    def state_dim(self):
        return 10

    def control_dim(self):
        return 3

    def disturbance_dim(self):
        return 3

    def control_bounds(self):
        return [self.x.control_bounds()[0], self.y.control_bounds()[0], self.z.control_bounds()[0]]

    def disturbance_rows(self):
        return [1, 5, 9]

    def drift_terms(self):
        def shift(terms, off):
            return [[(k, a + off if k in (abi.TERM_COORD, abi.TERM_TAN) else a, s) for (k, a, s) in row]
                    for row in terms]
        return shift(self.x.drift_terms(), 0) + shift(self.y.drift_terms(), 4) + shift(self.z.drift_terms(), 8)

    def control_matrix(self):
        B = np.zeros((10, 3))
        B[0:4, 0:1] = self.x.control_matrix()
        B[4:8, 1:2] = self.y.control_matrix()
        B[8:10, 2:3] = self.z.control_matrix()
        return B

    def disturbance_matrix(self):
        Cm = np.zeros((10, 3))
        Cm[0:4, 0:1] = self.x.disturbance_matrix()
        Cm[4:8, 1:2] = self.y.disturbance_matrix()
        Cm[8:10, 2:3] = self.z.disturbance_matrix()
        return Cm


def make_model(name: str) -> DynamicsModel:
    """make_model, dynamics.cpp:200-209."""
    table = {
        "quad2d_vert": lambda: Quad2DVert(),
        "near_hover_x4d": lambda: NearHoverPlanar4D("x"),
        "near_hover_y4d": lambda: NearHoverPlanar4D("y"),
        "near_hover_z2d": lambda: NearHoverVertical2D(),
        "near_hover_10d": lambda: NearHover10D(),
        "double_integrator": lambda: DoubleIntegrator(),
        "twin_double_integrator": lambda: TwinDoubleIntegrator(),
    }
    if name not in table:
        raise InvalidArgument("unknown model: " + name)
    return table[name]()


# ------------------------------------------------------------------ solver
GODUNOV = "godunov"
LAX_FRIEDRICHS = "lax_friedrichs"
PER_NODE = "per_node"
GLOBAL = "global"


@dataclass
class SolveConfig:
    """solver.hpp:12-25 plus B200 extensions (orders, horizon)."""
    cfl_factor: float = 0.8
    tolerance: float = 1e-3
    max_iters: int = 20000
    scheme: str = GODUNOV
    dissipation: str = PER_NODE
    threads: int = 0
    spatial_order: int = 1
    time_order: int = 1
    time_horizon: float = 0.0
    flags: int = 0  # HJB_FLAG_FORCE_HO = 1: ENO/RK machinery at order 1 (verification)

    def validate(self):
        if not (self.cfl_factor > 0.0) or self.cfl_factor > 1.0:
            raise InvalidArgument("SolveConfig: cfl_factor must be in (0,1]")
        if not (self.tolerance > 0.0):
            raise InvalidArgument("SolveConfig: tolerance must be > 0")

    def to_c(self) -> abi.HjbSolveConfig:
        c = abi.HjbSolveConfig()
        c.cfl_factor = self.cfl_factor
        c.tolerance = self.tolerance
        c.max_iters = int(self.max_iters)
        c.scheme = abi.GODUNOV if self.scheme == GODUNOV else abi.LAX_FRIEDRICHS
        c.dissipation = abi.PER_NODE if self.dissipation == PER_NODE else abi.GLOBAL
        c.spatial_order = self.spatial_order
        c.time_order = self.time_order
        c.time_horizon = self.time_horizon
        c.threads = self.threads
        c.flags = self.flags
        return c


@dataclass
class SolveResult:
    value: ScalarField
    iterations: int = 0
    dt: float = 0.0
    wall_seconds: float = 0.0
    converged: bool = False
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    wall_ms_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    nodes_per_sweep: int = 0
    final_residual: float = 0.0
    kernel: str = ""  # the kernel family that ran the sweeps (HJB_KERNEL_*)


KERNELS = {0: "none", 1: "generic", 2: "fast4d", 3: "fast4d_multisweep", 4: "small2d",
           5: "ho_generic", 6: "ho4d", 7: "small2d_ho", 8: "fast4d_gen"}


@dataclass
class CoarseToFineResult:
    coarse: SolveResult
    fine: SolveResult
    wall_seconds: float = 0.0


def _ctx(ctx):
    return (ctx or default_context()).handle


def _c_result(cap: int):
    r = abi.HjbSolveResult()
    rh = np.zeros(max(cap, 0), dtype=np.float64)
    wh = np.zeros(max(cap, 0), dtype=np.float64)
    r.residual_history = rh.ctypes.data_as(C.POINTER(C.c_double))
    r.wall_ms_history = wh.ctypes.data_as(C.POINTER(C.c_double))
    r.history_capacity = cap
    return r, rh, wh


def _to_result(grid, value, r, rh, wh) -> SolveResult:
    n = min(int(r.iterations), int(r.history_capacity))
    return SolveResult(value=ScalarField(grid, value, check=False), iterations=int(r.iterations),
                       dt=float(r.dt), wall_seconds=float(r.wall_seconds),
                       converged=bool(r.converged), residual_history=rh[:n].copy(),
                       wall_ms_history=wh[:n].copy(), nodes_per_sweep=int(r.nodes_per_sweep),
                       final_residual=float(r.final_residual),
                       kernel=KERNELS.get(int(r.kernel), str(int(r.kernel))))


def cfl_dt(grid: Grid, model: DynamicsModel, dbounds: IntervalField, cfl_factor: float,
           threads: int = 0, ctx: Context | None = None) -> float:
    """solver.hpp:48-49."""
    lib = abi.load()
    if not (dbounds.grid() == grid):
        raise InvalidArgument("solver: disturbance bounds grid mismatch")
    out = C.c_double()
    g, m, d = grid.to_c(), model.to_c(), dbounds.to_c()
    _check(lib.hjb_cfl_dt(_ctx(ctx), C.byref(g), C.byref(m), C.byref(d), cfl_factor, C.byref(out)))
    return out.value


def _target_ok(target, grid):
    if target is not None and not (target.grid() == grid):
        raise InvalidArgument("solve: target grid mismatch")


def vi_step(value: ScalarField, constraint: ScalarField, model: DynamicsModel,
            dbounds: IntervalField, dt: float, cfg: SolveConfig | None = None,
            ctx: Context | None = None, target: ScalarField | None = None) -> ScalarField:
    """solver.hpp:55-57.  ``target`` (extension, no reference counterpart):
    reach-avoid update max(c, min(l, stepped)) against the target field l."""
    cfg = cfg or SolveConfig()
    _target_ok(target, value.grid())
    if not (value.grid() == constraint.grid()):
        raise InvalidArgument("vi_step: value/constraint grid mismatch")
    if not (dbounds.grid() == value.grid()):
        raise InvalidArgument("solver: disturbance bounds grid mismatch")
    lib = abi.load()
    out = np.empty(value.size(), dtype=np.float64)
    g, m, d, c = value.grid().to_c(), model.to_c(), dbounds.to_c(), cfg.to_c()
    if target is not None:
        c.target = target.ptr()
    _check(lib.hjb_vi_step(_ctx(ctx), C.byref(g), C.byref(m), C.byref(d), value.ptr(),
                           constraint.ptr(), dt, C.byref(c), out.ctypes.data_as(C.c_void_p)))
    return ScalarField(value.grid(), out, check=False)


def solve(init: ScalarField, constraint: ScalarField, model: DynamicsModel,
          dbounds: IntervalField, cfg: SolveConfig | None = None,
          ctx: Context | None = None, history_capacity: int | None = None,
          out: np.ndarray | None = None, target: ScalarField | None = None) -> SolveResult:
    """solver.hpp:63-65: iterate vi_step to a fixed point on the GPU.

    ``out`` (optional, float64, grid size, C-contiguous) receives V*; pass a
    page-locked array to make the device->host copy a direct DMA.
    ``target`` (extension; the reference has the avoid set only,
    solver.cpp:178-179): every update becomes the reach-avoid
    max(c, min(l, V + dt*H)) against the target field l."""
    cfg = cfg or SolveConfig()
    cfg.validate()
    _target_ok(target, init.grid())
    if not (init.grid() == constraint.grid()):
        raise InvalidArgument("solve: init/constraint grid mismatch")
    if not (dbounds.grid() == init.grid()):
        raise InvalidArgument("solver: disturbance bounds grid mismatch")
    lib = abi.load()
    cap = int(cfg.max_iters if history_capacity is None else history_capacity)
    r, rh, wh = _c_result(cap)
    if out is None:
        out = np.empty(init.size(), dtype=np.float64)
    elif (out.dtype != np.float64 or out.size != init.size() or not out.flags.c_contiguous
          or not out.flags.writeable):
        raise InvalidArgument("solve: out must be a writeable C-contiguous float64 array of grid size")
    out = out.reshape(-1)
    g, m, d, c = init.grid().to_c(), model.to_c(), dbounds.to_c(), cfg.to_c()
    if target is not None:
        c.target = target.ptr()
    _check(lib.hjb_solve(_ctx(ctx), C.byref(g), C.byref(m), C.byref(d), init.ptr(),
                         constraint.ptr(), C.byref(c), out.ctypes.data_as(C.c_void_p), C.byref(r)))
    return _to_result(init.grid(), out, r, rh, wh)


def solve_coarse_to_fine(constraint_fine: ScalarField, model: DynamicsModel,
                         dbounds_fine: IntervalField, coarse_grid: Grid,
                         cfg: SolveConfig | None = None,
                         warm_init_fine: ScalarField | None = None,
                         ctx: Context | None = None) -> CoarseToFineResult:
    """solver.hpp:70-74, on the device end to end."""
    cfg = cfg or SolveConfig()
    cfg.validate()
    fg = constraint_fine.grid()
    if coarse_grid.ndims() != fg.ndims():
        raise InvalidArgument("solve_coarse_to_fine: grid rank mismatch")
    lib = abi.load()
    cap = int(cfg.max_iters)
    rc_, rhc, whc = _c_result(cap)
    rf_, rhf, whf = _c_result(cap)
    cout = np.empty(coarse_grid.size(), dtype=np.float64)
    fout = np.empty(fg.size(), dtype=np.float64)
    wall = C.c_double()
    g, cg, m, d, c = fg.to_c(), coarse_grid.to_c(), model.to_c(), dbounds_fine.to_c(), cfg.to_c()
    warm = warm_init_fine.ptr() if warm_init_fine is not None else None
    _check(lib.hjb_solve_coarse_to_fine(
        _ctx(ctx), C.byref(g), C.byref(m), C.byref(d), constraint_fine.ptr(), C.byref(cg),
        C.byref(c), warm, cout.ctypes.data_as(C.c_void_p), C.byref(rc_),
        fout.ctypes.data_as(C.c_void_p), C.byref(rf_), C.byref(wall)))
    return CoarseToFineResult(coarse=_to_result(coarse_grid, cout, rc_, rhc, whc),
                              fine=_to_result(fg, fout, rf_, rhf, whf), wall_seconds=wall.value)


@dataclass
class MultiLevelResult:
    levels: list  # SolveResult per level, coarse to fine
    wall_seconds: float = 0.0


def solve_multilevel(constraint_fine: ScalarField, model: DynamicsModel,
                     dbounds_fine: IntervalField, coarse_grids: Sequence[Grid],
                     cfg: SolveConfig | None = None,
                     warm_init_fine: ScalarField | None = None,
                     ctx: Context | None = None) -> MultiLevelResult:
    """N-level adaptive solve (coarse grids listed coarse to fine, then the fine
    grid of constraint_fine), generalising solve_coarse_to_fine
    (solver.cpp:387-425); device-resident end to end."""
    cfg = cfg or SolveConfig()
    cfg.validate()
    grids = list(coarse_grids) + [constraint_fine.grid()]
    for g in grids:
        if g.ndims() != constraint_fine.grid().ndims():
            raise InvalidArgument("solve_coarse_to_fine: grid rank mismatch")
    lib = abi.load()
    nl = len(grids)
    cg = (abi.HjbGrid * nl)(*[g.to_c() for g in grids])
    res = (abi.HjbSolveResult * nl)()
    keep = []
    for l in range(nl):
        rh = np.zeros(int(cfg.max_iters))
        wh = np.zeros(int(cfg.max_iters))
        keep.append((rh, wh))
        res[l].residual_history = rh.ctypes.data_as(C.POINTER(C.c_double))
        res[l].wall_ms_history = wh.ctypes.data_as(C.POINTER(C.c_double))
        res[l].history_capacity = int(cfg.max_iters)
    outs = [np.empty(g.size()) for g in grids]
    optr = (C.c_void_p * nl)(*[o.ctypes.data for o in outs])
    wall = C.c_double()
    m, d, c = model.to_c(), dbounds_fine.to_c(), cfg.to_c()
    warm = warm_init_fine.ptr() if warm_init_fine is not None else None
    _check(lib.hjb_solve_multilevel(_ctx(ctx), nl, cg, C.byref(m), C.byref(d), constraint_fine.ptr(),
                                    C.byref(c), warm, optr, res, C.byref(wall)))
    return MultiLevelResult([_to_result(grids[l], outs[l], res[l], *keep[l]) for l in range(nl)],
                            wall.value)


def solve_multilevel_dev(grids: Sequence[Grid], model: DynamicsModel,
                         dbounds_fine: IntervalField, c_fine_ptr: int,
                         cfg: SolveConfig | None = None, out_ptrs: Sequence[int] | None = None,
                         warm_ptr: int = 0, ctx: Context | None = None,
                         history_capacity: int = 0) -> MultiLevelResult:
    """hjb_solve_multilevel_dev: the N-level chain with every field in HBM
    (grids coarse to fine, the last one c_fine's); out_ptrs[l] (device, may
    be 0) receive V*_l.  Results carry no host value."""
    cfg = cfg or SolveConfig()
    cfg.validate()
    lib = abi.load()
    nl = len(grids)
    cg = (abi.HjbGrid * nl)(*[g.to_c() for g in grids])
    res = (abi.HjbSolveResult * nl)()
    keep = []
    for l in range(nl):
        rh = np.zeros(int(history_capacity))
        wh = np.zeros(int(history_capacity))
        keep.append((rh, wh))
        res[l].residual_history = rh.ctypes.data_as(C.POINTER(C.c_double))
        res[l].wall_ms_history = wh.ctypes.data_as(C.POINTER(C.c_double))
        res[l].history_capacity = int(history_capacity)
    optr = (C.c_void_p * nl)(*[(out_ptrs[l] if out_ptrs else 0) or None for l in range(nl)])
    wall = C.c_double()
    m, d, c = model.to_c(), dbounds_fine.to_c(), cfg.to_c()
    _check(lib.hjb_solve_multilevel_dev(_ctx(ctx), nl, cg, C.byref(m), C.byref(d),
                                        C.c_void_p(c_fine_ptr), C.byref(c),
                                        C.c_void_p(warm_ptr) if warm_ptr else None, optr, res,
                                        C.byref(wall)))
    out = []
    for l in range(nl):
        r = res[l]
        n = min(int(r.iterations), int(r.history_capacity))
        out.append(SolveResult(value=None, iterations=int(r.iterations), dt=float(r.dt),
                               wall_seconds=float(r.wall_seconds), converged=bool(r.converged),
                               residual_history=keep[l][0][:n].copy(),
                               wall_ms_history=keep[l][1][:n].copy(),
                               nodes_per_sweep=int(r.nodes_per_sweep),
                               final_residual=float(r.final_residual)))
    return MultiLevelResult(out, wall.value)


def resample(f, target: Grid, ctx: Context | None = None):
    """grid.hpp:108-109 (ScalarField) and solver.hpp:77 (IntervalField)."""
    if isinstance(f, IntervalField):
        if f.is_constant():
            lo = [resample(f.lo(c), target, ctx).values() for c in range(f.channels())]
            hi = [resample(f.hi(c), target, ctx).values() for c in range(f.channels())]
        else:
            lo = [resample(f.lo(c), target, ctx).values() for c in range(f.channels())]
            hi = [resample(f.hi(c), target, ctx).values() for c in range(f.channels())]
        return IntervalField(target, f.channels(), lo=lo, hi=hi)
    if target.ndims() != f.grid().ndims():
        raise InvalidArgument("resample: dimension mismatch")
    lib = abi.load()
    out = np.empty(target.size(), dtype=np.float64)
    sg, dg = f.grid().to_c(), target.to_c()
    _check(lib.hjb_resample(_ctx(ctx), C.byref(sg), f.ptr(), C.byref(dg),
                            out.ctypes.data_as(C.c_void_p)))
    return ScalarField(target, out, check=False)


def max_adjacent_jump(f: ScalarField, ctx: Context | None = None) -> float:
    """grid.hpp:104."""
    lib = abi.load()
    out = C.c_double()
    g = f.grid().to_c()
    _check(lib.hjb_max_adjacent_jump(_ctx(ctx), C.byref(g), f.ptr(), C.byref(out)))
    return out.value


def seed_from(src: ScalarField, target: Grid, constraint: ScalarField,
              ctx: Context | None = None) -> ScalarField:
    """The seed_from lambda of solver.cpp:404-411 as a device kernel."""
    lib = abi.load()
    out = np.empty(target.size(), dtype=np.float64)
    sg, dg = src.grid().to_c(), target.to_c()
    _check(lib.hjb_seed_from(_ctx(ctx), C.byref(sg), src.ptr(), C.byref(dg), constraint.ptr(),
                             out.ctypes.data_as(C.c_void_p)))
    return ScalarField(target, out, check=False)


def signed_distance_band(grid: Grid, dim: int, lo: float, hi: float,
                         ctx: Context | None = None) -> ScalarField:
    """levelset.hpp:31."""
    lib = abi.load()
    out = np.empty(grid.size(), dtype=np.float64)
    g = grid.to_c()
    _check(lib.hjb_signed_distance_band(_ctx(ctx), C.byref(g), int(dim), float(lo), float(hi),
                                        out.ctypes.data_as(C.c_void_p)))
    return ScalarField(grid, out, check=False)


def field_max(a: ScalarField, b: ScalarField) -> ScalarField:
    """levelset.cpp:81-95 semantics (std::max); host-side set algebra helper."""
    if not (a.grid() == b.grid()):
        raise InvalidArgument("field_max: grid mismatch")
    x, y = a.values(), b.values()
    return ScalarField(a.grid(), np.where(x < y, y, x), check=False)


def field_min(a: ScalarField, b: ScalarField) -> ScalarField:
    if not (a.grid() == b.grid()):
        raise InvalidArgument("field_min: grid mismatch")
    x, y = a.values(), b.values()
    return ScalarField(a.grid(), np.where(y < x, y, x), check=False)


# ------------------------------------------------- device-resident entry points
def solve_dev(grid: Grid, model: DynamicsModel, dbounds: IntervalField, init_ptr: int,
              c_ptr: int, out_ptr: int, cfg: SolveConfig | None = None,
              ctx: Context | None = None, history_capacity: int = 0,
              target_ptr: int = 0) -> SolveResult:
    """hjb_solve_dev: init/c/out are device pointers (e.g. torch CUDA tensors'
    data_ptr()); the value stays in HBM.  Returns the result metadata with an
    empty value field."""
    cfg = cfg or SolveConfig()
    lib = abi.load()
    r, rh, wh = _c_result(int(history_capacity))
    g, m, d, c = grid.to_c(), model.to_c(), dbounds.to_c(), cfg.to_c()
    if target_ptr:
        c.target = C.c_void_p(target_ptr)
    _check(lib.hjb_solve_dev(_ctx(ctx), C.byref(g), C.byref(m), C.byref(d), C.c_void_p(init_ptr),
                             C.c_void_p(c_ptr), C.byref(c), C.c_void_p(out_ptr), C.byref(r)))
    n = min(int(r.iterations), int(r.history_capacity))
    return SolveResult(value=None, iterations=int(r.iterations), dt=float(r.dt),
                       wall_seconds=float(r.wall_seconds), converged=bool(r.converged),
                       residual_history=rh[:n].copy(), wall_ms_history=wh[:n].copy(),
                       nodes_per_sweep=int(r.nodes_per_sweep), final_residual=float(r.final_residual),
                       kernel=KERNELS.get(int(r.kernel), str(int(r.kernel))))


def signed_distance_band_dev(grid: Grid, dim: int, lo: float, hi: float, out_ptr: int,
                             ctx: Context | None = None) -> None:
    lib = abi.load()
    g = grid.to_c()
    _check(lib.hjb_signed_distance_band_dev(_ctx(ctx), C.byref(g), int(dim), float(lo), float(hi),
                                            C.c_void_p(out_ptr)))


def field_max_dev(n: int, a_ptr: int, b_ptr: int, out_ptr: int, ctx: Context | None = None) -> None:
    lib = abi.load()
    _check(lib.hjb_field_max_dev(_ctx(ctx), int(n), C.c_void_p(a_ptr), C.c_void_p(b_ptr),
                                 C.c_void_p(out_ptr)))


def field_min_dev(n: int, a_ptr: int, b_ptr: int, out_ptr: int, ctx: Context | None = None) -> None:
    """field_min (levelset.cpp:84-86) on device pointers."""
    lib = abi.load()
    _check(lib.hjb_field_min_dev(_ctx(ctx), int(n), C.c_void_p(a_ptr), C.c_void_p(b_ptr),
                                 C.c_void_p(out_ptr)))


def field_negate_dev(n: int, a_ptr: int, out_ptr: int, ctx: Context | None = None) -> None:
    """out = -a: the complement of a level-set field (obstacle -> avoid set)."""
    lib = abi.load()
    _check(lib.hjb_field_negate_dev(_ctx(ctx), int(n), C.c_void_p(a_ptr), C.c_void_p(out_ptr)))


# SafetyFilter / Decomposition (safety.hpp, decomposition.hpp) live in
# safety.py; re-exported here so the reference's names resolve from hjsafe.
from .safety import (CombinedDecision, Decomposition, FilterDecision, SafetyFilter,  # noqa: E402
                     Subsystem, Violation, project, scatter)
# GP disturbance bounds (gp.hpp) live in gp.py.
from . import gp as gp_module  # noqa: E402
from .gp import (DisturbanceMeasurement, GpConfig, GpHyperparams, GpModel,  # noqa: E402
                 ViolationCheck, bounds_on_grid, bounds_on_grid_dev, violation_check)
