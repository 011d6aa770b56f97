"""The five BASELINE.json workloads, as seeded synthetic inputs.

Every input is analytic or seeded (no dataset is involved).  Decisions on the
points BASELINE.json leaves open are recorded here and in DESIGN.md §2:
  * 4D models put the wind on the position row (``d_row=0``, BASELINE text)
    with g = 9.81 and u in [-pi/9, pi/9];
  * config 1 maps ``u in [0, 2g/kT]`` onto NearHoverVertical2D with
    thrust_frac_lo = 0, thrust_frac_hi = 2 (control_bounds = frac * g/kT);
  * config 4 draws its 10 bound updates as 0.3 + 0.7*U with U from a
    GaussianRng-equivalent uniform (mt19937_64, ldexp(x>>11,-53),
    reference sim.cpp:17-19), seed 2101;
  * config 5 places 3 obstacle intervals on the x axis (centre in
    [-3.5, 3.5], half width in [0.15, 0.45], same generator, seed 5916);
    the avoid set is the union, i.e. c = max(band, -obstacle bands).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

from . import hjsafe as hj

MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the engine behind the reference's GaussianRng)."""

    def __init__(self, seed: int = 5489):
        self.mt = [0] * 312
        self.mti = 312
        self.mt[0] = seed & MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & MASK64

    def __call__(self) -> int:
        if self.mti >= 312:
            upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
            for i in range(312):
                x = (self.mt[i] & upper) | (self.mt[(i + 1) % 312] & lower)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[i] = self.mt[(i + 156) % 312] ^ xa
            self.mti = 0
        x = self.mt[self.mti]
        self.mti += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & MASK64


class UniformRng:
    """GaussianRng::uniform of the reference (sim.cpp:17-19)."""

    def __init__(self, seed: int):
        self.eng = MT19937_64(seed)

    def uniform(self) -> float:
        return math.ldexp(float(self.eng() >> 11), -53)


G = 9.81
WIND = 0.5


def planar_model() -> hj.NearHoverPlanar4D:
    return hj.NearHoverPlanar4D("x", hj.Planar4DParams(d0=10.0, d1=8.0, n0=10.0, gravity=G,
                                                       max_angle_cmd=math.pi / 9.0), d_row=0)


def vertical_model() -> hj.NearHoverVertical2D:
    return hj.NearHoverVertical2D(hj.Vertical2DParams(gravity=G, thrust_gain=0.91,
                                                      thrust_frac_lo=0.0, thrust_frac_hi=2.0))


def planar_grid(n: int) -> hj.Grid:
    return hj.Grid([(-5.0, 5.0, n), (-2.0, 2.0, n), (-0.35, 0.35, n), (-1.5, 1.5, n)])


def vertical_grid(n: int = 101) -> hj.Grid:
    return hj.Grid([(-2.0, 4.0, n), (-4.0, 4.0, n)])


@dataclass
class Workload:
    name: str
    grid: hj.Grid
    model: hj.DynamicsModel
    wind: float
    bands: list  # [(dim, lo, hi, sign)] combined with max; sign -1 = obstacle
    cfg: hj.SolveConfig = field(default_factory=hj.SolveConfig)

    def dbounds(self, wind: float | None = None) -> hj.IntervalField:
        w = self.wind if wind is None else wind
        return hj.IntervalField.constant(self.grid, [hj.Interval(-w, w)])

    def constraint_dev(self, out_ptr: int, scratch_ptr: int, ctx=None) -> None:
        """c on the device: signed_distance_band per listed band (obstacles
        negated: their complement), combined with field_max — the reference's
        set algebra (levelset.cpp:54-66, 80-82) as device kernels.  out /
        scratch: device buffers of grid size (float64)."""
        n = self.grid.size()
        for k, (dim, lo, hi, sign) in enumerate(self.bands):
            dst = out_ptr if k == 0 else scratch_ptr
            hj.signed_distance_band_dev(self.grid, dim, lo, hi, dst, ctx=ctx)
            if sign < 0:
                hj.field_negate_dev(n, dst, dst, ctx=ctx)
            if k > 0:
                hj.field_max_dev(n, out_ptr, scratch_ptr, out_ptr, ctx=ctx)

    def constraint(self, band: Callable, fmax: Callable):
        """c = max over the listed signed-distance bands (obstacles negated).

        ``band(grid, dim, lo, hi) -> ndarray`` and ``fmax(a, b)`` are supplied
        by the caller: device kernels in the product, the oracle in tests."""
        out = None
        for dim, lo, hi, sign in self.bands:
            f = band(self.grid, dim, lo, hi)
            if sign < 0:
                f = -f
            out = f if out is None else fmax(out, f)
        return out


def obstacles(seed: int = 5916, count: int = 3):
    rng = UniformRng(seed)
    out = []
    for _ in range(count):
        centre = -3.5 + 7.0 * rng.uniform()
        half = 0.15 + 0.30 * rng.uniform()
        out.append((centre - half, centre + half))
    return out


def bound_sequence(seed: int = 2101, count: int = 10):
    """Config 4: cold 0.5, warm 0.8, then 10 draws 0.3 + 0.7*U."""
    rng = UniformRng(seed)
    return [0.5, 0.8] + [0.3 + 0.7 * rng.uniform() for _ in range(count)]


def config1(tol: float = 1e-4) -> Workload:
    return Workload("cfg1_vertical2d_101", vertical_grid(101), vertical_model(), WIND,
                    [(0, 0.0, 3.0, 1)], hj.SolveConfig(cfl_factor=0.8, tolerance=tol))


def config2(n: int = 51, tol: float = 1e-4, max_iters: int = 20000) -> Workload:
    return Workload(f"cfg2_planar4d_{n}", planar_grid(n), planar_model(), WIND,
                    [(0, -4.0, 4.0, 1)],
                    hj.SolveConfig(cfl_factor=0.8, tolerance=tol, max_iters=max_iters))


def config3(n: int = 101, tol: float = 1e-4, max_iters: int = 20000) -> Workload:
    w = config2(n, tol, max_iters)
    w.name = f"cfg3_planar4d_{n}"
    return w


def config4_subsystems(n4: int = 71, n2: int = 101, tol: float = 1e-4):
    x = config2(n4, tol)
    x.name = f"cfg4_x4d_{n4}"
    y = config2(n4, tol)
    y.name = f"cfg4_y4d_{n4}"
    y.model = hj.NearHoverPlanar4D("y", planar_model().p, d_row=0)
    z = config1(tol)
    z.name = f"cfg4_z2d_{n2}"
    z.grid = vertical_grid(n2)
    return [z, x, y]


def config5(levels=(26, 51, 101), tol: float = 1e-4, wind: float = 0.6):
    out = []
    bands = [(0, -4.0, 4.0, 1)] + [(0, lo, hi, -1) for lo, hi in obstacles()]
    for n in levels:
        out.append(Workload(f"cfg5_planar4d_{n}", planar_grid(n), planar_model(), wind, list(bands),
                            hj.SolveConfig(cfl_factor=0.8, tolerance=tol)))
    return out
