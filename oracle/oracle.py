"""TEST INFRASTRUCTURE ONLY — Python loader of the CPU oracles.

Two checkers live here, both CPU-only:
  * ``Restatement``: oracle/libhjoracle.so, the plain-C restatement of the
    reference hot path (oracle/hj_oracle.c);
  * ``Reference``: oracle/_ref/libhjref.so, the reference's own sources
    compiled in place (oracle/Makefile `ref`) behind oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module.  The product (paper_2101_05916_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2101_05916_b200 import abi
from paper_2101_05916_b200 import hjsafe as hj

HERE = Path(__file__).resolve().parent
RESTATEMENT_SO = HERE / "libhjoracle.so"
REF_SO = HERE / "_ref" / "libhjref.so"
REF_SRC = Path("/root/reference/proj")


def build(ref: bool = True) -> None:
    """Compile the restatement (always) and _ref (when the reference sources exist)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    if ref and REF_SRC.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


P = C.POINTER
_vp = C.c_void_p
_d = C.c_double


class ScanResult(C.Structure):
    _fields_ = [("max_speed_sum", C.c_double), ("max_alpha", C.c_double * abi.HJB_MAX_STATE),
                ("separable", C.c_int32)]


def _arr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def _vals(f) -> np.ndarray:
    return np.ascontiguousarray(f.values() if hasattr(f, "values") else f, dtype=np.float64)


class Restatement:
    """oracle/libhjoracle.so (plain C, OpenMP over node chunks)."""

    def __init__(self, path: os.PathLike | None = None, threads: int = 0):
        p = Path(path) if path else RESTATEMENT_SO
        if not p.exists():
            build(ref=False)
        self.lib = C.CDLL(str(p))
        L = self.lib
        L.hjo_last_error.restype = C.c_char_p
        L.hjo_set_threads.argtypes = [C.c_int]
        L.hjo_scan_alpha.argtypes = [P(abi.HjbGrid), P(abi.HjbModel), P(abi.HjbDbounds), P(ScanResult)]
        L.hjo_cfl_dt.argtypes = [P(abi.HjbGrid), P(abi.HjbModel), P(abi.HjbDbounds), _d, P(_d)]
        L.hjo_sweep.argtypes = [P(abi.HjbGrid), P(abi.HjbModel), P(abi.HjbDbounds), _vp, _vp, _d,
                                C.c_int32, _vp, _vp, P(_d)]
        L.hjo_vi_step.argtypes = [P(abi.HjbGrid), P(abi.HjbModel), P(abi.HjbDbounds), _vp, _vp, _d,
                                  P(abi.HjbSolveConfig), _vp]
        L.hjo_sweep_planes.argtypes = [P(abi.HjbGrid), P(abi.HjbModel), P(abi.HjbDbounds), _vp, _vp,
                                       _d, C.c_int32, _vp, C.c_int64, C.c_int64, _vp, P(_d)]
        L.hjo_solve.argtypes = [P(abi.HjbGrid), P(abi.HjbModel), P(abi.HjbDbounds), _vp, _vp,
                                P(abi.HjbSolveConfig), _vp, P(abi.HjbSolveResult)]
        L.hjo_interp.argtypes = [P(abi.HjbGrid), _vp, _vp, P(_d), P(C.c_int32)]
        L.hjo_resample.argtypes = [P(abi.HjbGrid), _vp, P(abi.HjbGrid), _vp]
        L.hjo_max_adjacent_jump.argtypes = [P(abi.HjbGrid), _vp, P(_d)]
        L.hjo_seed_from.argtypes = [P(abi.HjbGrid), _vp, P(abi.HjbGrid), _vp, _vp]
        L.hjo_solve_coarse_to_fine.argtypes = [P(abi.HjbGrid), P(abi.HjbModel), P(abi.HjbDbounds),
                                               _vp, P(abi.HjbGrid), P(abi.HjbSolveConfig), _vp, _vp,
                                               P(abi.HjbSolveResult), _vp, P(abi.HjbSolveResult)]
        L.hjo_solve_multilevel.argtypes = [C.c_int32, P(abi.HjbGrid), P(abi.HjbModel),
                                           P(abi.HjbDbounds), _vp, P(abi.HjbSolveConfig), _vp,
                                           P(_vp), P(abi.HjbSolveResult)]
        L.hjo_signed_distance_band.argtypes = [P(abi.HjbGrid), C.c_int32, _d, _d, _vp]
        L.hjo_signed_distance_box.argtypes = [P(abi.HjbGrid), _vp, _vp, _vp]
        L.hjo_hamiltonian.argtypes = [P(abi.HjbModel), _vp, _vp, P(abi.HjbInterval), P(_d)]
        L.hjo_flow_bounds.argtypes = [P(abi.HjbModel), _vp, P(abi.HjbInterval), _vp]
        L.hjo_ho_stage_planes.argtypes = [P(abi.HjbGrid), P(abi.HjbModel), P(abi.HjbDbounds),
                                          _vp, _vp, _vp, _d, C.c_int32, C.c_int32, C.c_int64,
                                          C.c_int64, _vp, P(_d)]
        L.hjo_filter_batch.argtypes = [P(abi.HjbGrid), P(abi.HjbModel), P(abi.HjbDbounds), _vp,
                                       C.c_int64, _vp, _vp, P(abi.HjbFilterConfig),
                                       P(abi.HjbFilterOut)]
        if threads:
            L.hjo_set_threads(threads)

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.lib.hjo_last_error().decode())

    def scan_alpha(self, grid, model, db):
        s = ScanResult()
        g, m, d = grid.to_c(), model.to_c(), db.to_c()
        self._chk(self.lib.hjo_scan_alpha(C.byref(g), C.byref(m), C.byref(d), C.byref(s)))
        return s.max_speed_sum, list(s.max_alpha)[:grid.ndims()], bool(s.separable)

    def cfl_dt(self, grid, model, db, cfl):
        out = C.c_double()
        g, m, d = grid.to_c(), model.to_c(), db.to_c()
        self._chk(self.lib.hjo_cfl_dt(C.byref(g), C.byref(m), C.byref(d), cfl, C.byref(out)))
        return out.value

    def sweep(self, grid, model, db, v, c, dt, scheme=abi.GODUNOV, global_alpha=None):
        v, c = _vals(v), _vals(c)
        out = np.empty_like(v)
        mx = C.c_double()
        ga = None
        if global_alpha is not None:
            ga_arr = np.zeros(abi.HJB_MAX_STATE)
            ga_arr[:len(global_alpha)] = global_alpha
            ga = _arr(ga_arr)
        g, m, d = grid.to_c(), model.to_c(), db.to_c()
        self._chk(self.lib.hjo_sweep(C.byref(g), C.byref(m), C.byref(d), _arr(v), _arr(c), dt,
                                     scheme, ga, _arr(out), C.byref(mx)))
        return out, mx.value

    def sweep_planes(self, grid, model, db, v, c, dt, pb, pe, out):
        """In-place update of planes [pb, pe) of `out` (numpy, full grid size)."""
        mx = C.c_double()
        g, m, d = grid.to_c(), model.to_c(), db.to_c()
        self._chk(self.lib.hjo_sweep_planes(C.byref(g), C.byref(m), C.byref(d), _arr(_vals(v)),
                                            _arr(_vals(c)), dt, abi.GODUNOV, None, pb, pe,
                                            _arr(out), C.byref(mx)))
        return mx.value

    def ho_stage_planes(self, grid, model, db, vs, vn, c, dt, order, kind, pb, pe, out):
        """One Godunov ENO/TVD-RK stage on planes [pb, pe) of `out` (numpy,
        full grid size); returns max|out - vn| over those planes."""
        mx = C.c_double()
        g, m, d = grid.to_c(), model.to_c(), db.to_c()
        self._chk(self.lib.hjo_ho_stage_planes(C.byref(g), C.byref(m), C.byref(d), _arr(vs),
                                               _arr(vn), _arr(_vals(c)), dt, order, kind, pb, pe,
                                               _arr(out), C.byref(mx)))
        return mx.value

    def vi_step(self, v, c, model, db, dt, cfg=None, target=None):
        cfg = cfg or hj.SolveConfig()
        grid = v.grid()
        vv, cc = _vals(v), _vals(c)
        out = np.empty_like(vv)
        g, m, d, k = grid.to_c(), model.to_c(), db.to_c(), cfg.to_c()
        tv = _vals(target) if target is not None else None
        if tv is not None:
            k.target = tv.ctypes.data_as(C.c_void_p)
        self._chk(self.lib.hjo_vi_step(C.byref(g), C.byref(m), C.byref(d), _arr(vv), _arr(cc), dt,
                                       C.byref(k), _arr(out)))
        return out

    def solve(self, init, c, model, db, cfg, history_capacity=None, target=None):
        """hjo_solve; ``target`` (extension, parity unpinned): the reach-avoid
        update max(c, min(l, stepped)) of every sweep / RK stage."""
        grid = init.grid()
        cap = int(cfg.max_iters if history_capacity is None else history_capacity)
        r, rh, wh = hj._c_result(cap)
        iv, cv = _vals(init), _vals(c)
        out = np.empty_like(iv)
        g, m, d, k = grid.to_c(), model.to_c(), db.to_c(), cfg.to_c()
        tv = _vals(target) if target is not None else None
        if tv is not None:
            k.target = tv.ctypes.data_as(C.c_void_p)
        self._chk(self.lib.hjo_solve(C.byref(g), C.byref(m), C.byref(d), _arr(iv), _arr(cv),
                                     C.byref(k), _arr(out), C.byref(r)))
        return hj._to_result(grid, out, r, rh, wh)

    def solve_coarse_to_fine(self, c_fine, model, db, coarse_grid, cfg, warm=None):
        fg = c_fine.grid()
        cap = int(cfg.max_iters)
        rc_, rhc, whc = hj._c_result(cap)
        rf_, rhf, whf = hj._c_result(cap)
        cout = np.empty(coarse_grid.size())
        fout = np.empty(fg.size())
        g, cg, m, d, k = fg.to_c(), coarse_grid.to_c(), model.to_c(), db.to_c(), cfg.to_c()
        wv = _vals(warm) if warm is not None else None
        self._chk(self.lib.hjo_solve_coarse_to_fine(
            C.byref(g), C.byref(m), C.byref(d), _arr(_vals(c_fine)), C.byref(cg), C.byref(k),
            _arr(wv) if wv is not None else None, _arr(cout), C.byref(rc_), _arr(fout), C.byref(rf_)))
        return hj.CoarseToFineResult(coarse=hj._to_result(coarse_grid, cout, rc_, rhc, whc),
                                     fine=hj._to_result(fg, fout, rf_, rhf, whf))

    def solve_multilevel(self, c_fine, model, db, coarse_grids, cfg, warm=None):
        grids = list(coarse_grids) + [c_fine.grid()]
        nl = len(grids)
        cg = (abi.HjbGrid * nl)(*[g.to_c() for g in grids])
        res = (abi.HjbSolveResult * nl)()
        keep = []
        for l in range(nl):
            r, rh, wh = hj._c_result(int(cfg.max_iters))
            res[l] = r
            keep.append((rh, wh))
        outs = [np.empty(g.size()) for g in grids]
        optr = (C.c_void_p * nl)(*[o.ctypes.data for o in outs])
        m, d, k = model.to_c(), db.to_c(), cfg.to_c()
        wv = _vals(warm) if warm is not None else None
        self._chk(self.lib.hjo_solve_multilevel(nl, cg, C.byref(m), C.byref(d), _arr(_vals(c_fine)),
                                                C.byref(k), _arr(wv) if wv is not None else None,
                                                optr, res))
        return hj.MultiLevelResult([hj._to_result(grids[l], outs[l], res[l], *keep[l])
                                    for l in range(nl)])

    def interp(self, f, x):
        val = C.c_double()
        ood = C.c_int32()
        xv = np.asarray(x, dtype=np.float64)
        g = f.grid().to_c()
        self._chk(self.lib.hjo_interp(C.byref(g), _arr(_vals(f)), _arr(xv), C.byref(val), C.byref(ood)))
        return val.value, bool(ood.value)

    def resample(self, f, target):
        out = np.empty(target.size())
        sg, dg = f.grid().to_c(), target.to_c()
        self._chk(self.lib.hjo_resample(C.byref(sg), _arr(_vals(f)), C.byref(dg), _arr(out)))
        return out

    def max_adjacent_jump(self, f):
        out = C.c_double()
        g = f.grid().to_c()
        self._chk(self.lib.hjo_max_adjacent_jump(C.byref(g), _arr(_vals(f)), C.byref(out)))
        return out.value

    def seed_from(self, src, target, c_dst):
        out = np.empty(target.size())
        sg, dg = src.grid().to_c(), target.to_c()
        self._chk(self.lib.hjo_seed_from(C.byref(sg), _arr(_vals(src)), C.byref(dg),
                                         _arr(_vals(c_dst)), _arr(out)))
        return out

    def signed_distance_band(self, grid, dim, lo, hi):
        out = np.empty(grid.size())
        g = grid.to_c()
        self._chk(self.lib.hjo_signed_distance_band(C.byref(g), dim, lo, hi, _arr(out)))
        return out

    def signed_distance_box(self, grid, lo, hi):
        out = np.empty(grid.size())
        lo = np.asarray(lo, dtype=np.float64)
        hi = np.asarray(hi, dtype=np.float64)
        g = grid.to_c()
        self._chk(self.lib.hjo_signed_distance_box(C.byref(g), _arr(lo), _arr(hi), _arr(out)))
        return out

    def hamiltonian(self, model, x, p, db):
        h = C.c_double()
        xv, pv = np.asarray(x, dtype=np.float64), np.asarray(p, dtype=np.float64)
        dbs = (abi.HjbInterval * abi.HJB_MAX_INPUT)(*[abi.HjbInterval(b.lo, b.hi) for b in db])
        m = model.to_c()
        self._chk(self.lib.hjo_hamiltonian(C.byref(m), _arr(xv), _arr(pv), dbs, C.byref(h)))
        return h.value

    def flow_bounds(self, model, x, db):
        out = np.zeros(abi.HJB_MAX_STATE)
        xv = np.asarray(x, dtype=np.float64)
        dbs = (abi.HjbInterval * abi.HJB_MAX_INPUT)(*[abi.HjbInterval(b.lo, b.hi) for b in db])
        m = model.to_c()
        self._chk(self.lib.hjo_flow_bounds(C.byref(m), _arr(xv), dbs, _arr(out)))
        return out[:model.state_dim()]


# ----------------------------------------------------------- reference
def _filter_out(nq, m, p):
    arrs = dict(value=np.empty(nq), band=np.empty(nq), control=np.empty((nq, m)),
                worst_disturbance=np.empty((nq, p)), flags=np.empty(nq, dtype=np.uint8))
    out = abi.HjbFilterOut(*(arrs[k].ctypes.data for k in
                             ("value", "band", "control", "worst_disturbance", "flags")))
    return arrs, out


def _restatement_filter_batch(self, v, model, db, x, u_perf=None, mode=abi.FILTER_OPTIMAL,
                              eta_floor=1e-5, lam=0.0):
    """hjo_filter_batch: SafetyFilter::optimal_control / filter restated."""
    grid = v.grid()
    X = np.ascontiguousarray(np.asarray(x, dtype=np.float64)).reshape(-1, grid.ndims())
    nq, m, p = X.shape[0], model.control_dim(), model.disturbance_dim()
    U = (np.ascontiguousarray(np.asarray(u_perf, dtype=np.float64)).reshape(nq, m)
         if u_perf is not None else np.zeros((nq, m)))
    arrs, out = _filter_out(nq, m, p)
    cfg = abi.HjbFilterConfig(mode, 0, eta_floor, lam)
    g, mm, d = grid.to_c(), model.to_c(), db.to_c()
    vv = _vals(v)
    self._chk(self.lib.hjo_filter_batch(C.byref(g), C.byref(mm), C.byref(d), _arr(vv), nq,
                                        _arr(X), _arr(U), C.byref(cfg), C.byref(out)))
    return arrs


Restatement.filter_batch = _restatement_filter_batch


def _restatement_gp_predict(self, model, X):
    """hjo_gp_predict per point (GpModel::predict restated): (mean, var)."""
    Xa = np.ascontiguousarray(np.asarray(X, dtype=np.float64)).reshape(-1, model.input_dim())
    cm = model.to_c()
    mean = np.empty(Xa.shape[0])
    var = np.empty(Xa.shape[0])
    fn = self.lib.hjo_gp_predict
    fn.argtypes = [P(abi.HjbGpModel), _vp, P(_d), P(_d)]
    for q in range(Xa.shape[0]):
        m, v = C.c_double(), C.c_double()
        self._chk(fn(C.byref(cm), _arr(Xa[q]), C.byref(m), C.byref(v)))
        mean[q], var[q] = m.value, v.value
    return mean, var


def _restatement_gp_bounds_on_grid(self, models, input_dims, grid, confidence=3.0):
    """hjo_gp_bounds_on_grid (bounds_on_grid restated, per node): (lo[], hi[])."""
    nch = len(models)
    arr = (abi.HjbGpModel * max(1, nch))()
    for ch, (m, dims) in enumerate(zip(models, input_dims)):
        arr[ch] = m.to_c(dims)
    lo = [np.empty(grid.size()) for _ in range(nch)]
    hi = [np.empty(grid.size()) for _ in range(nch)]
    plo = (_vp * max(1, nch))(*[a.ctypes.data for a in lo])
    phi = (_vp * max(1, nch))(*[a.ctypes.data for a in hi])
    fn = self.lib.hjo_gp_bounds_on_grid
    fn.argtypes = [P(abi.HjbGrid), C.c_int32, P(abi.HjbGpModel), _d, P(_vp), P(_vp)]
    g = grid.to_c()
    self._chk(fn(C.byref(g), nch, arr, float(confidence), plo, phi))
    return lo, hi


Restatement.gp_predict = _restatement_gp_predict
Restatement.gp_bounds_on_grid = _restatement_gp_bounds_on_grid


class ModelSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d_row", C.c_int32), ("p", C.c_double * 10)]


class RefResult(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("dt", C.c_double), ("wall_seconds", C.c_double),
                ("converged", C.c_int32), ("reserved", C.c_int32), ("nodes_per_sweep", C.c_int64),
                ("residual_history", P(C.c_double)), ("history_capacity", C.c_int64),
                ("wall_ms_history", P(C.c_double))]


def model_spec(model) -> ModelSpec:
    s = ModelSpec()
    if isinstance(model, hj.Quad2DVert):
        s.kind, vals = 0, [model.p.k_thrust, model.p.k_offset, model.p.gravity]
    elif isinstance(model, hj.NearHoverPlanar4D):
        p = model.p
        s.kind, vals = 1, [p.d0, p.d1, p.n0, p.gravity, p.max_angle_cmd]
        s.d_row = model.d_row
    elif isinstance(model, hj.NearHoverVertical2D):
        p = model.p
        s.kind, vals = 2, [p.gravity, p.thrust_gain, p.thrust_frac_lo, p.thrust_frac_hi]
    elif isinstance(model, hj.TwinDoubleIntegrator):
        s.kind, vals = 4, [model.p.a_min, model.p.a_max]
    elif isinstance(model, hj.DoubleIntegrator):
        s.kind, vals = 3, [model.p.a_min, model.p.a_max]
    elif isinstance(model, hj.ConstantAdvection):
        s.kind, vals = 5, list(model.speed)
        s.d_row = len(model.speed)
    else:
        raise TypeError(f"no reference model for {type(model).__name__}")
    for i, v in enumerate(vals):
        s.p[i] = v
    return s


class Reference:
    """oracle/_ref/libhjref.so: the reference's own code, compiled in place."""

    def __init__(self, path: os.PathLike | None = None):
        p = Path(path) if path else REF_SO
        if not p.exists():
            raise FileNotFoundError(f"{p} missing (build with `make -C oracle ref` where "
                                    "/root/reference exists)")
        self.lib = C.CDLL(str(p))
        L = self.lib
        E = [C.c_char_p, C.c_int]
        L.hjr_cfl_dt.argtypes = [P(abi.HjbGrid), P(ModelSpec), P(abi.HjbDbounds), _d, C.c_uint, P(_d)] + E
        L.hjr_vi_step.argtypes = [P(abi.HjbGrid), P(ModelSpec), P(abi.HjbDbounds), _vp, _vp, _d,
                                  P(abi.HjbSolveConfig), _vp] + E
        L.hjr_solve.argtypes = [P(abi.HjbGrid), P(ModelSpec), P(abi.HjbDbounds), _vp, _vp,
                                P(abi.HjbSolveConfig), _vp, P(RefResult)] + E
        L.hjr_solve_coarse_to_fine.argtypes = [P(abi.HjbGrid), P(ModelSpec), P(abi.HjbDbounds), _vp,
                                               P(abi.HjbGrid), P(abi.HjbSolveConfig), _vp, _vp,
                                               P(RefResult), _vp, P(RefResult)] + E
        L.hjr_solve_coarse_to_fine_w.argtypes = [P(abi.HjbGrid), P(ModelSpec), P(abi.HjbDbounds),
                                                 _vp, P(abi.HjbGrid), P(abi.HjbSolveConfig),
                                                 C.c_void_p, _vp, _vp, P(RefResult), _vp,
                                                 P(RefResult)] + E
        L.hjr_resample.argtypes = [P(abi.HjbGrid), _vp, P(abi.HjbGrid), _vp] + E
        L.hjr_max_adjacent_jump.argtypes = [P(abi.HjbGrid), _vp, P(_d)] + E
        L.hjr_signed_distance_band.argtypes = [P(abi.HjbGrid), C.c_int32, _d, _d, _vp] + E
        L.hjr_field_max.argtypes = [P(abi.HjbGrid), _vp, _vp, _vp] + E
        L.hjr_field_min.argtypes = [P(abi.HjbGrid), _vp, _vp, _vp] + E
        L.hjr_signed_distance_box.argtypes = [P(abi.HjbGrid), _vp, _vp, _vp] + E
        L.hjr_hamiltonian.argtypes = [P(ModelSpec), _vp, _vp, P(abi.HjbInterval), P(_d)] + E
        L.hjr_flow_bounds.argtypes = [P(ModelSpec), _vp, P(abi.HjbInterval), _vp] + E
        L.hjr_write_hjvf.argtypes = [C.c_char_p, P(abi.HjbGrid), _vp] + E
        L.hjr_filter_batch.argtypes = [P(abi.HjbGrid), P(ModelSpec), P(abi.HjbDbounds), _vp,
                                       C.c_int64, _vp, _vp, C.c_int32, _d, C.c_int64, _vp, P(_d),
                                       P(C.c_int32), P(abi.HjbFilterOut)] + E
        L.hjr_decomposition_batch.argtypes = [C.c_int32, _vp, _vp, _vp, _vp, _vp, C.c_int32,
                                              C.c_int32, C.c_int32, _d, C.c_int64, _vp,
                                              C.c_int64, _vp, _vp, P(_d), P(C.c_int32), _vp, _vp,
                                              _vp, _vp, _vp] + E

    def _call(self, fn, *args):
        err = C.create_string_buffer(512)
        rc = fn(*args, err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())

    def cfl_dt(self, grid, model, db, cfl, threads=0):
        out = C.c_double()
        g, m, d = grid.to_c(), model_spec(model), db.to_c()
        self._call(self.lib.hjr_cfl_dt, C.byref(g), C.byref(m), C.byref(d), cfl, threads, C.byref(out))
        return out.value

    def vi_step(self, v, c, model, db, dt, cfg=None):
        cfg = cfg or hj.SolveConfig()
        vv, cc = _vals(v), _vals(c)
        out = np.empty_like(vv)
        g, m, d, k = v.grid().to_c(), model_spec(model), db.to_c(), cfg.to_c()
        self._call(self.lib.hjr_vi_step, C.byref(g), C.byref(m), C.byref(d), _arr(vv), _arr(cc), dt,
                   C.byref(k), _arr(out))
        return out

    def solve(self, init, c, model, db, cfg):
        grid = init.grid()
        cap = int(cfg.max_iters)
        hist = np.zeros(max(cap, 1))
        whist = np.zeros(max(cap, 1))
        r = RefResult()
        r.residual_history = hist.ctypes.data_as(P(C.c_double))
        r.wall_ms_history = whist.ctypes.data_as(P(C.c_double))
        r.history_capacity = cap
        iv, cv = _vals(init), _vals(c)
        out = np.empty_like(iv)
        g, m, d, k = grid.to_c(), model_spec(model), db.to_c(), cfg.to_c()
        self._call(self.lib.hjr_solve, C.byref(g), C.byref(m), C.byref(d), _arr(iv), _arr(cv),
                   C.byref(k), _arr(out), C.byref(r))
        n = min(int(r.iterations), cap)
        return hj.SolveResult(value=hj.ScalarField(grid, out, check=False), iterations=int(r.iterations),
                              dt=r.dt, wall_seconds=r.wall_seconds, converged=bool(r.converged),
                              residual_history=hist[:n].copy(), wall_ms_history=whist[:n].copy(),
                              nodes_per_sweep=int(r.nodes_per_sweep))

    def solve_coarse_to_fine(self, c_fine, model, db, coarse_grid, cfg, warm=None):
        """The reference's own ``solve_coarse_to_fine`` (solver.cpp:387-425).

        ``warm`` is a ScalarField on ANY grid (the reference's seed_from
        resamples from the warm field's own grid, :404-414)."""
        fg = c_fine.grid()
        cap = int(cfg.max_iters)
        res = []
        for _ in range(2):
            h = np.zeros(max(cap, 1))
            r = RefResult()
            r.residual_history = h.ctypes.data_as(P(C.c_double))
            r.history_capacity = cap
            res.append((r, h))
        cout = np.empty(coarse_grid.size())
        fout = np.empty(fg.size())
        g, cg, m, d, k = fg.to_c(), coarse_grid.to_c(), model_spec(model), db.to_c(), cfg.to_c()
        wv = _vals(warm) if warm is not None else None
        wg = warm.grid().to_c() if warm is not None else None
        self._call(self.lib.hjr_solve_coarse_to_fine_w, C.byref(g), C.byref(m), C.byref(d),
                   _arr(_vals(c_fine)), C.byref(cg), C.byref(k),
                   C.cast(C.pointer(wg), C.c_void_p) if wg is not None else None,
                   _arr(wv) if wv is not None else None,
                   _arr(cout), C.byref(res[0][0]), _arr(fout), C.byref(res[1][0]))
        out = []
        for (r, h), grid, v in ((res[0], coarse_grid, cout), (res[1], fg, fout)):
            n = min(int(r.iterations), cap)
            out.append(hj.SolveResult(value=hj.ScalarField(grid, v, check=False),
                                      iterations=int(r.iterations), dt=r.dt,
                                      wall_seconds=r.wall_seconds, converged=bool(r.converged),
                                      residual_history=h[:n].copy()))
        return hj.CoarseToFineResult(coarse=out[0], fine=out[1])

    def solve_multilevel(self, c_fine, model, db, coarse_grids, cfg, warm=None):
        """N-level chain composed from the reference's own public pieces
        (SURVEY §8a row A10): levels 0..N-3 are ``resample`` of the fine
        constraint / bound fields (solver.cpp:378-385, grid.cpp:215-231) +
        ``solve``; the last two levels are the reference's own
        ``solve_coarse_to_fine`` warm-started from level N-3's V* (its private
        ``seed_from`` does the lowering, solver.cpp:404-414).  Only levels
        0..N-3 restate ``seed_from`` (max(resample - jump, c), the same
        expression) because the reference keeps it private."""
        grids = list(coarse_grids)
        fg = c_fine.grid()
        if not grids:
            return hj.MultiLevelResult([self.solve(c_fine, c_fine, model, db, cfg)])
        out = []
        prev = warm
        for l, g in enumerate(grids[:-1]):
            cl = hj.ScalarField(g, self.resample(c_fine, g), check=False)
            dl = self._resample_db(db, fg, g)
            if prev is None:
                init = cl
            else:
                a = self.resample(prev, g) - self.max_adjacent_jump(prev)
                init = hj.ScalarField(g, np.where(a < cl.values(), cl.values(), a), check=False)
            r = self.solve(init, cl, model, dl, cfg)
            out.append(r)
            prev = r.value
        ctf = self.solve_coarse_to_fine(c_fine, model, db, grids[-1], cfg, warm=prev)
        out += [ctf.coarse, ctf.fine]
        return hj.MultiLevelResult(out)

    def _resample_db(self, db, fg, g):
        """resample(IntervalField, Grid) (solver.cpp:378-385), channel by channel."""
        if db.channels() == 0:
            return hj.IntervalField.constant(g, [])
        lo, hi = [], []
        for ch in range(db.channels()):
            lo.append(self.resample(db.lo(ch), g))
            hi.append(self.resample(db.hi(ch), g))
        return hj.IntervalField(g, db.channels(), lo=lo, hi=hi)

    def resample(self, f, target):
        out = np.empty(target.size())
        sg, dg = f.grid().to_c(), target.to_c()
        self._call(self.lib.hjr_resample, C.byref(sg), _arr(_vals(f)), C.byref(dg), _arr(out))
        return out

    def max_adjacent_jump(self, f):
        out = C.c_double()
        g = f.grid().to_c()
        self._call(self.lib.hjr_max_adjacent_jump, C.byref(g), _arr(_vals(f)), C.byref(out))
        return out.value

    def signed_distance_band(self, grid, dim, lo, hi):
        out = np.empty(grid.size())
        g = grid.to_c()
        self._call(self.lib.hjr_signed_distance_band, C.byref(g), dim, lo, hi, _arr(out))
        return out

    def field_max(self, a, b):
        """levelset.cpp:80-82 (std::max per node)."""
        out = np.empty(a.grid().size())
        g = a.grid().to_c()
        self._call(self.lib.hjr_field_max, C.byref(g), _arr(_vals(a)), _arr(_vals(b)), _arr(out))
        return out

    def field_min(self, a, b):
        """levelset.cpp:84-86 (std::min per node)."""
        out = np.empty(a.grid().size())
        g = a.grid().to_c()
        self._call(self.lib.hjr_field_min, C.byref(g), _arr(_vals(a)), _arr(_vals(b)), _arr(out))
        return out

    def signed_distance_box(self, grid, lo, hi):
        out = np.empty(grid.size())
        g = grid.to_c()
        self._call(self.lib.hjr_signed_distance_box, C.byref(g), _arr(np.asarray(lo, float)),
                   _arr(np.asarray(hi, float)), _arr(out))
        return out

    def hamiltonian(self, model, x, p, db):
        h = C.c_double()
        dbs = (abi.HjbInterval * abi.HJB_MAX_INPUT)(*[abi.HjbInterval(b.lo, b.hi) for b in db])
        m = model_spec(model)
        self._call(self.lib.hjr_hamiltonian, C.byref(m), _arr(np.asarray(x, float)),
                   _arr(np.asarray(p, float)), dbs, C.byref(h))
        return h.value

    def flow_bounds(self, model, x, db):
        out = np.zeros(abi.HJB_MAX_STATE)
        dbs = (abi.HjbInterval * abi.HJB_MAX_INPUT)(*[abi.HjbInterval(b.lo, b.hi) for b in db])
        m = model_spec(model)
        self._call(self.lib.hjr_flow_bounds, C.byref(m), _arr(np.asarray(x, float)), dbs, _arr(out))
        return out[:model.state_dim()]

    def write_hjvf(self, path, f):
        g = f.grid().to_c()
        self._call(self.lib.hjr_write_hjvf, str(path).encode(), C.byref(g), _arr(_vals(f)))


def _reference_filter_batch(self, v, model, db, x, u_perf=None, mode=abi.FILTER_OPTIMAL,
                            eta_floor=1e-5, violations=()):
    """The reference's own SafetyFilter: contract(violations) then per-query
    filter / optimal_control.  Returns (arrays, lambda, emergency)."""
    grid = v.grid()
    nd = grid.ndims()
    X = np.ascontiguousarray(np.asarray(x, dtype=np.float64)).reshape(-1, nd)
    nq, m, p = X.shape[0], model.control_dim(), model.disturbance_dim()
    U = (np.ascontiguousarray(np.asarray(u_perf, dtype=np.float64)).reshape(nq, m)
         if u_perf is not None else np.zeros((nq, m)))
    Vx = np.ascontiguousarray(np.asarray(violations, dtype=np.float64)).reshape(-1, nd)
    arrs, out = _filter_out(nq, m, p)
    lam, em = C.c_double(), C.c_int32()
    g, mm, d = grid.to_c(), model_spec(model), db.to_c()
    vv = _vals(v)
    self._call(self.lib.hjr_filter_batch, C.byref(g), C.byref(mm), C.byref(d), _arr(vv), nq,
               _arr(X), _arr(U), mode, eta_floor, Vx.shape[0], _arr(Vx), C.byref(lam),
               C.byref(em), C.byref(out))
    return arrs, lam.value, bool(em.value)


def _reference_decomposition_batch(self, subs, values, dbounds, full_dims, x, u_perf,
                                   eta_floor=1e-5, violations=()):
    """The reference's Decomposition over SafetyFilters (subs: hjsafe
    Subsystem list, values: converged ScalarFields, dbounds: IntervalFields)."""
    n, m, p = full_dims
    k = len(subs)
    grids = (abi.HjbGrid * k)(*[v.grid().to_c() for v in values])
    specs = (ModelSpec * k)(*[model_spec(s.model) for s in subs])
    dbs = (abi.HjbDbounds * k)(*[d.to_c() for d in dbounds])
    vals = [np.ascontiguousarray(_vals(v)) for v in values]
    vptr = (C.c_void_p * k)(*[a.ctypes.data for a in vals])
    maps = np.array([i for s in subs for i in (list(s.state_map) + list(s.control_map)
                                                 + list(s.disturbance_map))], dtype=np.int32)
    X = np.ascontiguousarray(np.asarray(x, dtype=np.float64)).reshape(-1, n)
    nq = X.shape[0]
    U = np.ascontiguousarray(np.asarray(u_perf, dtype=np.float64)).reshape(nq, m)
    Vx = np.ascontiguousarray(np.asarray(violations, dtype=np.float64)).reshape(-1, n)
    cv, val, band = np.empty(nq), np.empty(nq), np.empty(nq)
    ctl, flg = np.empty((nq, m)), np.empty(nq, dtype=np.uint8)
    lam, em = C.c_double(), C.c_int32()
    self._call(self.lib.hjr_decomposition_batch, k, grids, specs, dbs, vptr, _arr(maps), n, m, p,
               eta_floor, Vx.shape[0], _arr(Vx), nq, _arr(X), _arr(U), C.byref(lam), C.byref(em),
               _arr(cv), _arr(val), _arr(band), _arr(ctl), _arr(flg))
    return dict(combined_value=cv, value=val, band=band, control=ctl, flags=flg), lam.value, \
        bool(em.value)


Reference.filter_batch = _reference_filter_batch
Reference.decomposition_batch = _reference_decomposition_batch


def reference_available() -> bool:
    return REF_SO.exists()


REF_GP_SO = HERE / "_ref" / "libhjref_gp.so"


class ReferenceGp:
    """oracle/_ref/libhjref_gp.so: the reference's own GpModel::predict and
    bounds_on_grid (proj/src/gp.cpp:188-249), compiled in place behind
    oracle/gp_shim.cpp.  The model's factor is pushed into the reference's
    GpModel as given (its fit needs Eigen, absent here)."""

    def __init__(self, path: os.PathLike | None = None, threads: int = 0):
        p = Path(path) if path else REF_GP_SO
        if not p.exists():
            raise FileNotFoundError(f"{p} missing (build with `make -C oracle ref` where "
                                    "/root/reference exists)")
        self.lib = C.CDLL(str(p))
        self.threads = threads
        E = [C.c_char_p, C.c_int]
        self.lib.hjr_gp_predict.argtypes = [P(abi.HjbGpModel), C.c_int64, _vp, _vp, _vp] + E
        self.lib.hjr_gp_bounds_on_grid.argtypes = [P(abi.HjbGrid), C.c_int32, P(abi.HjbGpModel),
                                                   _d, C.c_uint, P(_vp), P(_vp)] + E

    @staticmethod
    def _call(fn, *args):
        buf = C.create_string_buffer(512)
        rc = fn(*args, buf, 512)
        if rc:
            raise OracleError(rc, buf.value.decode())

    def gp_predict(self, model, X):
        """GpModel::predict per point: (mean, latent variance)."""
        Xa = np.ascontiguousarray(np.asarray(X, dtype=np.float64)).reshape(-1, model.input_dim())
        cm = model.to_c()
        mean = np.empty(Xa.shape[0])
        var = np.empty(Xa.shape[0])
        self._call(self.lib.hjr_gp_predict, C.byref(cm), Xa.shape[0], _arr(Xa), _arr(mean),
                   _arr(var))
        return mean, var

    def gp_bounds_on_grid(self, models, input_dims, grid, confidence=3.0):
        """bounds_on_grid: (lo[ch][], hi[ch][])."""
        nch = len(models)
        arr = (abi.HjbGpModel * max(1, nch))()
        for ch, (m, dims) in enumerate(zip(models, input_dims)):
            arr[ch] = m.to_c(dims)
        lo = [np.empty(grid.size()) for _ in range(nch)]
        hi = [np.empty(grid.size()) for _ in range(nch)]
        plo = (_vp * max(1, nch))(*[a.ctypes.data for a in lo])
        phi = (_vp * max(1, nch))(*[a.ctypes.data for a in hi])
        g = grid.to_c()
        self._call(self.lib.hjr_gp_bounds_on_grid, C.byref(g), nch, arr, float(confidence),
                   self.threads, plo, phi)
        return lo, hi
