"""ctypes mirror of the C ABI in ``include/hjb.h`` and the loader of ``libhjb.so``.

The structs below are field-for-field copies of the POD descriptors declared in
``include/hjb.h``; ``tests/test_abi.py`` checks their sizes against the header
and that every declared symbol is exported by the built library.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

HJB_MAX_DIMS = 6
HJB_MAX_STATE = 10
HJB_MAX_INPUT = 3
HJB_MAX_LEVELS = 8

HJB_OK = 0
HJB_ERR_INVALID_ARGUMENT = 1
HJB_ERR_RUNTIME = 2
HJB_ERR_CUDA = 3
HJB_ERR_UNSUPPORTED = 4
HJB_ERR_DIVERGED = 5
HJB_ERR_NCCL = 6

TERM_NONE, TERM_COORD, TERM_TAN, TERM_CONST, TERM_TABLE = 0, 1, 2, 3, 4
GODUNOV, LAX_FRIEDRICHS = 0, 1
PER_NODE, GLOBAL = 0, 1

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
HEADER = REPO_DIR / "include" / "hjb.h"
LIB_PATH = Path(os.environ["HJB_LIB"]) if os.environ.get("HJB_LIB") else PKG_DIR / "libhjb.so"


class GridDim(C.Structure):
    _fields_ = [("min", C.c_double), ("max", C.c_double), ("n", C.c_int64)]


class HjbGrid(C.Structure):
    _fields_ = [("ndims", C.c_int32), ("reserved", C.c_int32),
                ("dims", GridDim * HJB_MAX_DIMS)]


class HjbInterval(C.Structure):
    _fields_ = [("lo", C.c_double), ("hi", C.c_double)]


class DriftTerm(C.Structure):
    _fields_ = [("kind", C.c_int32), ("axis", C.c_int32), ("scale", C.c_double),
                ("table", C.POINTER(C.c_double))]


class HjbModel(C.Structure):
    _fields_ = [("state_dim", C.c_int32), ("control_dim", C.c_int32),
                ("disturbance_dim", C.c_int32), ("reserved", C.c_int32),
                ("drift", (DriftTerm * 2) * HJB_MAX_STATE),
                ("control", (C.c_double * HJB_MAX_INPUT) * HJB_MAX_STATE),
                ("disturbance", (C.c_double * HJB_MAX_INPUT) * HJB_MAX_STATE),
                ("ubounds", HjbInterval * HJB_MAX_INPUT)]


class HjbDbounds(C.Structure):
    _fields_ = [("channels", C.c_int32), ("per_node", C.c_int32),
                ("constant", HjbInterval * HJB_MAX_INPUT),
                ("lo", C.POINTER(C.c_double) * HJB_MAX_INPUT),
                ("hi", C.POINTER(C.c_double) * HJB_MAX_INPUT)]


class HjbSolveConfig(C.Structure):
    _fields_ = [("cfl_factor", C.c_double), ("tolerance", C.c_double),
                ("max_iters", C.c_int64), ("scheme", C.c_int32),
                ("dissipation", C.c_int32), ("spatial_order", C.c_int32),
                ("time_order", C.c_int32), ("time_horizon", C.c_double),
                ("threads", C.c_int32), ("flags", C.c_int32), ("target", C.c_void_p)]


class HjbSolveResult(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("dt", C.c_double),
                ("wall_seconds", C.c_double), ("converged", C.c_int32),
                ("kernel", C.c_int32), ("nodes_per_sweep", C.c_int64),
                ("final_residual", C.c_double),
                ("residual_history", C.POINTER(C.c_double)),
                ("wall_ms_history", C.POINTER(C.c_double)),
                ("history_capacity", C.c_int64)]


class HjbFilterConfig(C.Structure):
    _fields_ = [("mode", C.c_int32), ("reserved", C.c_int32), ("eta_floor", C.c_double),
                ("lambda_", C.c_double)]


class HjbFilterOut(C.Structure):
    _fields_ = [("value", C.c_void_p), ("band", C.c_void_p), ("control", C.c_void_p),
                ("worst_disturbance", C.c_void_p), ("flags", C.c_void_p)]


FILTER_OPTIMAL, FILTER_FILTER = 0, 1
FILTER_OVERRIDE, FILTER_DEGENERATE, FILTER_OOD = 1, 2, 4


class HjbGpModel(C.Structure):
    _fields_ = [("input_dim", C.c_int32), ("n_dims", C.c_int32),
                ("input_dims", C.c_int32 * HJB_MAX_DIMS), ("n_train", C.c_int64),
                ("signal_var", C.c_double), ("noise_var", C.c_double),
                ("lengthscales", C.c_double * HJB_MAX_DIMS),
                ("inputs", C.POINTER(C.c_double)), ("alpha", C.POINTER(C.c_double)),
                ("chol", C.POINTER(C.c_double))]


class HjbGpFitConfig(C.Structure):
    _fields_ = [("policy", C.c_int32), ("prior_n_lengthscales", C.c_int32),
                ("max_training", C.c_int64), ("search_subsample", C.c_int64),
                ("prior_signal_var", C.c_double), ("prior_noise_var", C.c_double),
                ("prior_lengthscales", C.c_double * HJB_MAX_DIMS)]


GP_FIXED, GP_SEARCH = 0, 1

P = C.POINTER
_d = C.c_double
_dp = P(C.c_double)
_vp = C.c_void_p
_i = C.c_int
_i32 = C.c_int32
_i64 = C.c_int64

# (name, restype, argtypes) for every function declared in include/hjb.h.
SIGNATURES = [
    ("hjb_version", C.c_char_p, []),
    ("hjb_last_error", C.c_char_p, []),
    ("hjb_solve_config_default", None, [P(HjbSolveConfig)]),
    ("hjb_context_create", _i, [_i, P(_vp)]),
    ("hjb_context_destroy", _i, [_vp]),
    ("hjb_device_count", _i, [P(_i)]),
    ("hjb_cfl_dt", _i, [_vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _d, _dp]),
    ("hjb_vi_step", _i, [_vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp, _vp, _d,
                         P(HjbSolveConfig), _vp]),
    ("hjb_solve", _i, [_vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp, _vp,
                       P(HjbSolveConfig), _vp, P(HjbSolveResult)]),
    ("hjb_solve_coarse_to_fine", _i, [_vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp,
                                      P(HjbGrid), P(HjbSolveConfig), _vp, _vp,
                                      P(HjbSolveResult), _vp, P(HjbSolveResult), _dp]),
    ("hjb_solve_multilevel", _i, [_vp, C.c_int32, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp,
                                  P(HjbSolveConfig), _vp, P(_vp), P(HjbSolveResult), _dp]),
    ("hjb_solve_multilevel_dev", _i, [_vp, C.c_int32, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp,
                                      P(HjbSolveConfig), _vp, P(_vp), P(HjbSolveResult), _dp]),
    ("hjb_resample", _i, [_vp, P(HjbGrid), _vp, P(HjbGrid), _vp]),
    ("hjb_max_adjacent_jump", _i, [_vp, P(HjbGrid), _vp, _dp]),
    ("hjb_seed_from", _i, [_vp, P(HjbGrid), _vp, P(HjbGrid), _vp, _vp]),
    ("hjb_signed_distance_band", _i, [_vp, P(HjbGrid), _i32, _d, _d, _vp]),
    ("hjb_vi_step_dev", _i, [_vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp, _vp, _d,
                             P(HjbSolveConfig), _vp]),
    ("hjb_solve_dev", _i, [_vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp, _vp,
                           P(HjbSolveConfig), _vp, P(HjbSolveResult)]),
    ("hjb_resample_dev", _i, [_vp, P(HjbGrid), _vp, P(HjbGrid), _vp]),
    ("hjb_max_adjacent_jump_dev", _i, [_vp, P(HjbGrid), _vp, _dp]),
    ("hjb_seed_from_dev", _i, [_vp, P(HjbGrid), _vp, P(HjbGrid), _vp, _vp]),
    ("hjb_signed_distance_band_dev", _i, [_vp, P(HjbGrid), _i32, _d, _d, _vp]),
    ("hjb_field_max_dev", _i, [_vp, _i64, _vp, _vp, _vp]),
    ("hjb_field_min_dev", _i, [_vp, _i64, _vp, _vp, _vp]),
    ("hjb_field_negate_dev", _i, [_vp, _i64, _vp, _vp]),
    ("hjb_slab_partition", _i, [_i64, _i32, _i32, P(_i64), P(_i64)]),
    ("hjb_slab_plan", _i, [_i64, _i32, _i32, _i32, P(_i64)]),
    ("hjb_nccl_unique_id", _i, [_vp]),
    ("hjb_comm_create", _i, [_vp, _i32, _i32, _vp, P(_vp)]),
    ("hjb_comm_destroy", _i, [_vp]),
    ("hjb_p2p_comm_create", _i, [_vp, _i32, _i32, P(_vp)]),
    ("hjb_comm_ctl_handle", _i, [_vp, _vp]),
    ("hjb_comm_open_peers", _i, [_vp, _vp]),
    ("hjb_solve_sharded_dev", _i, [_vp, _vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp, _vp,
                                   P(HjbSolveConfig), _vp, P(HjbSolveResult)]),
    ("hjb_solve_sharded_local_dev", _i, [_vp, _i32, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp,
                                         _vp, P(HjbSolveConfig), _vp, P(HjbSolveResult)]),
    ("hjb_sweep_planes_dev", _i, [_vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp, _vp, _i64,
                                  _i64, _d, _vp, _dp]),
    ("hjb_filter_batch", _i, [_vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp, _i64, _vp, _vp,
                              P(HjbFilterConfig), P(HjbFilterOut)]),
    ("hjb_filter_batch_dev", _i, [_vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp, _i64, _vp,
                                  _vp, P(HjbFilterConfig), P(HjbFilterOut)]),
    ("hjb_interp_batch_dev", _i, [_vp, P(HjbGrid), _vp, _i64, _vp, _vp, _vp]),
    ("hjb_field_reduce_dev", _i, [_vp, _i64, _vp, _dp, _dp]),
    ("hjb_malloc_dev", _i, [_vp, C.c_uint64, P(_vp)]),
    ("hjb_free_dev", _i, [_vp, _vp]),
    ("hjb_copy_h2d", _i, [_vp, _vp, _vp, C.c_uint64]),
    ("hjb_copy_d2h", _i, [_vp, _vp, _vp, C.c_uint64]),
    ("hjb_copy_d2d", _i, [_vp, _vp, _vp, C.c_uint64]),
    ("hjb_ho_stage_planes_dev", _i, [_vp, P(HjbGrid), P(HjbModel), P(HjbDbounds), _vp, _vp, _vp,
                                     _d, _i32, _i32, _i64, _i64, _vp, _dp]),
    ("hjb_gp_bounds_on_grid_dev", _i, [_vp, P(HjbGrid), _i32, P(HjbGpModel), _d, P(_vp),
                                       P(_vp)]),
    ("hjb_gp_bounds_on_grid", _i, [_vp, P(HjbGrid), _i32, P(HjbGpModel), _d, P(_vp), P(_vp)]),
    ("hjb_gp_predict_batch", _i, [_vp, P(HjbGpModel), _i64, _vp, _vp, _vp]),
    ("hjb_gp_fit", _i, [_i64, _i32, _vp, _vp, P(HjbGpFitConfig), _vp, _vp, _vp, P(HjbGpModel),
                        _dp]),
    ("hjb_context_stream", _vp, [_vp]),
    ("hjb_context_synchronize", _i, [_vp]),
    ("hjb_context_launch_count", _i64, [_vp]),
]


def header_functions(path: Path = HEADER) -> list[str]:
    """Names of every function declared in include/hjb.h (for the ABI test)."""
    text = path.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hjb_[a-z0-9_]+)\s*\(", text)))


_lib = None


class HjbLibraryMissing(RuntimeError):
    pass


def load(path: os.PathLike | None = None):
    """Load libhjb.so (built in-tree by __graft_entry__.build()).

    There is deliberately no fallback: a missing library is an error.
    """
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise HjbLibraryMissing(
            f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(p))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
