"""The C ABI: libhjb.so loads without a GPU, exports every symbol include/hjb.h
declares, the ctypes mirror matches the header's struct layouts, and compute
calls fail loudly (no CPU fallback) when no device is present."""
import ctypes as C
import subprocess
import tempfile
from pathlib import Path

import pytest

from paper_2101_05916_b200 import abi

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    from paper_2101_05916_b200 import build
    build.build()
    return abi.load()


def test_every_header_symbol_exported(lib):
    names = abi.header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    declared = {n for n, _, _ in abi.SIGNATURES}
    assert set(names) == declared, set(names) ^ declared


def test_struct_layouts_match_header():
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "hjb.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(hjb_grid), sizeof(hjb_model),
         sizeof(hjb_dbounds), sizeof(hjb_solve_config), sizeof(hjb_solve_result),
         sizeof(hjb_drift_term), offsetof(hjb_model, ubounds), offsetof(hjb_solve_result, history_capacity));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = Path(d) / "sz.c"
        c.write_text(src)
        exe = Path(d) / "sz"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), "-o", str(exe), str(c)], check=True)
        got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [C.sizeof(abi.HjbGrid), C.sizeof(abi.HjbModel), C.sizeof(abi.HjbDbounds),
            C.sizeof(abi.HjbSolveConfig), C.sizeof(abi.HjbSolveResult), C.sizeof(abi.DriftTerm),
            abi.HjbModel.ubounds.offset, abi.HjbSolveResult.history_capacity.offset]
    assert got == want


def test_defaults_match_reference(lib):
    """SolveConfig defaults, solver.hpp:13-22."""
    cfg = abi.HjbSolveConfig()
    lib.hjb_solve_config_default(C.byref(cfg))
    assert (cfg.cfl_factor, cfg.tolerance, cfg.max_iters) == (0.8, 1e-3, 20000)
    assert (cfg.scheme, cfg.dissipation, cfg.spatial_order, cfg.time_order) == (0, 0, 1, 1)


def test_no_device_fails_loudly(lib):
    n = C.c_int(-1)
    lib.hjb_device_count(C.byref(n))
    if n.value > 0:
        pytest.skip("a CUDA device is present")
    h = C.c_void_p()
    rc = lib.hjb_context_create(0, C.byref(h))
    assert rc == abi.HJB_ERR_CUDA
    assert lib.hjb_last_error()


def test_kernels_are_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(abi.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_kernel_family_ids_match_header():
    """hjb_solve_result.kernel ids (include/hjb.h) and their names in hjsafe."""
    import re
    from pathlib import Path
    from paper_2101_05916_b200 import hjsafe as hj
    hdr = (Path(__file__).resolve().parent.parent / "include" / "hjb.h").read_text()
    ids = {int(v): k for k, v in re.findall(r"#define HJB_KERNEL_(\w+) (\d+)", hdr)}
    assert set(ids) == set(hj.KERNELS)
    assert ids[8] == "FAST4D_GEN" and hj.KERNELS[8] == "fast4d_gen"


def test_separable_affine_model_descriptor():
    """SeparableAffineModel -> hjb_model: drift terms, B, C and control bounds
    as given; inconsistent shapes are rejected on the host."""
    import numpy as np
    import pytest
    from paper_2101_05916_b200 import abi
    from paper_2101_05916_b200 import hjsafe as hj
    B = np.zeros((4, 1))
    B[3, 0] = 4.0
    C = np.zeros((4, 1))
    C[0, 0] = 1.0
    m = hj.SeparableAffineModel(
        [[(abi.TERM_COORD, 3, 1.0)], [(abi.TERM_COORD, 2, -2.0), (abi.TERM_COORD, 3, 0.5)],
         [(abi.TERM_TAN, 2, 9.8)], [(abi.TERM_CONST, 0, -1.5)]], B, C, [hj.Interval(-0.4, 0.4)])
    d = m.to_c()
    assert (d.state_dim, d.control_dim, d.disturbance_dim) == (4, 1, 1)
    assert d.drift[1][1].kind == abi.TERM_COORD and d.drift[1][1].axis == 3
    assert d.drift[1][1].scale == 0.5 and d.drift[2][0].kind == abi.TERM_TAN
    assert d.control[3][0] == 4.0 and d.disturbance[0][0] == 1.0
    assert (d.ubounds[0].lo, d.ubounds[0].hi) == (-0.4, 0.4)
    assert m.disturbance_rows() == [0]
    assert m.drift_at([0.0, 0.0, 0.0, 2.0])[0] == 2.0
    with pytest.raises(ValueError):
        hj.SeparableAffineModel([[(abi.TERM_COORD, 1, 1.0)]] * 4, B, C, [])
    with pytest.raises(ValueError):
        hj.SeparableAffineModel([[(abi.TERM_COORD, 1, 1.0)] * 3] + [[]] * 3)
