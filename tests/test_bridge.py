"""The header-only C++ drop-in (include/hjb_bridge.hpp) against the reference
in one process (tests/cpp/bridge_demo.cpp, built where /root/reference exists).
"""
import subprocess
from pathlib import Path

import pytest

EXE = Path(__file__).resolve().parent / "cpp" / "_build" / "bridge_demo"


def _run():
    if not EXE.exists():
        pytest.skip("bridge_demo not built (needs /root/reference at build time)")
    return subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)


def test_bridge_without_gpu_fails_loudly():
    import ctypes
    from paper_2101_05916_b200 import abi
    n = ctypes.c_int(0)
    abi.load().hjb_device_count(ctypes.byref(n))
    if n.value > 0:
        pytest.skip("GPU present")
    p = _run()
    assert p.returncode == 3, p.stdout + p.stderr


@pytest.mark.gpu
def test_bridge_matches_reference_on_gpu():
    p = _run()
    assert p.returncode == 0, p.stdout + p.stderr
    assert "FAIL" not in p.stdout
