"""Test harness: markers, paths and shared fixtures.

`-m "not gpu"` runs here (no GPU): oracle vs reference, oracle vs golden
fixtures, host logic, ABI exports.  `-m gpu` runs on a B200: the CUDA path
through the C ABI against the oracle.
"""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Restatement, build, RESTATEMENT_SO
    if not RESTATEMENT_SO.exists():
        build(ref=False)
    return Restatement()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libhjref.so not built (needs /root/reference)")
    return Reference()


@pytest.fixture(scope="session")
def ref_gp():
    from oracle.oracle import ReferenceGp, REF_GP_SO
    if not REF_GP_SO.exists():
        pytest.skip("oracle/_ref/libhjref_gp.so not built (needs /root/reference)")
    return ReferenceGp()


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2101_05916_b200 import hjsafe as hj
    return hj.Context(0)
