"""Constraint set-up: signed_distance_band, field_max /
field_min (reference proj/src/levelset.cpp:54-66, 80-86) and the config-5
avoid set c = max(band(x,-4,4), -band(x, obstacle_i)) built on the device,
pinned bitwise to the reference's own functions (oracle/_ref)."""
import numpy as np
import pytest
import torch

from paper_2101_05916_b200 import configs
from paper_2101_05916_b200 import hjsafe as hj

from cases import band_np, fmax_np, same


def _fields(g, seed=4):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(g.size())
    b = rng.standard_normal(g.size())
    # ties and signed zeros: std::max / std::min keep the FIRST argument on a tie
    b[::7] = a[::7]
    a[::11], b[::11] = 0.0, -0.0
    a[::13], b[::13] = -0.0, 0.0
    return a, b


def _bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def test_reference_field_ops_are_std_max_min(ref):
    """The reference's field_max / field_min are std::max / std::min per
    node: on ties (including +0 vs -0) the first argument is kept."""
    g = configs.planar_grid(7)
    a, b = _fields(g)
    fa, fb = hj.ScalarField(g, a), hj.ScalarField(g, b)
    mx, mn = ref.field_max(fa, fb), ref.field_min(fa, fb)
    assert np.array_equal(_bits(mx), _bits(np.where(a < b, b, a)))
    assert np.array_equal(_bits(mn), _bits(np.where(b < a, b, a)))


def test_config5_constraint_composition_matches_reference(ref):
    """configs.config5's avoid set composed from the reference's own
    signed_distance_band and field_max (obstacles: the negated band) equals
    the numpy composition the CPU tests use."""
    w = configs.config5(levels=(13,))[0]
    g = w.grid
    c = None
    for dim, lo, hi, sign in w.bands:
        f = ref.signed_distance_band(g, dim, lo, hi)
        f = -f if sign < 0 else f
        c = f if c is None else ref.field_max(hj.ScalarField(g, c), hj.ScalarField(g, f))
    assert np.array_equal(_bits(c), _bits(w.constraint(band_np, fmax_np)))


@pytest.mark.gpu
def test_gpu_field_ops_bitwise_vs_reference(gpu_ctx, ref):
    g = configs.planar_grid(9)
    a, b = _fields(g, 8)
    fa, fb = hj.ScalarField(g, a), hj.ScalarField(g, b)
    at, bt = torch.tensor(a, device="cuda"), torch.tensor(b, device="cuda")
    out = torch.empty_like(at)
    torch.cuda.synchronize()
    hj.field_max_dev(g.size(), at.data_ptr(), bt.data_ptr(), out.data_ptr(), ctx=gpu_ctx)
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(ref.field_max(fa, fb)))
    hj.field_min_dev(g.size(), at.data_ptr(), bt.data_ptr(), out.data_ptr(), ctx=gpu_ctx)
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(ref.field_min(fa, fb)))
    hj.field_negate_dev(g.size(), at.data_ptr(), out.data_ptr(), ctx=gpu_ctx)
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(-a))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [26, 51])
def test_gpu_config5_constraint_on_device(gpu_ctx, ref, n):
    """configs.Workload.constraint_dev (band + negate + field_max kernels)
    equals the reference's composition bit for bit."""
    w = configs.config5(levels=(n,))[0]
    g = w.grid
    out = torch.empty(g.size(), dtype=torch.float64, device="cuda")
    scratch = torch.empty_like(out)
    torch.cuda.synchronize()
    w.constraint_dev(out.data_ptr(), scratch.data_ptr(), ctx=gpu_ctx)
    want = None
    for dim, lo, hi, sign in w.bands:
        f = ref.signed_distance_band(g, dim, lo, hi)
        f = -f if sign < 0 else f
        want = f if want is None else ref.field_max(hj.ScalarField(g, want), hj.ScalarField(g, f))
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(want))
