"""GPU: batched SafetyFilter queries (hjb_filter_batch[_dev] kernels) and the
decomposition over device-resident value functions against the C
restatement and the reference's own SafetyFilter / Decomposition.  Bitwise."""
import ctypes as C

import numpy as np
import pytest

from paper_2101_05916_b200 import abi
from paper_2101_05916_b200 import hjsafe as hj
from paper_2101_05916_b200 import safety

from filter_cases import converged, decomposition_10d, planar_case, queries, vertical_case

pytestmark = pytest.mark.gpu


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def check(got: safety.FilterBatch, want: dict):
    assert same(got.value, want["value"])
    assert same(got.band, want["band"])
    assert same(got.control, want["control"])
    assert same(got.worst_disturbance, want["worst_disturbance"])
    assert same(got.flags, want["flags"])


@pytest.mark.parametrize("case", ["vertical", "planar", "planar_per_node"])
def test_filter_batch_matches_restatement(gpu_ctx, oracle, case):
    if case == "vertical":
        g, model, db, V = vertical_case(oracle)
        U = np.random.default_rng(2).uniform(-1, 3, size=(3000, 1))
    else:
        g, model, db, V = planar_case(n=11, per_node=case.endswith("per_node"))
        U = np.random.default_rng(2).uniform(-1, 1, size=(3000, 1))
    X = queries(g, 3000, 7)
    f = hj.SafetyFilter(model, converged(V), db, hj.SafetyFilter.Config(eta_floor=2e-3), ctx=gpu_ctx)
    check(f.optimal_control_batch(X),
          oracle.filter_batch(V, model, db, X, U, mode=abi.FILTER_OPTIMAL, eta_floor=2e-3))
    check(f.filter_batch(X, U),
          oracle.filter_batch(V, model, db, X, U, mode=abi.FILTER_FILTER, eta_floor=2e-3))


def test_single_queries_and_contract_match_reference(gpu_ctx, oracle, ref):
    g, model, db, V = vertical_case(oracle)
    X = queries(g, 200, 3)
    U = np.random.default_rng(4).uniform(-1, 3, size=(len(X), 1))
    f = hj.SafetyFilter(model, converged(V), db, ctx=gpu_ctx)
    assert f.lambda_() == 0.0 and f.emergency() is False
    lam = f.contract([hj.Violation(list(x)) for x in X[:40]])
    want, rlam, rem = ref.filter_batch(V, model, db, X, U, mode=abi.FILTER_FILTER,
                                       violations=X[:40])
    assert lam == rlam == f.lambda_() and f.emergency() == rem
    assert f.contract([]) == lam
    for q in range(0, len(X), 37):
        d = f.filter(list(X[q]), list(U[q]))
        assert d.value == want["value"][q] and d.band == want["band"][q]
        assert d.control == list(want["control"][q])
        assert d.override_active == bool(want["flags"][q] & abi.FILTER_OVERRIDE)
        assert d.out_of_domain == bool(want["flags"][q] & abi.FILTER_OOD)
        assert f.value_at(list(X[q])) == want["value"][q]
    b = f.dbound_at(0, list(X[5]))
    lo = oracle.interp(hj.ScalarField(g, np.full(g.size(), db.at_node(0, 0).lo)), X[5])
    assert b.lo == lo[0]


def test_interp_batch_matches_oracle(gpu_ctx, oracle):
    g, model, db, V = planar_case(n=13)
    X = queries(g, 1000, 11, spread=0.2)
    f = hj.SafetyFilter(model, converged(V), db, ctx=gpu_ctx)
    v = f.value_at_batch(X)
    for q in range(0, len(X), 50):
        want, _ = oracle.interp(V, X[q])
        assert v[q] == want


def test_host_pointer_abi_matches_restatement(gpu_ctx, oracle):
    g, model, db, V = planar_case(n=9, per_node=True)
    X = queries(g, 500, 13)
    U = np.random.default_rng(1).uniform(-1, 1, size=(len(X), 1))
    want = oracle.filter_batch(V, model, db, X, U, mode=abi.FILTER_FILTER, lam=0.1)
    nq = len(X)
    got = dict(value=np.empty(nq), band=np.empty(nq), control=np.empty((nq, 1)),
               worst_disturbance=np.empty((nq, 1)), flags=np.empty(nq, dtype=np.uint8))
    out = abi.HjbFilterOut(*(got[k].ctypes.data for k in
                             ("value", "band", "control", "worst_disturbance", "flags")))
    cfg = abi.HjbFilterConfig(abi.FILTER_FILTER, 0, 1e-5, 0.1)
    gg, mm, dd = g.to_c(), model.to_c(), db.to_c()
    vv = np.ascontiguousarray(V.values())
    hj._check(abi.load().hjb_filter_batch(gpu_ctx.handle, C.byref(gg), C.byref(mm), C.byref(dd),
                                          vv.ctypes.data, nq, X.ctypes.data, U.ctypes.data,
                                          C.byref(cfg), C.byref(out)))
    for k in want:
        assert same(got[k], want[k]), k


def test_decomposition_matches_reference(gpu_ctx, ref):
    subs, values, dbs, dims, X, U = decomposition_10d()
    dec = hj.Decomposition(subs, *dims)
    dec.attach([hj.SafetyFilter(s.model, converged(v), d, ctx=gpu_ctx)
                for s, v, d in zip(subs, values, dbs)])
    for viol in ((), X[:7]):
        want, lam, em = ref.decomposition_batch(subs, values, dbs, dims, X, U, violations=viol)
        if len(viol):
            assert dec.contract([hj.Violation(list(x)) for x in viol]) == lam
        got = dec.combined_control_batch(X, U)
        assert same(dec.combined_value_batch(X), want["combined_value"])
        assert same(got.value, want["value"]) and same(got.band, want["band"])
        assert same(got.control, want["control"])
        d = dec.combined_control(list(X[3]), list(U[3]))
        assert d.value == want["value"][3] and d.control == list(want["control"][3])
    dec.adopt([converged(v) for v in values], dbs)
    assert dec.lambda_() == 0.0


def test_filter_errors(gpu_ctx, oracle):
    g, model, db, V = planar_case()
    with pytest.raises(hj.InvalidArgument, match="not converged"):
        hj.SafetyFilter(model, hj.SolveResult(value=V, converged=False), db, ctx=gpu_ctx)
    with pytest.raises(hj.InvalidArgument, match="grid rank"):
        hj.SafetyFilter(hj.NearHoverVertical2D(), converged(V), db, ctx=gpu_ctx)
    f = hj.SafetyFilter(model, converged(V), db, ctx=gpu_ctx)
    X = queries(g, 8, 1)
    X[3, 2] = np.inf
    with pytest.raises(hj.InvalidArgument, match="non-finite"):
        f.optimal_control_batch(X)
    with pytest.raises(hj.InvalidArgument, match="control dim"):
        f.filter(list(X[0]), [0.0, 1.0])
    with pytest.raises(hj.InvalidArgument, match="rank mismatch"):
        f.value_at([0.0, 1.0])


def test_device_resident_warm_update(gpu_ctx, oracle):
    """The online update loop (sim.cpp:339-363) with V* never leaving HBM:
    warm solves from every filter's device V* under new bounds, adopted
    straight from the device, answer exactly like the host path (warm solve
    of the host V*, adopt of the host result) and like the restatement."""
    from paper_2101_05916_b200 import configs
    subs, _, _, dims, X, U = decomposition_10d(n4=9, n2=21)
    cfg = hj.SolveConfig(tolerance=5e-3, max_iters=40000)
    from cases import band_np
    ws = []
    for s in subs:
        g = {4: configs.planar_grid(9), 2: configs.vertical_grid(21)}[s.model.state_dim()]
        c = band_np(g, 0, 0.0, 3.0) if s.model.state_dim() == 2 else band_np(g, 0, -4.0, 4.0)
        ws.append((g, hj.ScalarField(g, c)))
    b0 = [hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)]) for g, _ in ws]
    b1 = [hj.IntervalField.constant(g, [hj.Interval(-0.8, 0.8)]) for g, _ in ws]
    cold = [hj.solve(c, c, s.model, b, cfg, ctx=gpu_ctx) for s, (g, c), b in zip(subs, ws, b0)]
    assert all(r.converged for r in cold)
    dec = hj.Decomposition(subs, *dims)
    dec.attach([hj.SafetyFilter(s.model, r, b, ctx=gpu_ctx) for s, r, b in zip(subs, cold, b0)])
    cdev = []
    for g, c in ws:
        buf = safety.DeviceBuffer(gpu_ctx, g.size() * 8)
        buf.upload(c.values())
        cdev.append(buf)
    upd = dec.warm_update(cdev, b1, cfg)
    host = [hj.solve(r.value, c, s.model, b, cfg, ctx=gpu_ctx)
            for s, r, (g, c), b in zip(subs, cold, ws, b1)]
    want = [oracle.solve(r.value, c, s.model, b, cfg) for s, r, (g, c), b in zip(subs, cold, ws, b1)]
    for u, h, w in zip(upd, host, want):
        assert u.iterations == h.iterations == w.iterations and u.converged
        assert same(u.to_host().value.values(), h.value.values())
        assert same(h.value.values(), w.value.values())
    dec.adopt(upd, b1)
    ref_dec = hj.Decomposition(subs, *dims)
    ref_dec.attach([hj.SafetyFilter(s.model, h, b, ctx=gpu_ctx) for s, h, b in zip(subs, host, b1)])
    a, b = dec.combined_control_batch(X, U), ref_dec.combined_control_batch(X, U)
    assert same(a.value, b.value) and same(a.control, b.control) and same(a.band, b.band)
    for i in range(dec.count()):
        assert dec.filter(i).min_value() == float(np.min(host[i].value.values()))
        assert same(dec.filter(i).value_snapshot().values(), host[i].value.values())
