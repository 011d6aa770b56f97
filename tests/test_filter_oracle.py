"""CPU: the C restatement of the SafetyFilter queries (oracle/hj_oracle.c,
hjo_filter_batch) against the reference's own SafetyFilter, and the
decomposition's host-side recombination (safety.py) over restatement-backed
filters against the reference's own Decomposition.  Bitwise (IEEE ==)."""
import numpy as np
import pytest

from paper_2101_05916_b200 import abi
from paper_2101_05916_b200 import hjsafe as hj
from paper_2101_05916_b200 import safety

from filter_cases import converged, decomposition_10d, planar_case, queries, vertical_case


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def check(a, b):
    for k in ("value", "band", "control", "worst_disturbance", "flags"):
        assert same(a[k], b[k]), k


@pytest.mark.parametrize("mode", [abi.FILTER_OPTIMAL, abi.FILTER_FILTER])
def test_vertical_2d(oracle, ref, mode):
    g, model, db, V = vertical_case(oracle)
    X = queries(g, 1500, 1)
    U = np.random.default_rng(2).uniform(-1, 3, size=(len(X), 1))
    a = oracle.filter_batch(V, model, db, X, U, mode=mode)
    b, lam, em = ref.filter_batch(V, model, db, X, U, mode=mode)
    check(a, b)
    assert lam == 0.0 and not em
    flags = a["flags"]
    assert (flags & abi.FILTER_OOD).any() and (flags & abi.FILTER_DEGENERATE).any()
    if mode == abi.FILTER_FILTER:
        assert ((flags & abi.FILTER_OVERRIDE) == 0).any()


@pytest.mark.parametrize("per_node", [False, True])
@pytest.mark.parametrize("mode", [abi.FILTER_OPTIMAL, abi.FILTER_FILTER])
def test_planar_4d(oracle, ref, mode, per_node):
    g, model, db, V = planar_case(per_node=per_node)
    X = queries(g, 2000, 5)
    U = np.random.default_rng(6).uniform(-1, 1, size=(len(X), 1))
    a = oracle.filter_batch(V, model, db, X, U, mode=mode, eta_floor=1e-3)
    b, _, _ = ref.filter_batch(V, model, db, X, U, mode=mode, eta_floor=1e-3)
    check(a, b)


def test_contract_then_filter(oracle, ref):
    g, model, db, V = vertical_case(oracle)
    X = queries(g, 800, 8)
    U = np.zeros((len(X), 1))
    for viol in (X[:10], X[100:101], X[:300]):
        b, lam, em = ref.filter_batch(V, model, db, X, U, mode=abi.FILTER_FILTER,
                                      violations=viol)
        a = oracle.filter_batch(V, model, db, X, U, mode=abi.FILTER_FILTER, lam=lam)
        check(a, b)


def test_non_finite_query_rejected(oracle, ref):
    g, model, db, V = planar_case()
    X = queries(g, 4, 1)
    X[2, 1] = np.nan
    with pytest.raises(Exception, match="non-finite"):
        oracle.filter_batch(V, model, db, X)
    with pytest.raises(Exception, match="non-finite"):
        ref.filter_batch(V, model, db, X)


class _OracleFilter:
    """Test adapter: the SafetyFilter query surface safety.Decomposition uses,
    answered by the C restatement (CPU) instead of the device kernels."""

    def __init__(self, oracle, model, value, db, eta_floor=1e-5):
        self.o, self.m, self.v, self.db, self.eta = oracle, model, value, db, eta_floor

    def _batch(self, X, U, mode):
        a = self.o.filter_batch(self.v, self.m, self.db, X, U, mode=mode, eta_floor=self.eta)
        return safety.FilterBatch(**a)

    def optimal_control_batch(self, X):
        return self._batch(X, None, abi.FILTER_OPTIMAL)

    def filter_batch(self, X, U):
        return self._batch(X, U, abi.FILTER_FILTER)

    def min_value(self):
        return float(np.min(self.v.values()))


def test_decomposition_recombination(oracle, ref):
    subs, values, dbs, dims, X, U = decomposition_10d()
    dec = hj.Decomposition(subs, *dims)
    dec.attach([_OracleFilter(oracle, s.model, v, d) for s, v, d in zip(subs, values, dbs)])
    passed = []
    for viol in ((), X[:5], X[:60]):
        want, lam, em = ref.decomposition_batch(subs, values, dbs, dims, X, U, violations=viol)
        if len(viol):
            assert dec.contract([hj.Violation(list(x)) for x in viol]) == lam
            assert dec.emergency() == em
        cv = dec.combined_value_batch(X)
        got = dec.combined_control_batch(X, U)
        assert same(cv, want["combined_value"])
        assert same(got.value, want["value"]) and same(got.band, want["band"])
        assert same(got.control, want["control"])
        flags = (got.override_active * abi.FILTER_OVERRIDE) | (got.out_of_domain * abi.FILTER_OOD)
        assert same(flags.astype(np.uint8), want["flags"])
        passed.append(int((~got.override_active).sum()))
    assert np.isinf(cv).any() and passed[0] > 0 and passed[-1] < passed[0]


def test_decomposition_validation():
    subs, values, dbs, dims, X, U = decomposition_10d()
    with pytest.raises(hj.InvalidArgument, match="no subsystems"):
        hj.Decomposition([], *dims)
    bad = [hj.Subsystem(s.name, s.model, list(s.state_map), list(s.control_map),
                        list(s.disturbance_map)) for s in subs]
    bad[1].state_map = [0, 5, 6, 7]
    with pytest.raises(hj.InvalidArgument, match="state_map: index maps overlap"):
        hj.Decomposition(bad, *dims)
    with pytest.raises(hj.InvalidArgument, match="do not cover"):
        hj.Decomposition(subs[:2], *dims)
    dec = hj.Decomposition(subs, *dims)
    with pytest.raises(RuntimeError, match="filters not attached"):
        dec.combined_value(list(X[0]))
    with pytest.raises(hj.InvalidArgument, match="one filter per subsystem"):
        dec.attach([None])
