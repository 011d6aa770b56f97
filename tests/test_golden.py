"""Pin the CPU restatement to golden fixtures produced by the REFERENCE
(tests/golden/make_golden.py, run against oracle/_ref).  Runs everywhere,
including where /root/reference is absent."""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2101_05916_b200 import configs, hjvf
from paper_2101_05916_b200 import hjsafe as hj

from cases import hash_field, quad_setup, same, solve_cases, with_iters, workload_case

G = Path(__file__).resolve().parent / "golden"
META = json.loads((G / "golden_v1.json").read_text())
ARR = np.load(G / "golden_v1.npz")


@pytest.mark.parametrize("case,iters", solve_cases(), ids=lambda x: getattr(x, "name", str(x)))
def test_oracle_matches_reference_golden(oracle, case, iters):
    c = with_iters(case, iters)
    r = oracle.solve(c.init_field(), c.c_field(), c.model, c.db, c.cfg)
    m = META[c.name]
    assert r.iterations == m["iterations"] and r.converged == m["converged"] and r.dt == m["dt"]
    assert hash_field(r.value.values()) == m["value_sha256"]
    assert hash_field(r.residual_history) == m["history_sha256"]
    if c.name + "/value" in ARR:
        assert same(r.value.values(), ARR[c.name + "/value"])


def test_cfg2_21_golden(oracle):
    c = with_iters(workload_case(configs.config2(21)), 200)
    r = oracle.solve(c.init_field(), c.c_field(), c.model, c.db, c.cfg)
    m = META["cfg2_21_k200"]
    assert r.iterations == 200 and r.dt == m["dt"]
    assert hash_field(r.value.values()) == m["value_sha256"]
    assert same(r.residual_history, ARR["cfg2_21_k200/history"])


def test_resample_and_ctf_golden(oracle):
    src_g, dst_g = configs.planar_grid(7), configs.planar_grid(13)
    f = hj.ScalarField(src_g, ARR["resample/src"])
    assert hash_field(oracle.resample(f, dst_g)) == META["resample_7_13"]["value_sha256"]
    assert oracle.max_adjacent_jump(f) == META["resample_7_13"]["max_adjacent_jump"]
    q = quad_setup(41)
    coarse = hj.Grid([(0.0, 3.2, 21), (-5.0, 5.0, 21)])
    r = oracle.solve_coarse_to_fine(q.c_field(), q.model, q.db, coarse, q.cfg)
    m = META["ctf_quad41_21"]
    assert (r.coarse.iterations, r.fine.iterations) == (m["coarse_iterations"], m["fine_iterations"])
    assert hash_field(r.coarse.value.values()) == m["coarse_sha256"]
    assert hash_field(r.fine.value.values()) == m["fine_sha256"]


def test_cfl_golden(oracle):
    for name, speeds, dims in (("cfl_1d", [10.1], [(0.0, 1.0, 21)]),
                               ("cfl_2d", [2.0, 10.1], [(0.0, 1.0, 21), (0.0, 1.4, 21)])):
        g = hj.Grid(dims)
        assert oracle.cfl_dt(g, hj.ConstantAdvection(speeds), hj.IntervalField.constant(g, []), 0.8) \
            == META[name]["dt"]


def test_hjvf_reads_reference_file_and_round_trips(oracle):
    """The reference's own HJVF writer output (hjvf.cpp:46-68) parses with
    the product reader, equals the config-1 fixed point, and re-serialises
    to identical bytes (test_grid.cpp:212-232)."""
    raw = (G / "cfg1_value.hjvf").read_bytes()
    f = hjvf.loads(raw)
    assert f.grid() == configs.vertical_grid(101)
    assert same(f.values(), ARR["cfg1_vertical2d_101/value"])
    assert hjvf.dumps(f) == raw
    with pytest.raises(RuntimeError):
        hjvf.loads(b"not a field")
    with pytest.raises(RuntimeError):
        hjvf.loads(raw[:-8])
