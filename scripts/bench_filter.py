"""Throughput of batched SafetyFilter queries on the GPU, with
the reference's own SafetyFilter timed on the host beside it.

usage: python scripts/bench_filter.py [--n 51] [--queries 1000000] [--sweeps 20000]

V* is the config-2 (4D planar, 51^4) value after `--sweeps` device sweeps
from V = c; the per-query cost does not depend on convergence, so the state
is marked converged for the filter.  Queries are uniform over the grid box
widened by 5 % (some out of domain), performance control uniform in the
control bounds.  Prints one JSON line.
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2101_05916_b200 import abi, configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=51)
    ap.add_argument("--queries", type=int, default=1_000_000)
    ap.add_argument("--sweeps", type=int, default=20000)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cpu-queries", type=int, default=20000)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = configs.config2(a.n)
    g, model, db = w.grid, w.model, w.dbounds()
    ctx = hj.Context(0)
    cells = g.size()
    c_t = torch.empty(cells, dtype=torch.float64, device=dev)
    v_t = torch.empty_like(c_t)
    torch.cuda.synchronize()
    hj.signed_distance_band_dev(g, 0, -4.0, 4.0, c_t.data_ptr(), ctx=ctx)
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.max_iters = a.sweeps
    hj.solve_dev(g, model, db, c_t.data_ptr(), c_t.data_ptr(), v_t.data_ptr(), cfg, ctx=ctx)
    V = hj.ScalarField(g, v_t.cpu().numpy(), check=False)

    rng = np.random.default_rng(5916)
    lo = np.array([d.min for d in g.dims()])
    hi = np.array([d.max for d in g.dims()])
    nq = a.queries
    X = lo + (hi - lo) * rng.uniform(-0.05, 1.05, size=(nq, 4))
    ub = model.control_bounds()[0]
    U = rng.uniform(ub.lo, ub.hi, size=(nq, 1))

    # device-resident timing of the raw batch (inputs already in HBM)
    x_t = torch.from_numpy(X).to(dev)
    u_t = torch.from_numpy(U).to(dev)
    o = dict(value=torch.empty(nq, dtype=torch.float64, device=dev),
             band=torch.empty(nq, dtype=torch.float64, device=dev),
             control=torch.empty(nq, 1, dtype=torch.float64, device=dev),
             worst=torch.empty(nq, 1, dtype=torch.float64, device=dev),
             flags=torch.empty(nq, dtype=torch.uint8, device=dev))
    out = abi.HjbFilterOut(o["value"].data_ptr(), o["band"].data_ptr(), o["control"].data_ptr(),
                           o["worst"].data_ptr(), o["flags"].data_ptr())
    fc = abi.HjbFilterConfig(abi.FILTER_FILTER, 0, 1e-5, 0.0)
    gg, mm, dd = g.to_c(), model.to_c(), db.to_c()
    lib = abi.load()
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    def run():
        hj._check(lib.hjb_filter_batch_dev(ctx.handle, C.byref(gg), C.byref(mm), C.byref(dd),
                                           v_t.data_ptr(), nq, x_t.data_ptr(), u_t.data_ptr(),
                                           C.byref(fc), C.byref(out)))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.reps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    dev_s = e0.elapsed_time(e1) * 1e-3 / a.reps

    # e2e through the reference-facing API: host states in, decisions out
    f = hj.SafetyFilter(model, hj.SolveResult(value=V, converged=True), db, ctx=ctx)
    f.filter_batch(X[:1000], U[:1000])
    t0 = time.perf_counter()
    fb = f.filter_batch(X, U)
    e2e_s = time.perf_counter() - t0
    passed = int((~fb.override_active).sum())

    # the reference's SafetyFilter::filter, one query at a time on the host
    cpu = None
    try:
        sys.path.insert(0, str(ROOT))
        from oracle.oracle import Reference
        ref = Reference()
        k = a.cpu_queries
        t0 = time.perf_counter()
        want, _, _ = ref.filter_batch(V, model, db, X[:k], U[:k], mode=abi.FILTER_FILTER)
        cpu_s = time.perf_counter() - t0
        cpu = {"value": k / cpu_s, "unit": "queries/s", "cores": 1, "kind": "reference",
               "sample": f"{k} SafetyFilter::filter calls (reference, one thread; includes one "
                         "filter construction over the 51^4 field)"}
        agree = all(np.array_equal(getattr(fb, key)[:k], want[key2]) for key, key2 in
                    (("value", "value"), ("band", "band"), ("control", "control"),
                     ("flags", "flags")))
        cpu["bitwise_agree_on_sample"] = bool(agree)
    except Exception as e:  # reference library absent on the box
        cpu = {"value": None, "error": str(e)}

    # algorithmic bytes per interior 4D query: 16 corners + 2 outer
    # neighbours per axis per corner face (16 + 4*2*8 = 80 nodes of V) +
    # x (32) + u (8) + outputs (8+8+8+8+1)
    bytes_q = 80 * 8 + 32 + 8 + 33
    line = {"metric": "SafetyFilter::filter queries/s (batched, 4D, V* resident)",
            "value": nq / dev_s, "unit": "queries/s", "queries": nq, "grid": f"{a.n}^4",
            "device_seconds_per_batch": dev_s, "bytes_per_query": bytes_q,
            "achieved_gbs": bytes_q * nq / dev_s / 1e9,
            "e2e": {"value": nq / e2e_s, "unit": "queries/s",
                    "path": "SafetyFilter.filter_batch: numpy states -> H2D -> kernel -> D2H",
                    "seconds": e2e_s},
            "passed_through": passed, "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
