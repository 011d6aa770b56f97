"""GP bounds on the solver grid: device bounds_on_grid against
the reference's per-node evaluation (the oracle restatement, which computes
exactly the reference's GpModel::predict per node) on a bounded sample.

usage: python scripts/bench_gp.py [--n 51] [--train 500] [--reps 5]

Model: a 1D GP over axis 0 (sim.cpp:605,647: "wind depends on altitude"),
fitted by the reference's hyperparameter search on `--train` synthetic
samples; grid: the config-2 box at n^4.  Prints one JSON line.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=51)
    ap.add_argument("--train", type=int, default=500)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu-nodes", type=int, default=4000)
    a = ap.parse_args()
    g = configs.planar_grid(a.n)
    rng = np.random.default_rng(5916)
    X = rng.uniform(-5.0, 5.0, size=(a.train, 1))
    y = 0.3 * np.sin(X[:, 0]) + rng.normal(0.0, 0.05, size=a.train)
    t0 = time.perf_counter()
    m = hj.GpModel.fit([hj.DisturbanceMeasurement(list(x), v) for x, v in zip(X, y)])
    fit_s = time.perf_counter() - t0
    ctx = hj.Context(0)
    cells = g.size()
    lo = torch.empty(cells, dtype=torch.float64, device="cuda")
    hi = torch.empty_like(lo)
    torch.cuda.synchronize()

    def run():
        hj.bounds_on_grid_dev([m], [[0]], g, [lo.data_ptr()], [hi.data_ptr()], 3.0, ctx=ctx)

    for _ in range(3):
        run()
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.reps):
        run()
    ctx.synchronize()
    dev_s = (time.perf_counter() - t0) / a.reps

    # host-buffer entry point (bounds come back to host memory)
    t0 = time.perf_counter()
    b = hj.bounds_on_grid([m], [[0]], g, 3.0, ctx=ctx)
    e2e_s = time.perf_counter() - t0

    cpu = None
    try:
        from oracle.oracle import Restatement
        orc = Restatement(threads=1)
        k = a.cpu_nodes
        sub = hj.Grid([(g.dim(0).min, g.dim(0).max, g.dim(0).n), (0.0, 1.0, k // g.dim(0).n)])
        t0 = time.perf_counter()
        wl, wh = orc.gp_bounds_on_grid([m], [[0]], sub)
        cpu_s = time.perf_counter() - t0
        nodes = sub.size()
        cpu = {"value": nodes / cpu_s, "unit": "nodes/s", "cores": 1, "kind": "port",
               "sample": f"{nodes} nodes of per-node GpModel::predict (reference order, "
                         f"n_train={m.training_count()}), 1 thread",
               "extrapolated_full_grid_s": cells / (nodes / cpu_s)}
        lo_h = lo.cpu().numpy().reshape(g.dim(0).n, -1)[:, 0]
        cpu["bitwise_agree_on_sample"] = bool(np.array_equal(
            np.asarray(wl[0]).reshape(g.dim(0).n, -1)[:, 0], lo_h))
    except Exception as e:  # oracle absent
        cpu = {"value": None, "error": str(e)}
    line = {"metric": "bounds_on_grid nodes/s (1 channel, GP over axis 0)",
            "value": cells / dev_s, "unit": "nodes/s", "grid": f"{a.n}^4",
            "n_train": m.training_count(), "device_seconds": dev_s,
            "write_gbs": 16 * cells / dev_s / 1e9,
            "e2e": {"value": cells / e2e_s, "unit": "nodes/s", "seconds": e2e_s,
                    "path": "hj.bounds_on_grid -> host IntervalField"},
            "fit_seconds_host": fit_s, "cpu_baseline": cpu,
            "hyperparams": m.hyperparams().__dict__, "check_lo0": float(b.lo(0)[0])}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
