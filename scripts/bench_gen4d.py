"""Per-sweep device time of user models on the run-time-shape 4D kernel
(k_fast4d<ShapeGen>) against the generic kernel (HJB_FAST=0), next to the
compiled-shape kernel on the config-2 model, at one grid size.

usage: python scripts/bench_gen4d.py [n=51] [iters=300] [gd|lf] [const|axis0|node] [order=1] [rk=1]
(order / rk > 1: ENO + TVD-RK, one step = all RK stages)
Prints one JSON line per (model, kernel).
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402
from test_gpu_gen4d import MODELS, _per_node_db  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 51
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    ctx = hj.Context(0)
    g = hj.Grid([(-5.0, 5.0, n), (-2.0, 2.0, n), (-0.35, 0.35, n), (-1.5, 1.5, n)])
    c = hj.signed_distance_band(g, 0, -4.0, 4.0, ctx=ctx)
    scheme = sys.argv[3] if len(sys.argv) > 3 else "gd"
    cfg = hj.SolveConfig(tolerance=1e-12, max_iters=iters)
    if scheme == "lf":
        cfg.scheme = hj.LAX_FRIEDRICHS
    cfg.spatial_order = int(sys.argv[5]) if len(sys.argv) > 5 else 1
    cfg.time_order = int(sys.argv[6]) if len(sys.argv) > 6 else 1
    os.environ["HJB_MS"] = "0"
    bounds = sys.argv[4] if len(sys.argv) > 4 else "const"

    def db_of(nd):
        if bounds == "const" or nd == 0:
            return hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)] * nd)
        return _per_node_db(g, nd, bounds)
    runs = [(name, make(), db_of(nd)) for name, (make, nd) in sorted(MODELS.items())
            if bounds == "const" or nd > 0]
    w = configs.config2(n)
    runs.append(("config2 (compiled shape)", w.model, w.dbounds() if bounds == "const" else db_of(1)))
    for name, model, db in runs:
        for fast in ("1", "0"):
            os.environ["HJB_FAST"] = fast
            warm = hj.SolveConfig(max_iters=5)
            warm.scheme, warm.spatial_order, warm.time_order = (cfg.scheme, cfg.spatial_order,
                                                                cfg.time_order)
            hj.solve(c, c, model, db, warm, ctx=ctx)  # autotune, warm
            r = hj.solve(c, c, model, db, cfg, ctx=ctx)
            us = r.wall_seconds / r.iterations * 1e6
            print(json.dumps({"model": name, "grid": f"{n}^4", "scheme": scheme, "bounds": bounds,
                              "order": cfg.spatial_order, "rk": cfg.time_order,
                              "kernel": r.kernel,
                              "step_us": round(us, 2), "iterations": r.iterations,
                              "gcell_per_s": round(g.size() / us * 1e-3, 2)}), flush=True)
    os.environ.pop("HJB_FAST", None)


if __name__ == "__main__":
    main()
