"""Run the BASELINE.json workloads end to end on the GPU and report.

usage: python scripts/run_configs.py [cfg ...] [--max-iters N] [--json out.json]
  cfg in {1, 2, 3, 4, 5}; default: 1 2

Config 1: 2D vertical subsystem 101^2 to convergence (tol 1e-4).
Config 2: 4D planar 51^4 to convergence (tol 1e-4) or --max-iters.
Config 3: 4D planar 101^4 (first-order reference scheme) to convergence or cap.
Config 4: decomposed 10D: 2D 101^2 + x/y 4D 71^4, cold at wind 0.5, warm 0.8,
          then 10 warm updates with seeded bounds; the three subsystem solves
          of every update run concurrently (one context + host thread each).
Config 5: adaptive 26^4 -> 51^4 -> 101^4 (wind 0.6, 3 seeded obstacles).
All timings are device times reported by the library.
"""
import argparse
import json
import sys
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402


def constraint(w, ctx):
    """c on the device kernels (signed_distance_band + max), then to host."""
    out = None
    for dim, lo, hi, sign in w.bands:
        f = hj.signed_distance_band(w.grid, dim, lo, hi, ctx=ctx).values()
        f = -f if sign < 0 else f
        out = f if out is None else np.where(out < f, f, out)
    return hj.ScalarField(w.grid, out)


def summarize(r, cells):
    return {"iterations": r.iterations, "converged": r.converged, "dt": r.dt,
            "device_seconds": r.wall_seconds, "final_residual": r.final_residual,
            "cell_updates_per_s": cells * r.iterations / max(r.wall_seconds, 1e-12),
            "safe_cells": int(np.sum(r.value.values() <= 0)) if r.value is not None else None}


def run_single(w, max_iters, ctx):
    c = constraint(w, ctx)
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.max_iters = max_iters
    r = hj.solve(c, c, w.model, w.dbounds(), cfg, ctx=ctx, history_capacity=max_iters)
    out = summarize(r, w.grid.size())
    h = r.residual_history
    marks = [k for k in (1, 10, 100, 1000, 10000, 100000, 1000000) if k <= len(h)]
    out["residual_at"] = {str(k): float(h[k - 1]) for k in marks}
    return out


def run_config4(max_iters, ctx0, tol):
    subs = configs.config4_subsystems(tol=tol)
    bounds = configs.bound_sequence()
    ctxs = [ctx0] + [hj.Context(0) for _ in subs[1:]]
    cs = [constraint(w, ctxs[i]) for i, w in enumerate(subs)]
    values = [c for c in cs]
    report = []
    for u, wind in enumerate(bounds):
        results = [None] * len(subs)

        def job(i):
            w = subs[i]
            cfg = hj.SolveConfig(**w.cfg.__dict__)
            cfg.max_iters = max_iters
            results[i] = hj.solve(values[i], cs[i], w.model, w.dbounds(wind), cfg, ctx=ctxs[i],
                                  history_capacity=0)

        t0 = time.perf_counter()
        th = [threading.Thread(target=job, args=(i,)) for i in range(len(subs))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        wall = time.perf_counter() - t0
        values = [r.value for r in results]
        report.append({"update": u, "wind": wind, "latency_s": wall,
                       "subsystems": {w.name: summarize(r, w.grid.size()) for w, r in zip(subs, results)},
                       "x_equals_y": bool(np.array_equal(results[1].value.values(),
                                                         results[2].value.values()))})
        print(json.dumps(report[-1]), flush=True)
    return report


def run_config5(max_iters, ctx):
    ws = configs.config5()
    fine = ws[-1]
    c = constraint(fine, ctx)
    cfg = hj.SolveConfig(**fine.cfg.__dict__)
    cfg.max_iters = max_iters
    r = hj.solve_multilevel(c, fine.model, fine.dbounds(), [w.grid for w in ws[:-1]], cfg, ctx=ctx)
    return {"levels": [dict(grid=str(w.grid.shape), **summarize(x, w.grid.size()))
                       for w, x in zip(ws, r.levels)], "wall_seconds": r.wall_seconds,
            "obstacles": configs.obstacles()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="*", default=["1", "2"])
    ap.add_argument("--max-iters", type=int, default=200000)
    ap.add_argument("--json", default=None)
    ap.add_argument("--tol4", type=float, default=5e-3,
                    help="config-4 tolerance (BASELINE leaves it open; the reference's own 10D "
                         "scenario uses 5e-3 for the 4D hover tail, sim.cpp:679)")
    a = ap.parse_args()
    ctx = hj.Context(0)
    out = {}
    for k in a.cfgs:
        t0 = time.perf_counter()
        if k == "1":
            out["1"] = run_single(configs.config1(), 20000, ctx)
        elif k == "2":
            out["2"] = run_single(configs.config2(51), a.max_iters, ctx)
        elif k == "3":
            out["3"] = run_single(configs.config3(101), a.max_iters, ctx)
        elif k == "4":
            out["4"] = run_config4(a.max_iters, ctx, a.tol4)
        elif k == "5":
            out["5"] = run_config5(a.max_iters, ctx)
        print(f"config {k}: {time.perf_counter() - t0:.1f} s wall", flush=True)
        if k != "4":
            print(json.dumps(out[k]), flush=True)
    if a.json:
        Path(a.json).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
