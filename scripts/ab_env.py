"""Sustained A/B of environment-selected variants, interleaved in one process.

    python scripts/ab_env.py --n 101 --order 1 --iters 4000 --rounds 2 \
        --variants '{"default": {}, "tile 4x2": {"HJB_TILE": "4x2"}}'

Each sample is one device-resident solve of --iters steps from V = c (seconds
of load: the board sits at its power cap, as in a long solve).
"""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=101)
    ap.add_argument("--order", type=int, default=1)
    ap.add_argument("--lf", action="store_true")
    ap.add_argument("--iters", type=int, default=4000)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--variants", required=True)
    a = ap.parse_args()
    variants = json.loads(a.variants)
    keys = sorted({k for v in variants.values() for k in v})
    w = configs.config3(a.n)
    g = w.grid
    ctx = hj.Context(0)
    c = torch.empty(g.size(), dtype=torch.float64, device="cuda")
    out = torch.empty_like(c)
    torch.cuda.synchronize()
    hj.signed_distance_band_dev(g, 0, -4.0, 4.0, c.data_ptr(), ctx=ctx)
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.max_iters, cfg.tolerance = a.iters, 1e-30
    cfg.spatial_order = cfg.time_order = a.order
    if a.lf:
        cfg.scheme = hj.LAX_FRIEDRICHS
    res = {k: [] for k in variants}
    for rnd in range(a.rounds):
        for name, env in variants.items():
            for k in keys:
                os.environ.pop(k, None)
            os.environ.update(env)
            r = hj.solve_dev(g, w.model, w.dbounds(), c.data_ptr(), c.data_ptr(), out.data_ptr(),
                             cfg, ctx=ctx)
            res[name].append(r.wall_seconds / r.iterations * 1e6)
            print(json.dumps({"round": rnd, "variant": name, "us_per_step": res[name][-1]}),
                  flush=True)
    print(json.dumps({k: statistics.median(v) for k, v in res.items()}, indent=1))


if __name__ == "__main__":
    main()
