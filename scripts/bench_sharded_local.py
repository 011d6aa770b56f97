"""Time the slab-partitioned protocol on ONE GPU with in-process ranks.

hjb_solve_sharded_local_dev runs every rank's plan (boundary planes first,
halo copies on a second stream while the interior sweeps, pipelined residual
reduction + epilogue) on one device, so the ranks' sweeps execute one after
another: the per-sweep time of P local ranks minus the unsharded sweep time is
the protocol's own cost on the critical path (extra launches, waits, copies
that were not hidden).  Variants: HJB_SHARD_OVERLAP / HJB_SHARD_PIPE / HJB_SHARD_P2P.

    python scripts/bench_sharded_local.py [--n 101] [--sweeps 200] > out.json
"""
import argparse
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402
from paper_2101_05916_b200 import sharded  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=101)
    ap.add_argument("--sweeps", type=int, default=200)
    ap.add_argument("--ho-steps", type=int, default=6)
    ap.add_argument("--ranks", default="1,2,4,8")
    a = ap.parse_args()
    w = configs.config3(a.n)
    g, cells = w.grid, w.grid.size()
    ctx = hj.Context(0)
    c = torch.empty(cells, dtype=torch.float64, device="cuda")
    out = torch.empty_like(c)
    torch.cuda.synchronize()
    hj.signed_distance_band_dev(g, 0, -4.0, 4.0, c.data_ptr(), ctx=ctx)
    res = {"grid": f"{a.n}^4", "cells": cells, "first_order": {}, "eno3_rk3": {}}

    def run(order, rk, iters, P, env):
        for k, v in env.items():
            os.environ[k] = v
        cfg = hj.SolveConfig(**w.cfg.__dict__)
        cfg.max_iters, cfg.spatial_order, cfg.time_order = iters, order, rk
        f = (lambda: hj.solve_dev(g, w.model, w.dbounds(), c.data_ptr(), c.data_ptr(),
                                  out.data_ptr(), cfg, ctx=ctx)) if P == 0 else \
            (lambda: sharded.solve_sharded_local_dev(P, g, w.model, w.dbounds(), c.data_ptr(),
                                                     c.data_ptr(), out.data_ptr(), cfg, ctx))
        f()
        best = min(f().wall_seconds for _ in range(3))
        for k in env:
            os.environ.pop(k, None)
        return best / iters * 1e6

    variants = {"overlap+pipe": {}, "peer_store": {"HJB_SHARD_P2P": "1"},
                "serial": {"HJB_SHARD_OVERLAP": "0", "HJB_SHARD_PIPE": "0"},
                "overlap_only": {"HJB_SHARD_PIPE": "0"},
                "serial_one_launch": {"HJB_SHARD_OVERLAP": "0", "HJB_SHARD_PIPE": "0",
                                      "HJB_SHARD_SPLIT": "0"}}
    ranks = [int(x) for x in a.ranks.split(",")]
    res["first_order"]["unsharded_us"] = run(1, 1, a.sweeps, 0, {})
    for name, env in variants.items():
        res["first_order"][name] = {str(P): run(1, 1, a.sweeps, P, env) for P in ranks}
    res["eno3_rk3"]["unsharded_us"] = run(3, 3, a.ho_steps, 0, {})
    for name, env in variants.items():
        if name == "peer_store":  # first order only
            continue
        res["eno3_rk3"][name] = {str(P): run(3, 3, a.ho_steps, P, env) for P in ranks if P <= 8}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
