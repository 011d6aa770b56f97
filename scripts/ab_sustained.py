"""Sustained (power-capped) per-sweep time of the 101^4 first-order sweep for
kernel variants, interleaved in one process: each sample is one solve of
--sweeps sweeps (seconds of load, so the board reaches its power-cap clocks).

    python scripts/ab_sustained.py [--sweeps 4000] [--rounds 3]
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

VARIANTS_B = {
    "default (autotuned)": {},
    "2 cells x 448": {"HJB_KCELLS": "2", "HJB_MAXT": "448"},
    "cplane 2 x 576": {"HJB_CPLANE": "1", "HJB_KCELLS": "2", "HJB_MAXT": "576"},
    "cplane 2 x 448": {"HJB_CPLANE": "1", "HJB_KCELLS": "2", "HJB_MAXT": "448"},
    "cplane 4 x 384": {"HJB_CPLANE": "1", "HJB_KCELLS": "4"},
}
VARIANTS = {
    "default (autotuned)": {},
    "2 cells x 576": {"HJB_KCELLS": "2", "HJB_MAXT": "576"},
    "2 cells x 448": {"HJB_KCELLS": "2", "HJB_MAXT": "448"},
    "4 cells x 384": {"HJB_KCELLS": "4"},
    "constraint per plane": {"HJB_CPLANE": "1", "HJB_KCELLS": "2", "HJB_MAXT": "576"},
    "no PDL": {"HJB_PDL": "0", "HJB_KCELLS": "2", "HJB_MAXT": "576"},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=101)
    ap.add_argument("--sweeps", type=int, default=4000)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--set", default="a", choices=["a", "b"])
    a = ap.parse_args()
    w = configs.config3(a.n)
    g = w.grid
    ctx = hj.Context(0)
    c = torch.empty(g.size(), dtype=torch.float64, device="cuda")
    out = torch.empty_like(c)
    torch.cuda.synchronize()
    hj.signed_distance_band_dev(g, 0, -4.0, 4.0, c.data_ptr(), ctx=ctx)
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.max_iters, cfg.tolerance = a.sweeps, 1e-30
    variants = VARIANTS if a.set == "a" else VARIANTS_B
    res = {k: [] for k in variants}
    for rnd in range(a.rounds):
        for name, env in variants.items():
            for k in ("HJB_KCELLS", "HJB_MAXT", "HJB_CPLANE", "HJB_PDL"):
                os.environ.pop(k, None)
            os.environ.update(env)
            r = hj.solve_dev(g, w.model, w.dbounds(), c.data_ptr(), c.data_ptr(), out.data_ptr(),
                             cfg, ctx=ctx)
            res[name].append(r.wall_seconds / r.iterations * 1e6)
            print(json.dumps({"round": rnd, "variant": name, "us_per_sweep": res[name][-1]}),
                  flush=True)
    print(json.dumps({k: {"median_us": statistics.median(v), "samples": v} for k, v in res.items()},
                     indent=1))


if __name__ == "__main__":
    main()
