"""Per-sweep device time of config-5 level grids solved on their own vs inside
the multilevel chain (diagnostic).

usage: python scripts/diag_levels.py [iters=300]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402
from scripts.run_configs import constraint  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    ctx = hj.Context(0)
    ws = configs.config5()
    for w in ws[:2]:
        c = constraint(w, ctx)
        cfg = hj.SolveConfig(**w.cfg.__dict__)
        cfg.max_iters, cfg.tolerance = iters, 1e-300
        n = w.grid.size()
        pn = hj.IntervalField(w.grid, 1, lo=[np.full(n, -0.6)], hi=[np.full(n, 0.6)])
        rng = np.random.default_rng(1)
        noise = 1e-16 * rng.standard_normal(n)
        pv = hj.IntervalField(w.grid, 1, lo=[-0.6 + noise], hi=[0.6 + noise])
        for label, db in (("constant", w.dbounds()), ("per-node constant", pn),
                          ("per-node noisy", pv)):
            l0 = ctx.launches
            r = hj.solve(c, c, w.model, db, cfg, ctx=ctx)
            print(f"{w.grid.shape} {label}: {r.wall_seconds / r.iterations * 1e6:.1f} us/sweep, "
                  f"launches {ctx.launches - l0}")


if __name__ == "__main__":
    main()
