"""Time ENO/TVD-RK solve chunks (BASELINE config 3 scheme) on the device.

usage: python scripts/prof_ho.py [n=101] [iters=20] [order=3] [rk=3] [reps=2] [scheme=gd|lf|lfg]
Prints per-step device time and the algorithmic HBM rate (24 + 32*(rk-1) B
per cell-step).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402


def main():
    args = sys.argv[1:6]
    a = [int(x) for x in args] + [101, 20, 3, 3, 2][len(args):]
    n, iters, order, rk, reps = a[:5]
    scheme = sys.argv[6] if len(sys.argv) > 6 else "gd"
    w = configs.config2(n)
    ctx = hj.Context(0)
    cells = w.grid.size()
    c = torch.empty(cells, dtype=torch.float64, device="cuda")
    out = torch.empty_like(c)
    torch.cuda.synchronize()
    hj.signed_distance_band_dev(w.grid, 0, -4.0, 4.0, c.data_ptr(), ctx=ctx)
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.max_iters, cfg.spatial_order, cfg.time_order = iters, order, rk
    if scheme != "gd":
        cfg.scheme = hj.LAX_FRIEDRICHS
        cfg.dissipation = hj.GLOBAL if scheme == "lfg" else hj.PER_NODE
    bpc = 24 + 32 * (rk - 1)
    for _ in range(reps):
        r = hj.solve_dev(w.grid, w.model, w.dbounds(), c.data_ptr(), c.data_ptr(), out.data_ptr(),
                         cfg, ctx=ctx)
        us = r.wall_seconds / r.iterations * 1e6
        print(f"n={n} {scheme} ENO{order}/RK{rk} iters={r.iterations} step={us:.1f} us -> "
              f"{cells / us * 1e-3:.2f} Gcell/s, {bpc * cells / us * 1e-3:.0f} GB/s algorithmic "
              f"({bpc} B/cell-step)")


if __name__ == "__main__":
    main()
