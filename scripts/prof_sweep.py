"""Run a short device-resident config-2/3 solve chunk (for ncu / timing).

usage: python scripts/prof_sweep.py [n=51] [iters=20] [reps=3]
Prints the average sweep time from the library's device events.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 51
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    w = configs.config2(n)
    ctx = hj.Context(0)
    cells = w.grid.size()
    c = torch.empty(cells, dtype=torch.float64, device="cuda")
    out = torch.empty_like(c)
    torch.cuda.synchronize()
    hj.signed_distance_band_dev(w.grid, 0, -4.0, 4.0, c.data_ptr(), ctx=ctx)
    cfg = hj.SolveConfig(**w.cfg.__dict__)
    cfg.max_iters = iters
    for r in range(reps):
        res = hj.solve_dev(w.grid, w.model, w.dbounds(), c.data_ptr(), c.data_ptr(), out.data_ptr(),
                           cfg, ctx=ctx)
        us = res.wall_seconds / res.iterations * 1e6
        print(f"n={n} cells={cells} iters={res.iterations} sweep={us:.1f} us "
              f"-> {cells / us * 1e-3:.2f} Gcell/s, {24 * cells / us * 1e-3:.0f} GB/s algorithmic")


if __name__ == "__main__":
    main()
