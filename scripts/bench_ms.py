"""Per-sweep device time of the 4D fast path: graph loop (one k_fast4d launch
per sweep, PDL) vs the multi-sweep persistent kernel (HJB_MS=1), constant
and per-node bounds, several grid sizes.  Prints JSON."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402


def main():
    sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "21,26,31,41,51,71").split(",")]
    ctx = hj.Context(0)
    out = {}
    for n in sizes:
        w = configs.config2(n)
        g = w.grid
        c = torch.empty(g.size(), dtype=torch.float64, device="cuda")
        o = torch.empty_like(c)
        torch.cuda.synchronize()
        hj.signed_distance_band_dev(g, 0, -4.0, 4.0, c.data_ptr(), ctx=ctx)
        rng = np.random.default_rng(1)
        lo = torch.tensor(-0.5 - 1e-12 * rng.random(g.size()), device="cuda")
        hi = torch.tensor(0.5 + 1e-12 * rng.random(g.size()), device="cuda")
        iters = max(200, int(2e9 / g.size()) // 8 * 8)
        rec = {}
        for bounds in ("constant", "per_node"):
            for ms in ("0", "1"):
                os.environ["HJB_MS"] = ms
                cfg = hj.SolveConfig(**w.cfg.__dict__)
                cfg.max_iters, cfg.tolerance = iters, 1e-30
                if bounds == "constant":
                    f = lambda: hj.solve_dev(g, w.model, w.dbounds(), c.data_ptr(), c.data_ptr(),
                                             o.data_ptr(), cfg, ctx=ctx)
                else:
                    import ctypes as C
                    from paper_2101_05916_b200 import abi
                    d = abi.HjbDbounds()
                    d.channels, d.per_node = 1, 1
                    d.lo[0] = C.cast(C.c_void_p(lo.data_ptr()), C.POINTER(C.c_double))
                    d.hi[0] = C.cast(C.c_void_p(hi.data_ptr()), C.POINTER(C.c_double))

                    def f():
                        r, rh, wh = hj._c_result(0)
                        gg, m, k = g.to_c(), w.model.to_c(), cfg.to_c()
                        hj._check(abi.load().hjb_solve_dev(ctx.handle, C.byref(gg), C.byref(m),
                                                           C.byref(d), C.c_void_p(c.data_ptr()),
                                                           C.c_void_p(c.data_ptr()), C.byref(k),
                                                           C.c_void_p(o.data_ptr()), C.byref(r)))
                        return r
                f()
                ts = [f().wall_seconds for _ in range(3)]
                rec[f"{bounds}_ms{ms}_us"] = min(ts) / iters * 1e6
        os.environ.pop("HJB_MS", None)
        rec["sweeps"] = iters
        out[f"{n}^4"] = rec
        print(json.dumps({f"{n}^4": rec}), flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
