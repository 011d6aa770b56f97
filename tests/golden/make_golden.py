"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref).

Run in the build container, where /root/reference exists:
    python tests/golden/make_golden.py
Writes tests/golden/golden_v1.npz (small arrays), golden_v1.json (scalars,
iteration counts, SHA-256 of larger fields with -0 normalised to +0) and
cfg1_value.hjvf (the config-1 converged V* in the reference's own HJVF
format, written by the reference's write_hjvf).
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent))

from oracle.oracle import Reference  # noqa: E402
from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402
from cases import band_np, quad_setup, solve_cases, twin_case, with_iters, workload_case  # noqa: E402


def h(v):
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64) + 0.0)
    return hashlib.sha256(v.tobytes()).hexdigest()


def main():
    ref = Reference()
    arrays, meta = {}, {}
    for case, iters in solve_cases():
        c = with_iters(case, iters)
        r = ref.solve(c.init_field(), c.c_field(), c.model, c.db, c.cfg)
        meta[c.name] = {"iterations": r.iterations, "converged": r.converged, "dt": r.dt,
                        "value_sha256": h(r.value.values()),
                        "history_sha256": h(r.residual_history), "max_iters": iters}
        if c.grid.size() <= 20000:
            arrays[c.name + "/value"] = r.value.values()
            arrays[c.name + "/history"] = r.residual_history
    # config 2 at 21^4, 200 sweeps (reference parity at a size the CPU runs fast)
    c = with_iters(workload_case(configs.config2(21)), 200)
    r = ref.solve(c.init_field(), c.c_field(), c.model, c.db, c.cfg)
    meta["cfg2_21_k200"] = {"iterations": r.iterations, "dt": r.dt, "value_sha256": h(r.value.values()),
                            "history_sha256": h(r.residual_history)}
    arrays["cfg2_21_k200/history"] = r.residual_history
    # resample / seed known answers
    rng = np.random.default_rng(11)
    src_g, dst_g = configs.planar_grid(7), configs.planar_grid(13)
    f = hj.ScalarField(src_g, rng.standard_normal(src_g.size()))
    arrays["resample/src"] = f.values()
    meta["resample_7_13"] = {"value_sha256": h(ref.resample(f, dst_g)),
                             "max_adjacent_jump": ref.max_adjacent_jump(f)}
    # coarse to fine (test_solver.cpp:253-278 setup)
    q = quad_setup(41)
    coarse = hj.Grid([(0.0, 3.2, 21), (-5.0, 5.0, 21)])
    ctf = ref.solve_coarse_to_fine(q.c_field(), q.model, q.db, coarse, q.cfg)
    meta["ctf_quad41_21"] = {"coarse_iterations": ctf.coarse.iterations,
                             "fine_iterations": ctf.fine.iterations,
                             "coarse_sha256": h(ctf.coarse.value.values()),
                             "fine_sha256": h(ctf.fine.value.values())}
    # cfl_dt known answers (test_solver.cpp:48-78)
    for name, speeds, dims in (("cfl_1d", [10.1], [(0.0, 1.0, 21)]),
                               ("cfl_2d", [2.0, 10.1], [(0.0, 1.0, 21), (0.0, 1.4, 21)])):
        g = hj.Grid(dims)
        meta[name] = {"dt": ref.cfl_dt(g, hj.ConstantAdvection(speeds), hj.IntervalField.constant(g, []), 0.8)}
    # the reference's own HJVF file of the config-1 fixed point
    c1 = workload_case(configs.config1())
    r1 = ref.solve(c1.init_field(), c1.c_field(), c1.model, c1.db, c1.cfg)
    ref.write_hjvf(HERE / "cfg1_value.hjvf", r1.value)
    np.savez_compressed(HERE / "golden_v1.npz", **arrays)
    (HERE / "golden_v1.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(f"wrote {len(arrays)} arrays, {len(meta)} records")


if __name__ == "__main__":
    main()
