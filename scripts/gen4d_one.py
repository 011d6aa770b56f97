import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2101_05916_b200 import hjsafe as hj
from test_gpu_gen4d import MODELS
name = sys.argv[1]
make, nd = MODELS[name]
n = 101
ctx = hj.Context(0)
g = hj.Grid([(-5.0, 5.0, n), (-2.0, 2.0, n), (-0.35, 0.35, n), (-1.5, 1.5, n)])
c = hj.signed_distance_band(g, 0, -4.0, 4.0, ctx=ctx)
db = hj.IntervalField.constant(g, [hj.Interval(-0.5, 0.5)] * nd)
r = hj.solve(c, c, make(), db, hj.SolveConfig(tolerance=1e-12, max_iters=12), ctx=ctx)
print(name, r.kernel, r.wall_seconds / r.iterations * 1e6, "us per sweep")
