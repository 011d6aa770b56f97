"""One first-order solve of the config-2 model (for ncu captures):
python scripts/fo_one.py [n=51] [iters=12]"""
import sys
sys.path.insert(0, ".")
from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 51
it = int(sys.argv[2]) if len(sys.argv) > 2 else 12
w = configs.config2(n)
ctx = hj.Context(0)
c = hj.signed_distance_band(w.grid, 0, -4.0, 4.0, ctx=ctx)
r = hj.solve(c, c, w.model, w.dbounds(), hj.SolveConfig(tolerance=1e-12, max_iters=it), ctx=ctx)
print(n, r.kernel, r.wall_seconds / r.iterations * 1e6, "us per sweep")
