// bridge_demo.cpp — TEST: the C++ drop-in (include/hjb_bridge.hpp) against
// the reference itself, in one process.  Built only where /root/reference
// exists (the reference sources are linked in as the checker); the binary
// travels to the GPU box.  Exit codes: 0 parity ok, 1 mismatch, 3 no GPU.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "hjsafe/levelset.hpp"
#include "hjsafe/solver.hpp"
// after the reference headers
#include "hjb_bridge.hpp"

using namespace hjsafe;

namespace {

class ConstantAdvection final : public DynamicsModel {  // test_solver.cpp:14-29
 public:
  explicit ConstantAdvection(std::vector<double> s) : s_(std::move(s)) {}
  std::size_t state_dim() const override { return s_.size(); }
  std::size_t control_dim() const override { return 0; }
  std::size_t disturbance_dim() const override { return 0; }
  std::string name() const override { return "advection"; }
  std::vector<Interval> control_bounds() const override { return {}; }
  void affine(std::span<const double>, AffineFlow& out) const override {
    out.reset(s_.size(), 0, 0);
    for (std::size_t i = 0; i < s_.size(); ++i) out.drift[i] = s_[i];
  }

 private:
  std::vector<double> s_;
};

// A user's own 4D model (no reference class, no compiled kernel shape): the
// bridge probes affine() into one-axis drift tables, and the solve runs the
// run-time-shape 4D sweep (k_fast4d<ShapeGen>).
class UserModel4D final : public DynamicsModel {
 public:
  std::size_t state_dim() const override { return 4; }
  std::size_t control_dim() const override { return 1; }
  std::size_t disturbance_dim() const override { return 1; }
  std::string name() const override { return "user4d"; }
  std::vector<Interval> control_bounds() const override { return {{-1.0, 1.0}}; }
  void affine(std::span<const double> x, AffineFlow& out) const override {
    out.reset(4, 1, 1);
    out.drift[0] = x[1];
    out.drift[1] = -0.2 * x[3] * x[3] * x[3];
    out.drift[2] = x[3];
    out.drift[3] = -9.8 * std::sin(x[2]);
    out.control[3][0] = 2.0;
    out.disturbance[0][0] = 1.0;
  }
};

bool same(const ScalarField& a, const ScalarField& b) {
  if (a.size() != b.size()) return false;
  for (std::size_t i = 0; i < a.size(); ++i)
    if (!(a[i] == b[i])) return false;
  return true;
}

int fails = 0;
void expect(bool ok, const char* what) {
  std::printf("%s %s\n", ok ? "ok  " : "FAIL", what);
  if (!ok) ++fails;
}

}  // namespace

int main() {
  try {
    int n = 0;
    hjb_device_count(&n);
    if (n == 0) {
      std::printf("no CUDA device\n");
      return 3;
    }
    // config-1 model: NearHoverVertical2D{g=9.81, kT=0.91, 0, 2}, band z in [0,3]
    NearHoverVertical2D::Params vp;
    vp.gravity = 9.81;
    vp.thrust_gain = 0.91;
    vp.thrust_frac_lo = 0.0;
    vp.thrust_frac_hi = 2.0;
    NearHoverVertical2D vert(vp);
    Grid g({{-2.0, 4.0, 101}, {-4.0, 4.0, 101}});
    ScalarField c = signed_distance_band(g, 0, 0.0, 3.0);
    auto db = IntervalField::constant(g, std::vector<Interval>{{-0.5, 0.5}});
    SolveConfig cfg;
    cfg.tolerance = 1e-4;
    SolveResult ref = solve(c, c, vert, db, cfg);
    SolveResult gpu = hjb_bridge::solve(c, c, vert, db, cfg);
    expect(ref.iterations == gpu.iterations && ref.iterations == 146, "config 1: 146 iterations");
    expect(same(ref.value, gpu.value), "config 1: V* bitwise equal to the reference");
    expect(ref.residual_history == gpu.residual_history, "config 1: residual history equal");

    // stock NearHoverPlanar4D (reference class, d on row 1), 9^4, 40 sweeps
    NearHoverPlanar4D planar("x");
    Grid g4({{-5.0, 5.0, 9}, {-2.0, 2.0, 9}, {-0.35, 0.35, 9}, {-1.5, 1.5, 9}});
    ScalarField c4 = signed_distance_band(g4, 0, -4.0, 4.0);
    auto db4 = IntervalField::constant(g4, std::vector<Interval>{{-0.5, 0.5}});
    SolveConfig cfg4;
    cfg4.max_iters = 40;
    SolveResult r4 = solve(c4, c4, planar, db4, cfg4);
    SolveResult g4r = hjb_bridge::solve(c4, c4, planar, db4, cfg4);
    expect(same(r4.value, g4r.value) && r4.iterations == g4r.iterations,
           "NearHoverPlanar4D 9^4: bitwise equal");

    // full config-2 grid size through the drop-in, timed: stock
    // NearHoverPlanar4D on 51^4, 20 sweeps.  The reference IntervalField is
    // per node; the bridge detects the uniform channel and ships 2 doubles.
    {
      Grid g51({{-5.0, 5.0, 51}, {-2.0, 2.0, 51}, {-0.35, 0.35, 51}, {-1.5, 1.5, 51}});
      ScalarField c51 = signed_distance_band(g51, 0, -4.0, 4.0);
      auto db51 = IntervalField::constant(g51, std::vector<Interval>{{-0.5, 0.5}});
      SolveConfig k20;
      k20.max_iters = 20;
      hjb_bridge::solve(c51, c51, planar, db51, k20);  // warm-up (autotuner, context)
      auto t0 = std::chrono::steady_clock::now();
      SolveResult rg = hjb_bridge::solve(c51, c51, planar, db51, k20);
      auto t1 = std::chrono::steady_clock::now();
      SolveResult rr = solve(c51, c51, planar, db51, k20);
      auto t2 = std::chrono::steady_clock::now();
      const double sg = std::chrono::duration<double>(t1 - t0).count();
      const double sr = std::chrono::duration<double>(t2 - t1).count();
      std::printf("51^4 x 20 sweeps: bridge %.1f ms (host buffers in and out), reference %.1f ms"
                  " (%.0fx)\n", sg * 1e3, sr * 1e3, sr / sg);
      expect(same(rr.value, rg.value) && rr.iterations == rg.iterations &&
                 rr.residual_history == rg.residual_history,
             "NearHoverPlanar4D 51^4 x 20: bitwise equal, constant bounds detected");
    }

    // a user-defined 4D model through the drop-in: probed tables, run-time
    // row shapes; bitwise on 21^4 x 40 sweeps, then 51^4 x 20 sweeps timed
    {
      UserModel4D user;
      Grid gu({{-5.0, 5.0, 21}, {-2.0, 2.0, 21}, {-0.35, 0.35, 21}, {-1.5, 1.5, 21}});
      ScalarField cu = signed_distance_band(gu, 0, -4.0, 4.0);
      auto dbu = IntervalField::constant(gu, std::vector<Interval>{{-0.5, 0.5}});
      SolveConfig k40;
      k40.max_iters = 40;
      SolveResult ru = solve(cu, cu, user, dbu, k40);
      SolveResult gu40 = hjb_bridge::solve(cu, cu, user, dbu, k40);
      expect(same(ru.value, gu40.value) && ru.iterations == gu40.iterations &&
                 ru.residual_history == gu40.residual_history,
             "user-defined 4D model 21^4 x 40: bitwise equal");
      Grid g51({{-5.0, 5.0, 51}, {-2.0, 2.0, 51}, {-0.35, 0.35, 51}, {-1.5, 1.5, 51}});
      ScalarField c51 = signed_distance_band(g51, 0, -4.0, 4.0);
      auto db51 = IntervalField::constant(g51, std::vector<Interval>{{-0.5, 0.5}});
      SolveConfig k20;
      k20.max_iters = 20;
      hjb_bridge::solve(c51, c51, user, db51, k20);  // warm-up
      auto t0 = std::chrono::steady_clock::now();
      SolveResult rg = hjb_bridge::solve(c51, c51, user, db51, k20);
      auto t1 = std::chrono::steady_clock::now();
      SolveResult rr = solve(c51, c51, user, db51, k20);
      auto t2 = std::chrono::steady_clock::now();
      const double sg = std::chrono::duration<double>(t1 - t0).count();
      const double sr = std::chrono::duration<double>(t2 - t1).count();
      std::printf("user 4D model 51^4 x 20 sweeps: bridge %.1f ms (host buffers in and out), "
                  "reference %.1f ms (%.0fx)\n", sg * 1e3, sr * 1e3, sr / sg);
      expect(same(rr.value, rg.value) && rr.iterations == rg.iterations,
             "user-defined 4D model 51^4 x 20: bitwise equal");
    }

    // coarse-to-fine (test_solver.cpp:253-278 setup)
    Quad2DVert quad;
    Grid gq({{0.0, 3.2, 41}, {-5.0, 5.0, 41}});
    Grid gc({{0.0, 3.2, 21}, {-5.0, 5.0, 21}});
    ScalarField cq = signed_distance_band(gq, 0, 0.35, 2.8);
    auto dbq = IntervalField::constant(gq, std::vector<Interval>{{-0.3, 0.3}});
    SolveConfig cq_cfg;
    auto a = solve_coarse_to_fine(cq, quad, dbq, gc, cq_cfg);
    auto b = hjb_bridge::solve_coarse_to_fine(cq, quad, dbq, gc, cq_cfg);
    expect(same(a.coarse.value, b.coarse.value) && same(a.fine.value, b.fine.value) &&
               a.fine.iterations == b.fine.iterations,
           "solve_coarse_to_fine: both stages bitwise equal");

    // probed model (reference test model): cfl_dt formula and exceptions
    ConstantAdvection adv({2.0, 10.1});
    Grid ga({{0.0, 1.0, 21}, {0.0, 1.4, 21}});
    auto dba = IntervalField::constant(ga, std::vector<Interval>{});
    expect(cfl_dt(ga, adv, dba, 0.8) == hjb_bridge::cfl_dt(ga, adv, dba, 0.8),
           "cfl_dt of a probed test model equal");
    bool threw = false;
    try {
      ConstantAdvection zero({0.0});
      Grid gz({{0.0, 1.0, 11}});
      hjb_bridge::cfl_dt(gz, zero, IntervalField::constant(gz, std::vector<Interval>{}), 0.8);
    } catch (const std::runtime_error&) {
      threw = true;
    }
    expect(threw, "zero flow raises std::runtime_error");
    threw = false;
    try {
      SolveConfig bad;
      bad.cfl_factor = 1.5;
      hjb_bridge::solve(c, c, vert, db, bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    expect(threw, "bad cfl raises std::invalid_argument");
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 1;
  }
  return fails ? 1 : 0;
}
