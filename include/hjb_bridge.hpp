// hjb_bridge.hpp — header-only C++ drop-in for the reference solver API.
//
// Include AFTER the reference's own headers (hjsafe/solver.hpp etc.).  Each
// function has the signature and exception behaviour of its reference
// counterpart (proj/include/hjsafe/solver.hpp:45-77) and runs on the GPU
// through the C ABI of include/hjb.h:
//
//   hjb_bridge::cfl_dt(grid, model, dbounds, cfl)          == hjsafe::cfl_dt
//   hjb_bridge::vi_step(V, c, model, dbounds, dt, cfg)     == hjsafe::vi_step
//   hjb_bridge::solve(init, c, model, dbounds, cfg)        == hjsafe::solve
//   hjb_bridge::solve_coarse_to_fine(...)                  == hjsafe::solve_coarse_to_fine
//
// Models: the reference classes with public parameters (Quad2DVert,
// NearHoverPlanar4D, NearHoverVertical2D, DoubleIntegrator) map to exact
// descriptors; any other DynamicsModel is probed through its own affine():
// rows whose drift varies along at most one axis become exact per-node
// tables, constant B/C are read off; other models raise
// std::invalid_argument (use the C ABI descriptor directly for those).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hjb.h"

namespace hjb_bridge {

namespace detail {

inline void check(int rc) {
  if (rc == HJB_OK) return;
  const std::string msg = hjb_last_error();
  if (rc == HJB_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);  // runtime / diverged / CUDA
}

struct Context {
  hjb_context* ctx = nullptr;
  Context() { check(hjb_context_create(0, &ctx)); }
  ~Context() { hjb_context_destroy(ctx); }
};

inline hjb_context* context() {
  thread_local Context c;  // one stream + workspace per calling thread (re-entrant)
  return c.ctx;
}

inline hjb_grid to_c(const hjsafe::Grid& g) {
  if (g.ndims() > HJB_MAX_DIMS)
    throw std::invalid_argument("hjb: grid rank above the device limit");
  hjb_grid o;
  std::memset(&o, 0, sizeof o);
  o.ndims = static_cast<int32_t>(g.ndims());
  for (std::size_t d = 0; d < g.ndims(); ++d)
    o.dims[d] = {g.dim(d).min, g.dim(d).max, static_cast<int64_t>(g.dim(d).n)};
  return o;
}

// every node holds the same bits (a field built by IntervalField::constant,
// interval_field.cpp:16-27, or any other uniform field)
inline bool uniform(const hjsafe::ScalarField& f) {
  const auto& v = f.values();
  if (v.empty()) return true;
  std::uint64_t b0;
  std::memcpy(&b0, v.data(), sizeof b0);
  for (std::size_t i = 1; i < v.size(); ++i) {
    std::uint64_t b;
    std::memcpy(&b, v.data() + i, sizeof b);
    if (b != b0) return false;
  }
  return true;
}

// The reference stores every IntervalField per node.  A field whose channels
// are uniform (bit for bit) is passed as constant bounds: 2 doubles per
// channel instead of 2N (1.66 GB at 101^4), and the solve takes the
// folded-slope kernels directly.  The values the solver reads are identical.
inline hjb_dbounds to_c(const hjsafe::IntervalField& f) {
  hjb_dbounds o;
  std::memset(&o, 0, sizeof o);
  o.channels = static_cast<int32_t>(f.channels());
  bool constant = true;
  for (std::size_t ch = 0; ch < f.channels() && constant; ++ch)
    constant = uniform(f.lo(ch)) && uniform(f.hi(ch));
  o.per_node = constant ? 0 : 1;
  for (std::size_t ch = 0; ch < f.channels(); ++ch) {
    if (constant) {
      o.constant[ch] = {f.lo(ch).values().empty() ? 0.0 : f.lo(ch)[0],
                        f.hi(ch).values().empty() ? 0.0 : f.hi(ch)[0]};
    } else {
      o.lo[ch] = f.lo(ch).values().data();
      o.hi[ch] = f.hi(ch).values().data();
    }
  }
  return o;
}

inline hjb_drift_term coord(int axis, double scale) { return {HJB_TERM_COORD, axis, scale, nullptr}; }
inline hjb_drift_term konst(double v) { return {HJB_TERM_CONST, 0, v, nullptr}; }

// Descriptor of a reference model; `tables` keeps probed tables alive.
inline hjb_model to_c(const hjsafe::DynamicsModel& m, const hjsafe::Grid& g,
                      std::vector<std::vector<double>>& tables) {
  hjb_model o;
  std::memset(&o, 0, sizeof o);
  o.state_dim = static_cast<int32_t>(m.state_dim());
  o.control_dim = static_cast<int32_t>(m.control_dim());
  o.disturbance_dim = static_cast<int32_t>(m.disturbance_dim());
  const auto ub = m.control_bounds();
  for (std::size_t j = 0; j < ub.size(); ++j) o.ubounds[j] = {ub[j].lo, ub[j].hi};
  if (auto* p = dynamic_cast<const hjsafe::NearHoverPlanar4D*>(&m)) {  // dynamics.cpp:134-143
    const auto& q = p->params();
    o.drift[0][0] = coord(1, 1.0);
    o.drift[1][0] = {HJB_TERM_TAN, 2, q.gravity, nullptr};
    o.drift[2][0] = coord(2, -q.d1);
    o.drift[2][1] = coord(3, 1.0);
    o.drift[3][0] = coord(2, -q.d0);
    o.control[3][0] = q.n0;
    o.disturbance[1][0] = 1.0;
    return o;
  }
  if (auto* p = dynamic_cast<const hjsafe::NearHoverVertical2D*>(&m)) {  // dynamics.cpp:145-151
    o.drift[0][0] = coord(1, 1.0);
    o.drift[1][0] = konst(-p->params().gravity);
    o.control[1][0] = p->params().thrust_gain;
    o.disturbance[1][0] = 1.0;
    return o;
  }
  if (auto* p = dynamic_cast<const hjsafe::Quad2DVert*>(&m)) {  // dynamics.cpp:126-132
    o.drift[0][0] = coord(1, 1.0);
    o.drift[1][0] = konst(p->params().gravity + p->params().k_offset);
    o.control[1][0] = p->params().k_thrust;
    o.disturbance[1][0] = 1.0;
    return o;
  }
  // Generic: probe affine() at grid nodes.
  const std::size_t nd = g.ndims();
  std::vector<double> x0(nd);
  for (std::size_t d = 0; d < nd; ++d) x0[d] = g.coord(d, 0);
  hjsafe::AffineFlow base;
  m.affine(x0, base);
  for (std::size_t i = 0; i < nd; ++i) {
    for (std::size_t j = 0; j < m.control_dim(); ++j) o.control[i][j] = base.control[i][j];
    for (std::size_t k = 0; k < m.disturbance_dim(); ++k)
      o.disturbance[i][k] = base.disturbance[i][k];
  }
  for (std::size_t i = 0; i < nd; ++i) {
    int axis = -1;
    std::vector<double> tab;
    for (std::size_t a = 0; a < nd; ++a) {
      std::vector<double> vals(g.dim(a).n);
      bool varies = false;
      for (std::size_t k = 0; k < g.dim(a).n; ++k) {
        std::vector<double> x = x0;
        x[a] = g.coord(a, k);
        hjsafe::AffineFlow af;
        m.affine(x, af);
        vals[k] = af.drift[i];
        for (std::size_t j = 0; j < m.control_dim(); ++j)
          if (af.control[i][j] != base.control[i][j])
            throw std::invalid_argument("hjb: state-dependent input matrix not supported");
        if (!(vals[k] == base.drift[i])) varies = true;
      }
      if (varies) {
        if (axis >= 0)
          throw std::invalid_argument("hjb: drift row depends on two axes; build the descriptor");
        axis = static_cast<int>(a);
        tab = std::move(vals);
      }
    }
    if (axis < 0) {
      o.drift[i][0] = konst(base.drift[i]);
    } else {
      tables.push_back(std::move(tab));
      o.drift[i][0] = {HJB_TERM_TABLE, axis, 0.0, tables.back().data()};
    }
  }
  return o;
}

inline hjb_solve_config to_c(const hjsafe::SolveConfig& c) {
  hjb_solve_config o;
  hjb_solve_config_default(&o);
  o.cfl_factor = c.cfl_factor;
  o.tolerance = c.tolerance;
  o.max_iters = static_cast<int64_t>(c.max_iters);
  o.scheme = c.scheme == hjsafe::SolveConfig::Scheme::kGodunov ? HJB_GODUNOV : HJB_LAX_FRIEDRICHS;
  o.dissipation = c.dissipation == hjsafe::SolveConfig::Dissipation::kGlobal ? HJB_GLOBAL
                                                                              : HJB_PER_NODE;
  return o;
}

}  // namespace detail

inline double cfl_dt(const hjsafe::Grid& grid, const hjsafe::DynamicsModel& model,
                     const hjsafe::IntervalField& dbounds, double cfl_factor, unsigned = 0) {
  std::vector<std::vector<double>> tabs;
  hjb_grid g = detail::to_c(grid);
  hjb_model m = detail::to_c(model, grid, tabs);
  hjb_dbounds d = detail::to_c(dbounds);
  double dt = 0.0;
  detail::check(hjb_cfl_dt(detail::context(), &g, &m, &d, cfl_factor, &dt));
  return dt;
}

inline hjsafe::ScalarField vi_step(const hjsafe::ScalarField& value,
                                   const hjsafe::ScalarField& constraint,
                                   const hjsafe::DynamicsModel& model,
                                   const hjsafe::IntervalField& dbounds, double dt,
                                   const hjsafe::SolveConfig& cfg = {}) {
  if (!(value.grid() == constraint.grid()))
    throw std::invalid_argument("vi_step: value/constraint grid mismatch");
  std::vector<std::vector<double>> tabs;
  hjb_grid g = detail::to_c(value.grid());
  hjb_model m = detail::to_c(model, value.grid(), tabs);
  hjb_dbounds d = detail::to_c(dbounds);
  hjb_solve_config c = detail::to_c(cfg);
  std::vector<double> out(value.size());
  detail::check(hjb_vi_step(detail::context(), &g, &m, &d, value.values().data(),
                            constraint.values().data(), dt, &c, out.data()));
  return hjsafe::ScalarField(value.grid(), std::move(out));
}

inline hjsafe::SolveResult solve(const hjsafe::ScalarField& init,
                                 const hjsafe::ScalarField& constraint,
                                 const hjsafe::DynamicsModel& model,
                                 const hjsafe::IntervalField& dbounds,
                                 const hjsafe::SolveConfig& cfg) {
  cfg.validate();
  if (!(init.grid() == constraint.grid()))
    throw std::invalid_argument("solve: init/constraint grid mismatch");
  std::vector<std::vector<double>> tabs;
  hjb_grid g = detail::to_c(init.grid());
  hjb_model m = detail::to_c(model, init.grid(), tabs);
  hjb_dbounds d = detail::to_c(dbounds);
  hjb_solve_config c = detail::to_c(cfg);
  std::vector<double> out(init.size());
  hjsafe::SolveResult r;
  r.residual_history.resize(cfg.max_iters);
  r.wall_ms_history.resize(cfg.max_iters);
  hjb_solve_result res;
  std::memset(&res, 0, sizeof res);
  res.residual_history = r.residual_history.data();
  res.wall_ms_history = r.wall_ms_history.data();
  res.history_capacity = static_cast<int64_t>(cfg.max_iters);
  detail::check(hjb_solve(detail::context(), &g, &m, &d, init.values().data(),
                          constraint.values().data(), &c, out.data(), &res));
  r.value = hjsafe::ScalarField(init.grid(), std::move(out));
  r.iterations = static_cast<std::size_t>(res.iterations);
  r.dt = res.dt;
  r.wall_seconds = res.wall_seconds;
  r.converged = res.converged != 0;
  r.nodes_per_sweep = static_cast<std::size_t>(res.nodes_per_sweep);
  r.residual_history.resize(r.iterations);
  r.wall_ms_history.resize(r.iterations);
  return r;
}

inline hjsafe::CoarseToFineResult solve_coarse_to_fine(
    const hjsafe::ScalarField& constraint_fine, const hjsafe::DynamicsModel& model,
    const hjsafe::IntervalField& dbounds_fine, const hjsafe::Grid& coarse_grid,
    const hjsafe::SolveConfig& cfg, const hjsafe::ScalarField* warm_init_fine = nullptr) {
  cfg.validate();
  if (coarse_grid.ndims() != constraint_fine.grid().ndims())
    throw std::invalid_argument("solve_coarse_to_fine: grid rank mismatch");
  std::vector<std::vector<double>> tabs;
  hjb_grid grids[2] = {detail::to_c(coarse_grid), detail::to_c(constraint_fine.grid())};
  hjb_model m = detail::to_c(model, constraint_fine.grid(), tabs);
  hjb_dbounds d = detail::to_c(dbounds_fine);
  hjb_solve_config c = detail::to_c(cfg);
  std::vector<double> vc(coarse_grid.size()), vf(constraint_fine.size());
  double* outs[2] = {vc.data(), vf.data()};
  std::vector<double> h[4];
  hjb_solve_result res[2];
  std::memset(res, 0, sizeof res);
  for (int l = 0; l < 2; ++l) {
    h[2 * l].resize(cfg.max_iters);
    h[2 * l + 1].resize(cfg.max_iters);
    res[l].residual_history = h[2 * l].data();
    res[l].wall_ms_history = h[2 * l + 1].data();
    res[l].history_capacity = static_cast<int64_t>(cfg.max_iters);
  }
  double wall = 0.0;
  detail::check(hjb_solve_multilevel(detail::context(), 2, grids, &m, &d,
                                     constraint_fine.values().data(), &c,
                                     warm_init_fine ? warm_init_fine->values().data() : nullptr,
                                     outs, res, &wall));
  hjsafe::CoarseToFineResult out;
  hjsafe::SolveResult* rs[2] = {&out.coarse, &out.fine};
  const hjsafe::Grid* gs[2] = {&coarse_grid, &constraint_fine.grid()};
  std::vector<double>* vs[2] = {&vc, &vf};
  for (int l = 0; l < 2; ++l) {
    rs[l]->value = hjsafe::ScalarField(*gs[l], std::move(*vs[l]));
    rs[l]->iterations = static_cast<std::size_t>(res[l].iterations);
    rs[l]->dt = res[l].dt;
    rs[l]->wall_seconds = res[l].wall_seconds;
    rs[l]->converged = res[l].converged != 0;
    rs[l]->nodes_per_sweep = static_cast<std::size_t>(res[l].nodes_per_sweep);
    rs[l]->residual_history.assign(h[2 * l].begin(), h[2 * l].begin() + res[l].iterations);
    rs[l]->wall_ms_history.assign(h[2 * l + 1].begin(), h[2 * l + 1].begin() + res[l].iterations);
  }
  out.wall_seconds = wall;
  return out;
}

}  // namespace hjb_bridge
