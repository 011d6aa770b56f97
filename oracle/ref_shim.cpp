// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (see ref_shim.h).
//
// Thin extern "C" adapter that builds the reference's own objects (Grid,
// ScalarField, IntervalField, DynamicsModel subclasses, SolveConfig) and
// calls the reference's own functions.  No reference source is copied here;
// the reference .cpp files are compiled in place by oracle/Makefile.

#include "ref_shim.h"

#include <cmath>
#include <cstring>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hjsafe/decomposition.hpp"
#include "hjsafe/dynamics.hpp"
#include "hjsafe/grid.hpp"
#include "hjsafe/hjvf.hpp"
#include "hjsafe/interval_field.hpp"
#include "hjsafe/levelset.hpp"
#include "hjsafe/safety.hpp"
#include "hjsafe/solver.hpp"

using namespace hjsafe;

namespace {

// BASELINE.json 4D lateral model: identical to NearHoverPlanar4D except the
// wind enters the position row (dx = vx + d).  Harness-side subclass, the
// plug-in pattern of proj/tests/test_solver.cpp:14-29.
class BaselinePlanar4D final : public DynamicsModel {
 public:
  explicit BaselinePlanar4D(NearHoverPlanar4D::Params p) : p_(p) {}
  std::size_t state_dim() const override { return 4; }
  std::size_t control_dim() const override { return 1; }
  std::size_t disturbance_dim() const override { return 1; }
  std::string name() const override { return "baseline_planar4d"; }
  std::vector<Interval> control_bounds() const override {
    return {{-p_.max_angle_cmd, p_.max_angle_cmd}};
  }
  void affine(std::span<const double> x, AffineFlow& out) const override {
    out.reset(4, 1, 1);
    const double theta = x[2];
    out.drift[0] = x[1];
    out.drift[1] = p_.gravity * std::tan(theta);
    out.drift[2] = -p_.d1 * theta + x[3];
    out.drift[3] = -p_.d0 * theta;
    out.control[3][0] = p_.n0;
    out.disturbance[0][0] = 1.0;
  }

 private:
  NearHoverPlanar4D::Params p_;
};

// drift-only model of the reference solver tests (test_solver.cpp:14-29)
class ConstantAdvection final : public DynamicsModel {
 public:
  explicit ConstantAdvection(std::vector<double> speed) : speed_(std::move(speed)) {}
  std::size_t state_dim() const override { return speed_.size(); }
  std::size_t control_dim() const override { return 0; }
  std::size_t disturbance_dim() const override { return 0; }
  std::string name() const override { return "advection"; }
  std::vector<Interval> control_bounds() const override { return {}; }
  void affine(std::span<const double>, AffineFlow& out) const override {
    out.reset(speed_.size(), 0, 0);
    for (std::size_t i = 0; i < speed_.size(); ++i) out.drift[i] = speed_[i];
  }

 private:
  std::vector<double> speed_;
};

std::unique_ptr<DynamicsModel> make(const hjr_model_spec* s) {
  switch (s->kind) {
    case HJR_QUAD2D_VERT: {
      Quad2DVert::Params p;
      p.k_thrust = s->p[0];
      p.k_offset = s->p[1];
      p.gravity = s->p[2];
      return std::make_unique<Quad2DVert>(p);
    }
    case HJR_PLANAR4D: {
      NearHoverPlanar4D::Params p;
      p.d0 = s->p[0];
      p.d1 = s->p[1];
      p.n0 = s->p[2];
      p.gravity = s->p[3];
      p.max_angle_cmd = s->p[4];
      if (s->d_row == 1) return std::make_unique<NearHoverPlanar4D>("x", p);
      if (s->d_row == 0) return std::make_unique<BaselinePlanar4D>(p);
      throw std::invalid_argument("ref_shim: planar4d d_row must be 0 or 1");
    }
    case HJR_VERTICAL2D: {
      NearHoverVertical2D::Params p;
      p.gravity = s->p[0];
      p.thrust_gain = s->p[1];
      p.thrust_frac_lo = s->p[2];
      p.thrust_frac_hi = s->p[3];
      return std::make_unique<NearHoverVertical2D>(p);
    }
    case HJR_DOUBLE_INT: {
      DoubleIntegrator::Params p;
      p.a_min = s->p[0];
      p.a_max = s->p[1];
      return std::make_unique<DoubleIntegrator>(p);
    }
    case HJR_TWIN_DI: {
      DoubleIntegrator::Params p;
      p.a_min = s->p[0];
      p.a_max = s->p[1];
      return std::make_unique<TwinDoubleIntegrator>(p);
    }
    case HJR_ADVECTION: {
      std::vector<double> sp(s->p, s->p + s->d_row);
      return std::make_unique<ConstantAdvection>(sp);
    }
    case HJR_NEAR_HOVER_10D: {
      NearHoverPlanar4D::Params pp;
      pp.d0 = s->p[0];
      pp.d1 = s->p[1];
      pp.n0 = s->p[2];
      pp.gravity = s->p[3];
      pp.max_angle_cmd = s->p[4];
      NearHoverVertical2D::Params vp;
      vp.gravity = s->p[5];
      vp.thrust_gain = s->p[6];
      vp.thrust_frac_lo = s->p[7];
      vp.thrust_frac_hi = s->p[8];
      return std::make_unique<NearHover10D>(pp, vp);
    }
  }
  throw std::invalid_argument("ref_shim: unknown model kind");
}

Grid make_grid(const hjb_grid* g) {
  std::vector<GridDim> dims;
  for (int d = 0; d < g->ndims; ++d)
    dims.push_back({g->dims[d].min, g->dims[d].max, static_cast<std::size_t>(g->dims[d].n)});
  return Grid(std::move(dims));
}

ScalarField make_field(const Grid& g, const double* v) {
  return ScalarField(g, std::vector<double>(v, v + g.size()));
}

IntervalField make_db(const Grid& g, const hjb_dbounds* db) {
  if (!db->per_node) {
    std::vector<Interval> b;
    for (int c = 0; c < db->channels; ++c) b.push_back({db->constant[c].lo, db->constant[c].hi});
    return IntervalField::constant(g, b);
  }
  IntervalField f(g, db->channels);
  for (int c = 0; c < db->channels; ++c) {
    f.lo(c) = make_field(g, db->lo[c]);
    f.hi(c) = make_field(g, db->hi[c]);
  }
  return f;
}

SolveConfig make_cfg(const hjb_solve_config* c) {
  if (c->target)  // the reference clamps against the avoid set only
    throw std::invalid_argument("ref_shim: the reference has no target set");
  SolveConfig cfg;
  cfg.cfl_factor = c->cfl_factor;
  cfg.tolerance = c->tolerance;
  cfg.max_iters = static_cast<std::size_t>(c->max_iters);
  cfg.scheme = c->scheme == 1 ? SolveConfig::Scheme::kLaxFriedrichs
                              : SolveConfig::Scheme::kGodunov;
  cfg.dissipation = c->dissipation == 1 ? SolveConfig::Dissipation::kGlobal
                                        : SolveConfig::Dissipation::kPerNode;
  cfg.threads = static_cast<unsigned>(c->threads);
  return cfg;
}

void fill_result(const SolveResult& r, hjr_result* out) {
  if (!out) return;
  out->iterations = static_cast<int64_t>(r.iterations);
  out->dt = r.dt;
  out->wall_seconds = r.wall_seconds;
  out->converged = r.converged ? 1 : 0;
  out->nodes_per_sweep = static_cast<int64_t>(r.nodes_per_sweep);
  if (out->residual_history) {
    const std::size_t n =
        std::min<std::size_t>(r.residual_history.size(), out->history_capacity);
    std::memcpy(out->residual_history, r.residual_history.data(), n * sizeof(double));
  }
  if (out->wall_ms_history) {
    const std::size_t n =
        std::min<std::size_t>(r.wall_ms_history.size(), out->history_capacity);
    std::memcpy(out->wall_ms_history, r.wall_ms_history.data(), n * sizeof(double));
  }
}

template <typename Fn>
int guarded(char* err, int errlen, Fn&& fn) {
  auto put = [&](const char* msg) {
    if (err && errlen > 0) {
      std::strncpy(err, msg, errlen - 1);
      err[errlen - 1] = 0;
    }
  };
  try {
    fn();
    put("");
    return 0;
  } catch (const std::invalid_argument& e) {
    put(e.what());
    return 1;
  } catch (const std::runtime_error& e) {
    put(e.what());
    return 2;
  } catch (const std::exception& e) {
    put(e.what());
    return 3;
  }
}

}  // namespace

extern "C" {

int hjr_cfl_dt(const hjb_grid* g, const hjr_model_spec* m, const hjb_dbounds* db, double cfl,
               unsigned threads, double* dt, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Grid grid = make_grid(g);
    auto model = make(m);
    *dt = cfl_dt(grid, *model, make_db(grid, db), cfl, threads);
  });
}

int hjr_vi_step(const hjb_grid* g, const hjr_model_spec* m, const hjb_dbounds* db,
                const double* v, const double* c, double dt, const hjb_solve_config* cfg,
                double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Grid grid = make_grid(g);
    auto model = make(m);
    ScalarField r = vi_step(make_field(grid, v), make_field(grid, c), *model, make_db(grid, db),
                            dt, make_cfg(cfg));
    std::memcpy(out, r.values().data(), grid.size() * sizeof(double));
  });
}

int hjr_solve(const hjb_grid* g, const hjr_model_spec* m, const hjb_dbounds* db,
              const double* init, const double* c, const hjb_solve_config* cfg, double* out,
              hjr_result* res, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Grid grid = make_grid(g);
    auto model = make(m);
    SolveResult r = solve(make_field(grid, init), make_field(grid, c), *model,
                          make_db(grid, db), make_cfg(cfg));
    std::memcpy(out, r.value.values().data(), grid.size() * sizeof(double));
    fill_result(r, res);
  });
}

int hjr_solve_coarse_to_fine(const hjb_grid* fine, const hjr_model_spec* m,
                             const hjb_dbounds* db_fine, const double* c_fine,
                             const hjb_grid* coarse, const hjb_solve_config* cfg,
                             const double* warm_init_fine, double* coarse_out,
                             hjr_result* coarse_res, double* fine_out, hjr_result* fine_res,
                             char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Grid fg = make_grid(fine);
    Grid cg = make_grid(coarse);
    auto model = make(m);
    ScalarField warm;
    if (warm_init_fine) warm = make_field(fg, warm_init_fine);
    CoarseToFineResult r =
        solve_coarse_to_fine(make_field(fg, c_fine), *model, make_db(fg, db_fine), cg,
                             make_cfg(cfg), warm_init_fine ? &warm : nullptr);
    std::memcpy(coarse_out, r.coarse.value.values().data(), cg.size() * sizeof(double));
    std::memcpy(fine_out, r.fine.value.values().data(), fg.size() * sizeof(double));
    fill_result(r.coarse, coarse_res);
    fill_result(r.fine, fine_res);
  });
}

int hjr_solve_coarse_to_fine_w(const hjb_grid* fine, const hjr_model_spec* m,
                               const hjb_dbounds* db_fine, const double* c_fine,
                               const hjb_grid* coarse, const hjb_solve_config* cfg,
                               const hjb_grid* warm_grid, const double* warm, double* coarse_out,
                               hjr_result* coarse_res, double* fine_out, hjr_result* fine_res,
                               char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Grid fg = make_grid(fine);
    Grid cg = make_grid(coarse);
    auto model = make(m);
    ScalarField w;
    if (warm) w = make_field(warm_grid ? make_grid(warm_grid) : fg, warm);
    CoarseToFineResult r =
        solve_coarse_to_fine(make_field(fg, c_fine), *model, make_db(fg, db_fine), cg,
                             make_cfg(cfg), warm ? &w : nullptr);
    std::memcpy(coarse_out, r.coarse.value.values().data(), cg.size() * sizeof(double));
    std::memcpy(fine_out, r.fine.value.values().data(), fg.size() * sizeof(double));
    fill_result(r.coarse, coarse_res);
    fill_result(r.fine, fine_res);
  });
}

int hjr_resample(const hjb_grid* src_g, const double* src, const hjb_grid* dst_g, double* dst,
                 char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Grid sg = make_grid(src_g);
    Grid dg = make_grid(dst_g);
    ScalarField r = resample(make_field(sg, src), dg);
    std::memcpy(dst, r.values().data(), dg.size() * sizeof(double));
  });
}

int hjr_max_adjacent_jump(const hjb_grid* g, const double* v, double* out, char* err,
                          int errlen) {
  return guarded(err, errlen, [&] {
    Grid grid = make_grid(g);
    *out = max_adjacent_jump(make_field(grid, v));
  });
}

int hjr_field_max(const hjb_grid* g, const double* a, const double* b, double* out, char* err,
                  int errlen) {
  return guarded(err, errlen, [&] {
    Grid grid = make_grid(g);
    ScalarField r = field_max(make_field(grid, a), make_field(grid, b));
    std::memcpy(out, r.values().data(), grid.size() * sizeof(double));
  });
}

int hjr_field_min(const hjb_grid* g, const double* a, const double* b, double* out, char* err,
                  int errlen) {
  return guarded(err, errlen, [&] {
    Grid grid = make_grid(g);
    ScalarField r = field_min(make_field(grid, a), make_field(grid, b));
    std::memcpy(out, r.values().data(), grid.size() * sizeof(double));
  });
}

int hjr_signed_distance_band(const hjb_grid* g, int32_t dim, double lo, double hi, double* out,
                             char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Grid grid = make_grid(g);
    ScalarField r = signed_distance_band(grid, static_cast<std::size_t>(dim), lo, hi);
    std::memcpy(out, r.values().data(), grid.size() * sizeof(double));
  });
}

int hjr_signed_distance_box(const hjb_grid* g, const double* lo, const double* hi, double* out,
                            char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Grid grid = make_grid(g);
    std::vector<double> l(lo, lo + g->ndims), h(hi, hi + g->ndims);
    ScalarField r = signed_distance_box(grid, l, h);
    std::memcpy(out, r.values().data(), grid.size() * sizeof(double));
  });
}

int hjr_hamiltonian(const hjr_model_spec* m, const double* x, const double* p,
                    const hjb_interval* db, double* h, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    auto model = make(m);
    const std::size_t n = model->state_dim();
    std::vector<Interval> b;
    for (std::size_t k = 0; k < model->disturbance_dim(); ++k) b.push_back({db[k].lo, db[k].hi});
    *h = hamiltonian(*model, std::span<const double>(x, n), std::span<const double>(p, n), b);
  });
}

int hjr_flow_bounds(const hjr_model_spec* m, const double* x, const hjb_interval* db,
                    double* alpha, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    auto model = make(m);
    const std::size_t n = model->state_dim();
    std::vector<Interval> b;
    for (std::size_t k = 0; k < model->disturbance_dim(); ++k) b.push_back({db[k].lo, db[k].hi});
    auto a = flow_bounds(*model, std::span<const double>(x, n), b);
    for (std::size_t i = 0; i < n; ++i) alpha[i] = a[i];
  });
}

int hjr_affine(const hjr_model_spec* m, const double* x, double* drift, double* control,
               double* disturbance, hjb_interval* ubounds, int32_t* dims, char* err,
               int errlen) {
  return guarded(err, errlen, [&] {
    auto model = make(m);
    AffineFlow af;
    model->affine(std::span<const double>(x, model->state_dim()), af);
    dims[0] = static_cast<int32_t>(af.state_dim);
    dims[1] = static_cast<int32_t>(af.control_dim);
    dims[2] = static_cast<int32_t>(af.disturbance_dim);
    for (std::size_t i = 0; i < kMaxStateDim; ++i) {
      drift[i] = af.drift[i];
      for (std::size_t j = 0; j < kMaxInputDim; ++j) {
        control[i * kMaxInputDim + j] = af.control[i][j];
        disturbance[i * kMaxInputDim + j] = af.disturbance[i][j];
      }
    }
    auto ub = model->control_bounds();
    for (std::size_t j = 0; j < ub.size(); ++j) ubounds[j] = {ub[j].lo, ub[j].hi};
  });
}

int hjr_filter_batch(const hjb_grid* g, const hjr_model_spec* m, const hjb_dbounds* db,
                     const double* value, int64_t nq, const double* x, const double* u_perf,
                     int32_t mode, double eta_floor, int64_t nviol, const double* viol_x,
                     double* lambda_out, int32_t* emergency_out, const hjb_filter_out* out,
                     char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Grid grid = make_grid(g);
    std::shared_ptr<const DynamicsModel> model(make(m).release());
    SolveResult solved{make_field(grid, value)};
    solved.converged = true;
    SafetyFilter::Config cfg;
    cfg.eta_floor = eta_floor;
    SafetyFilter filter(model, solved, make_db(grid, db), cfg);
    const std::size_t nd = grid.ndims();
    if (nviol > 0) {
      std::vector<Violation> vs;
      for (int64_t i = 0; i < nviol; ++i) {
        Violation v;
        v.x.assign(viol_x + i * nd, viol_x + (i + 1) * nd);
        vs.push_back(std::move(v));
      }
      filter.contract(vs);
    }
    if (lambda_out) *lambda_out = filter.lambda();
    if (emergency_out) *emergency_out = filter.emergency() ? 1 : 0;
    const std::size_t nu = model->control_dim(), np = model->disturbance_dim();
    for (int64_t q = 0; q < nq; ++q) {
      std::span<const double> xq(x + q * nd, nd);
      const FilterDecision d =
          mode == HJB_FILTER_FILTER
              ? filter.filter(xq, std::span<const double>(u_perf + q * nu, nu))
              : filter.optimal_control(xq);
      if (out->value) out->value[q] = d.value;
      if (out->band) out->band[q] = d.band;
      if (out->control)
        for (std::size_t j = 0; j < nu; ++j) out->control[q * nu + j] = d.control[j];
      if (out->worst_disturbance)
        for (std::size_t k = 0; k < np; ++k)
          out->worst_disturbance[q * np + k] =
              k < d.worst_disturbance.size() ? d.worst_disturbance[k] : 0.0;
      if (out->flags)
        out->flags[q] = static_cast<uint8_t>((d.override_active ? HJB_FILTER_OVERRIDE : 0) |
                                             (d.degenerate ? HJB_FILTER_DEGENERATE : 0) |
                                             (d.out_of_domain ? HJB_FILTER_OOD : 0));
    }
  });
}

int hjr_decomposition_batch(int32_t nsub, const hjb_grid* grids, const hjr_model_spec* models,
                            const hjb_dbounds* dbs, const double* const* values,
                            const int32_t* maps, int32_t full_n, int32_t full_m, int32_t full_p,
                            double eta_floor, int64_t nviol, const double* viol_x, int64_t nq,
                            const double* x, const double* u_perf, double* lambda_out,
                            int32_t* emergency_out, double* cv_out, double* value_out,
                            double* band_out, double* control_out, uint8_t* flags_out, char* err,
                            int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Subsystem> subs;
    std::vector<std::shared_ptr<SafetyFilter>> filters;
    const int32_t* mp = maps;
    for (int32_t i = 0; i < nsub; ++i) {
      std::shared_ptr<const DynamicsModel> model(make(&models[i]).release());
      Subsystem s;
      s.name = model->name();
      s.model = model;
      s.state_map.assign(mp, mp + model->state_dim());
      mp += model->state_dim();
      s.control_map.assign(mp, mp + model->control_dim());
      mp += model->control_dim();
      s.disturbance_map.assign(mp, mp + model->disturbance_dim());
      mp += model->disturbance_dim();
      Grid grid = make_grid(&grids[i]);
      SolveResult solved{make_field(grid, values[i])};
      solved.converged = true;
      SafetyFilter::Config cfg;
      cfg.eta_floor = eta_floor;
      filters.push_back(std::make_shared<SafetyFilter>(model, solved, make_db(grid, &dbs[i]), cfg));
      subs.push_back(std::move(s));
    }
    Decomposition dec(std::move(subs), full_n, full_m, full_p);
    dec.attach(filters);
    if (nviol > 0) {
      std::vector<Violation> vs;
      for (int64_t i = 0; i < nviol; ++i) {
        Violation v;
        v.x.assign(viol_x + i * full_n, viol_x + (i + 1) * full_n);
        vs.push_back(std::move(v));
      }
      dec.contract(vs);
    }
    if (lambda_out) *lambda_out = dec.lambda();
    if (emergency_out) *emergency_out = dec.emergency() ? 1 : 0;
    for (int64_t q = 0; q < nq; ++q) {
      std::span<const double> xq(x + q * full_n, full_n);
      if (cv_out) cv_out[q] = dec.combined_value(xq);
      const CombinedDecision d =
          dec.combined_control(xq, std::span<const double>(u_perf + q * full_m, full_m));
      if (value_out) value_out[q] = d.value;
      if (band_out) band_out[q] = d.band;
      if (control_out)
        for (int32_t j = 0; j < full_m; ++j) control_out[q * full_m + j] = d.control[j];
      if (flags_out)
        flags_out[q] = static_cast<uint8_t>((d.override_active ? HJB_FILTER_OVERRIDE : 0) |
                                            (d.out_of_domain ? HJB_FILTER_OOD : 0));
    }
  });
}

int hjr_write_hjvf(const char* path, const hjb_grid* g, const double* v, char* err,
                   int errlen) {
  return guarded(err, errlen, [&] {
    Grid grid = make_grid(g);
    write_hjvf(std::filesystem::path(path), make_field(grid, v));
  });
}

}  // extern "C"
