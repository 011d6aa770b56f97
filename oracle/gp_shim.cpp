// gp_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" access to the reference's own GP prediction path: the
// reference's gp.cpp, grid.cpp and interval_field.cpp are compiled in place
// by oracle/Makefile (target `ref`, -> oracle/_ref/libhjref_gp.so) against
// oracle/eigen_stub (gp.cpp's fit needs Eigen, absent from this image).
// Only Eigen-free functions are called: GpHyperparams::validate,
// GpModel::prior / kernel / predict and bounds_on_grid
// (proj/src/gp.cpp:14-38,188-249).  A fitted model's state (training
// inputs, alpha, the Cholesky factor) is written into the reference's
// GpModel directly -- it has no public constructor for it; fit is the only
// producer -- so any factor (the product's hjb_gp_fit, a hand-made one) can
// be pushed through the reference's own predict/bounds_on_grid loops.

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hjsafe/grid.hpp"
#include "hjsafe/interval_field.hpp"
#define private public  // GpModel's state is private and written only by fit
#include "hjsafe/gp.hpp"
#undef private

#include "../include/hjb.h"

using namespace hjsafe;

namespace {

Grid make_grid(const hjb_grid* g) {
  std::vector<GridDim> dims;
  for (int d = 0; d < g->ndims; ++d)
    dims.push_back({g->dims[d].min, g->dims[d].max, static_cast<std::size_t>(g->dims[d].n)});
  return Grid(std::move(dims));
}

GpModel make_model(const hjb_gp_model* c) {
  if (c->input_dim < 1 || c->input_dim > HJB_MAX_DIMS || c->n_train < 0)
    throw std::invalid_argument("gp_shim: bad model descriptor");
  const auto dim = static_cast<std::size_t>(c->input_dim);
  GpHyperparams hp;
  hp.signal_var = c->signal_var;
  hp.noise_var = c->noise_var;
  hp.lengthscales.assign(c->lengthscales, c->lengthscales + dim);
  if (c->n_train == 0) return GpModel::prior(std::move(hp));  // gp.cpp:32-38
  hp.validate(dim);
  GpModel m;
  const auto n = static_cast<std::size_t>(c->n_train);
  m.hp_ = std::move(hp);
  m.input_dim_ = dim;
  m.inputs_.resize(n);
  for (std::size_t i = 0; i < n; ++i) m.inputs_[i].assign(c->inputs + i * dim, c->inputs + (i + 1) * dim);
  m.alpha_.assign(c->alpha, c->alpha + n);
  m.chol_.assign(c->chol, c->chol + n * n);
  return m;
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
  } catch (const std::exception& e) {
    put(e.what());
    return 3;
  }
}

}  // namespace

extern "C" {

// GpModel::predict (gp.cpp:188-208) at nq points of input_dim coordinates.
int hjr_gp_predict(const hjb_gp_model* model, int64_t nq, const double* x, double* mean,
                   double* variance, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const GpModel m = make_model(model);
    const auto dim = static_cast<std::size_t>(model->input_dim);
    for (int64_t q = 0; q < nq; ++q) {
      const auto p = m.predict(std::span<const double>(x + q * dim, dim));
      mean[q] = p.mean;
      variance[q] = p.variance;
    }
  });
}

// bounds_on_grid (gp.cpp:211-249): lo[ch] / hi[ch] hold grid.size doubles.
int hjr_gp_bounds_on_grid(const hjb_grid* g, int32_t channels, const hjb_gp_model* models,
                          double confidence, uint32_t threads, double* const* lo,
                          double* const* hi, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const Grid grid = make_grid(g);
    std::vector<GpModel> ms;
    std::vector<std::vector<std::size_t>> dims;
    for (int32_t ch = 0; ch < channels; ++ch) {
      ms.push_back(make_model(&models[ch]));
      dims.emplace_back(models[ch].input_dims, models[ch].input_dims + models[ch].n_dims);
    }
    const IntervalField f = bounds_on_grid(ms, dims, grid, confidence, threads);
    for (int32_t ch = 0; ch < channels; ++ch) {
      std::memcpy(lo[ch], f.lo(ch).values().data(), grid.size() * sizeof(double));
      std::memcpy(hi[ch], f.hi(ch).values().data(), grid.size() * sizeof(double));
    }
  });
}

}  // extern "C"
