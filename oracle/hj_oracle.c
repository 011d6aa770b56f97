/*
 * hj_oracle.c — TEST INFRASTRUCTURE ONLY (see hj_oracle.h).
 *
 * Plain-C restatement of the reference solver hot path.  Arithmetic follows
 * the reference expression by expression (same operand order, same
 * ternaries, the zero-coefficient accumulations of dim_slopes/flow_bounds/
 * hamiltonian kept), so that built with -ffp-contract=off it is bitwise equal
 * to the reference compiled the same way.  OpenMP only splits the node loop;
 * every reduction is a max, so results do not depend on the thread count
 * (reference parallel.hpp:16-21 determinism contract).
 */
#include "hj_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static __thread char g_err[256];
static int g_threads = 0;

const char* hjo_last_error(void) { return g_err; }
void hjo_set_threads(int threads) { g_threads = threads; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* std::max / std::min as libstdc++ defines them (a<b ? b : a, b<a ? b : a) */
#define STD_MAX(a, b) ((a) < (b) ? (b) : (a))
#define STD_MIN(a, b) ((b) < (a) ? (b) : (a))

/* ------------------------------------------------------------------ grid */
typedef struct {
  int nd;
  int64_t n[HJB_MAX_DIMS];
  double min[HJB_MAX_DIMS], max[HJB_MAX_DIMS], spacing[HJB_MAX_DIMS];
  int64_t stride[HJB_MAX_DIMS];
  int64_t size;
} grid_t;

/* Grid::Grid, grid.cpp:10-31 */
static int grid_init(const hjb_grid* g, grid_t* o) {
  if (g->ndims < 1) return fail(HJB_ERR_INVALID_ARGUMENT, "Grid: ndims must be >= 1");
  if (g->ndims > HJB_MAX_DIMS) return fail(HJB_ERR_UNSUPPORTED, "Grid: too many dims");
  o->nd = g->ndims;
  o->size = 1;
  for (int i = 0; i < o->nd; ++i) {
    const hjb_grid_dim* d = &g->dims[i];
    if (!(d->min < d->max)) return fail(HJB_ERR_INVALID_ARGUMENT, "Grid: min must be < max");
    if (d->n < 2) return fail(HJB_ERR_INVALID_ARGUMENT, "Grid: need at least 2 nodes");
    if (!isfinite(d->min) || !isfinite(d->max))
      return fail(HJB_ERR_INVALID_ARGUMENT, "Grid: non-finite bounds");
    o->n[i] = d->n;
    o->min[i] = d->min;
    o->max[i] = d->max;
    o->spacing[i] = (d->max - d->min) / (double)(d->n - 1);
    o->size *= d->n;
  }
  o->stride[o->nd - 1] = 1;
  for (int i = o->nd - 1; i-- > 0;) o->stride[i] = o->stride[i + 1] * o->n[i + 1];
  return 0;
}

static int grid_same(const hjb_grid* a, const hjb_grid* b) {
  if (a->ndims != b->ndims) return 0;
  for (int i = 0; i < a->ndims; ++i)
    if (a->dims[i].min != b->dims[i].min || a->dims[i].max != b->dims[i].max ||
        a->dims[i].n != b->dims[i].n)
      return 0;
  return 1;
}

/* Grid::coord, grid.cpp:33-38 */
static inline double coord(const grid_t* g, int d, int64_t k) {
  if (k == g->n[d] - 1) return g->max[d];
  return g->min[d] + (double)k * g->spacing[d];
}

/* Grid::unravel, grid.cpp:52-57 */
static inline void unravel(const grid_t* g, int64_t lin, int64_t* idx) {
  for (int i = 0; i < g->nd; ++i) {
    idx[i] = lin / g->stride[i];
    lin -= idx[i] * g->stride[i];
  }
}

static inline void odometer(const grid_t* g, int64_t* idx) {
  for (int d = g->nd; d-- > 0;) {
    if (++idx[d] < g->n[d]) break;
    idx[d] = 0;
  }
}

/* -------------------------------------------------------------- dynamics */
typedef struct {
  int n, m, p;
  double drift[HJB_MAX_STATE];
  const double (*B)[HJB_MAX_INPUT];
  const double (*C)[HJB_MAX_INPUT];
} affine_t;

static int model_check(const hjb_model* m) {
  if (m->state_dim < 1 || m->state_dim > HJB_MAX_STATE || m->control_dim < 0 ||
      m->control_dim > HJB_MAX_INPUT || m->disturbance_dim < 0 ||
      m->disturbance_dim > HJB_MAX_INPUT)
    return fail(HJB_ERR_INVALID_ARGUMENT, "model: bad dimensions");
  return 0;
}

static inline double term_value(const hjb_drift_term* t, const double* x, const int64_t* idx) {
  switch (t->kind) {
    case HJB_TERM_COORD: return t->scale * x[t->axis];
    case HJB_TERM_TAN: return t->scale * tan(x[t->axis]);
    case HJB_TERM_CONST: return t->scale;
    case HJB_TERM_TABLE: return idx ? t->table[idx[t->axis]] : NAN;
    default: return 0.0;
  }
}

/* Model::affine (dynamics.cpp:126-198 for the stock models): drift terms,
 * AffineFlow::reset zero-fills (dynamics.cpp:9-16) so absent rows are 0.0. */
static inline void model_affine(const hjb_model* m, const double* x, const int64_t* idx,
                                affine_t* af) {
  af->n = m->state_dim;
  af->m = m->control_dim;
  af->p = m->disturbance_dim;
  af->B = m->control;
  af->C = m->disturbance;
  for (int i = 0; i < af->n; ++i) {
    const hjb_drift_term* t = m->drift[i];
    double v = 0.0;
    if (t[0].kind != HJB_TERM_NONE) {
      v = term_value(&t[0], x, idx);
      if (t[1].kind != HJB_TERM_NONE) v = v + term_value(&t[1], x, idx);
    }
    af->drift[i] = v;
  }
}

/* extremal_inputs + hamiltonian, dynamics.cpp:37-83 */
static double hamiltonian(const affine_t* f, const double* p, const hjb_interval* ub,
                          const hjb_interval* db) {
  double u[HJB_MAX_INPUT], d[HJB_MAX_INPUT];
  for (int j = 0; j < f->m; ++j) {
    double coeff = 0.0;
    for (int i = 0; i < f->n; ++i) coeff += p[i] * f->B[i][j];
    u[j] = coeff > 0.0 ? ub[j].lo : (coeff < 0.0 ? ub[j].hi : ub[j].lo);
  }
  for (int k = 0; k < f->p; ++k) {
    double coeff = 0.0;
    for (int i = 0; i < f->n; ++i) coeff += p[i] * f->C[i][k];
    d[k] = coeff > 0.0 ? db[k].hi : (coeff < 0.0 ? db[k].lo : db[k].lo);
  }
  double h = 0.0;
  for (int i = 0; i < f->n; ++i) {
    double fi = f->drift[i];
    for (int j = 0; j < f->m; ++j) fi += f->B[i][j] * u[j];
    for (int k = 0; k < f->p; ++k) fi += f->C[i][k] * d[k];
    h += p[i] * fi;
  }
  return h;
}

/* flow_bounds, dynamics.cpp:93-112 */
static void flow_bounds(const affine_t* f, const hjb_interval* ub, const hjb_interval* db,
                        double* alpha) {
  for (int i = 0; i < f->n; ++i) {
    double lo = f->drift[i];
    double hi = f->drift[i];
    for (int j = 0; j < f->m; ++j) {
      const double a = f->B[i][j] * ub[j].lo;
      const double b = f->B[i][j] * ub[j].hi;
      lo += STD_MIN(a, b);
      hi += STD_MAX(a, b);
    }
    for (int k = 0; k < f->p; ++k) {
      const double a = f->C[i][k] * db[k].lo;
      const double b = f->C[i][k] * db[k].hi;
      lo += STD_MIN(a, b);
      hi += STD_MAX(a, b);
    }
    alpha[i] = STD_MAX(fabs(lo), fabs(hi));
  }
}

/* rows_separable, solver.cpp:88-102 */
static int rows_separable(const affine_t* f) {
  for (int j = 0; j < f->m; ++j) {
    int rows = 0;
    for (int i = 0; i < f->n; ++i)
      if (f->B[i][j] != 0.0) ++rows;
    if (rows > 1) return 0;
  }
  for (int k = 0; k < f->p; ++k) {
    int rows = 0;
    for (int i = 0; i < f->n; ++i)
      if (f->C[i][k] != 0.0) ++rows;
    if (rows > 1) return 0;
  }
  return 1;
}

/* DimSlopes / kink_h / godunov_flux / dim_slopes, solver.cpp:39-86 */
typedef struct {
  double pos, neg;
} slopes_t;

static inline double kink_h(slopes_t s, double p) { return p > 0.0 ? s.pos * p : s.neg * p; }

static inline double godunov_flux(slopes_t s, double dminus, double dplus) {
  const double ha = kink_h(s, dminus);
  const double hb = kink_h(s, dplus);
  if (dminus <= dplus) {
    double h = ha > hb ? ha : hb;
    if (dminus <= 0.0 && 0.0 <= dplus && h < 0.0) h = 0.0;
    return h;
  }
  double h = ha < hb ? ha : hb;
  if (dplus <= 0.0 && 0.0 <= dminus && h > 0.0) h = 0.0;
  return h;
}

static inline void dim_slopes(const affine_t* f, const hjb_interval* ub, const hjb_interval* db,
                              slopes_t* out) {
  for (int d = 0; d < f->n; ++d) {
    double pos = f->drift[d];
    double neg = f->drift[d];
    for (int j = 0; j < f->m; ++j) {
      const double a = f->B[d][j] * ub[j].lo;
      const double b = f->B[d][j] * ub[j].hi;
      pos += a < b ? a : b;
      neg += a > b ? a : b;
    }
    for (int k = 0; k < f->p; ++k) {
      const double a = f->C[d][k] * db[k].lo;
      const double b = f->C[d][k] * db[k].hi;
      pos += a > b ? a : b;
      neg += a < b ? a : b;
    }
    out[d].pos = pos;
    out[d].neg = neg;
  }
}

/* IntervalField::at_node, interval_field.hpp:27-29 */
static inline void db_at(const hjb_dbounds* db, int64_t lin, hjb_interval* out) {
  for (int ch = 0; ch < db->channels; ++ch) {
    if (db->per_node) {
      out[ch].lo = db->lo[ch][lin];
      out[ch].hi = db->hi[ch][lin];
    } else {
      out[ch] = db->constant[ch];
    }
  }
}

static int check_ctx(const hjb_grid* gi, const hjb_model* m, const hjb_dbounds* db, grid_t* g) {
  int rc = grid_init(gi, g);
  if (rc) return rc;
  if ((rc = model_check(m))) return rc;
  /* make_context, solver.cpp:192-199 */
  if (g->nd != m->state_dim)
    return fail(HJB_ERR_INVALID_ARGUMENT, "solver: grid rank does not match model state");
  if (db->channels != m->disturbance_dim)
    return fail(HJB_ERR_INVALID_ARGUMENT, "solver: disturbance channel count mismatch");
  return 0;
}

static int nthreads(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}

#define CHUNK 4096 /* kChunk, solver.cpp:22 */

/* scan_alpha, solver.cpp:221-268 */
static void scan_alpha(const grid_t* g, const hjb_model* m, const hjb_dbounds* db,
                       hjo_scan* out) {
  const int nd = g->nd;
  const int64_t nchunks = (g->size + CHUNK - 1) / CHUNK;
  double best = 0.0;
  double best_alpha[HJB_MAX_STATE] = {0};
  int sep = 1;
  double inv[HJB_MAX_DIMS];
  for (int d = 0; d < nd; ++d) inv[d] = 1.0 / g->spacing[d];
#pragma omp parallel num_threads(nthreads())
  {
    double lbest = 0.0, lalpha[HJB_MAX_STATE] = {0};
    int lsep = 1;
#pragma omp for schedule(dynamic, 1)
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int64_t lo = ch * CHUNK;
      const int64_t hi = lo + CHUNK < g->size ? lo + CHUNK : g->size;
      int64_t idx[HJB_MAX_DIMS];
      double x[HJB_MAX_STATE], alpha[HJB_MAX_STATE];
      hjb_interval dbn[HJB_MAX_INPUT];
      affine_t af;
      unravel(g, lo, idx);
      for (int64_t lin = lo; lin < hi; ++lin) {
        for (int d = 0; d < nd; ++d) x[d] = coord(g, d, idx[d]);
        db_at(db, lin, dbn);
        model_affine(m, x, idx, &af);
        if (!rows_separable(&af)) lsep = 0;
        flow_bounds(&af, m->ubounds, dbn, alpha);
        double speed = 0.0;
        for (int d = 0; d < nd; ++d) {
          speed += alpha[d] * inv[d];
          lalpha[d] = STD_MAX(lalpha[d], alpha[d]);
        }
        lbest = STD_MAX(lbest, speed);
        odometer(g, idx);
      }
    }
#pragma omp critical
    {
      best = STD_MAX(best, lbest);
      for (int d = 0; d < nd; ++d) best_alpha[d] = STD_MAX(best_alpha[d], lalpha[d]);
      if (!lsep) sep = 0;
    }
  }
  out->max_speed_sum = best;
  for (int d = 0; d < HJB_MAX_STATE; ++d) out->max_alpha[d] = d < nd ? best_alpha[d] : 0.0;
  out->separable = sep;
}

int hjo_scan_alpha(const hjb_grid* gi, const hjb_model* m, const hjb_dbounds* db, hjo_scan* out) {
  grid_t g;
  int rc = check_ctx(gi, m, db, &g);
  if (rc) return rc;
  scan_alpha(&g, m, db, out);
  return 0;
}

/* cfl_dt, solver.cpp:272-282 */
int hjo_cfl_dt(const hjb_grid* gi, const hjb_model* m, const hjb_dbounds* db, double cfl,
               double* dt) {
  if (!(cfl > 0.0) || cfl > 1.0)
    return fail(HJB_ERR_INVALID_ARGUMENT, "SolveConfig: cfl_factor must be in (0,1]");
  hjo_scan s;
  int rc = hjo_scan_alpha(gi, m, db, &s);
  if (rc) return rc;
  if (!(s.max_speed_sum > 0.0))
    return fail(HJB_ERR_RUNTIME, "cfl_dt: flow is identically zero on the grid");
  *dt = cfl / s.max_speed_sum;
  return 0;
}

/* update_chunk, solver.cpp:106-190 */
static double update_range(const grid_t* g, const hjb_model* m, const hjb_dbounds* db,
                           const double* inv, int godunov, const double* global_alpha,
                           const double* v, const double* c, const double* tg, double* out,
                           double dt, int64_t lo, int64_t hi) {
  const int nd = g->nd;
  int64_t idx[HJB_MAX_DIMS];
  double x[HJB_MAX_STATE], dminus[HJB_MAX_STATE], dplus[HJB_MAX_STATE];
  double costate[HJB_MAX_STATE], alpha[HJB_MAX_STATE];
  slopes_t slopes[HJB_MAX_STATE];
  hjb_interval dbn[HJB_MAX_INPUT];
  affine_t af;
  unravel(g, lo, idx);
  double max_dv = 0.0;
  for (int64_t lin = lo; lin < hi; ++lin) {
    for (int d = 0; d < nd; ++d) x[d] = coord(g, d, idx[d]);
    for (int d = 0; d < nd; ++d) {
      const int64_t stride = g->stride[d];
      const int64_t k = idx[d];
      const int64_t n = g->n[d];
      double left, right;
      if (k > 0 && k < n - 1) {
        left = (v[lin] - v[lin - stride]) * inv[d];
        right = (v[lin + stride] - v[lin]) * inv[d];
      } else if (k == 0) {
        right = (v[lin + stride] - v[lin]) * inv[d];
        left = godunov ? 0.0 : right;
      } else {
        left = (v[lin] - v[lin - stride]) * inv[d];
        right = godunov ? 0.0 : left;
      }
      dminus[d] = left;
      dplus[d] = right;
    }
    db_at(db, lin, dbn);
    model_affine(m, x, idx, &af);
    double hhat = 0.0;
    if (godunov) {
      dim_slopes(&af, m->ubounds, dbn, slopes);
      for (int d = 0; d < nd; ++d) hhat += godunov_flux(slopes[d], dminus[d], dplus[d]);
    } else {
      for (int d = 0; d < nd; ++d) costate[d] = 0.5 * (dminus[d] + dplus[d]);
      hhat = hamiltonian(&af, costate, m->ubounds, dbn);
      if (!global_alpha) {
        flow_bounds(&af, m->ubounds, dbn, alpha);
        for (int d = 0; d < nd; ++d) hhat += alpha[d] * 0.5 * (dplus[d] - dminus[d]);
      } else {
        for (int d = 0; d < nd; ++d) hhat += global_alpha[d] * 0.5 * (dplus[d] - dminus[d]);
      }
    }
    double stepped = v[lin] + dt * hhat;
    /* target set (B200 extension, no reference counterpart; parity
     * unpinned): reach-avoid V' = max(c, min(l, V + dt*H)), std::min order */
    if (tg) stepped = tg[lin] < stepped ? tg[lin] : stepped;
    const double vnew = stepped > c[lin] ? stepped : c[lin];
    out[lin] = vnew;
    const double dv = fabs(vnew - v[lin]);
    if (dv > max_dv) max_dv = dv;
    odometer(g, idx);
  }
  return max_dv;
}

static double sweep(const grid_t* g, const hjb_model* m, const hjb_dbounds* db, const double* v,
                    const double* c, const double* tg, double dt, int godunov,
                    const double* global_alpha, double* out) {
  double inv[HJB_MAX_DIMS];
  for (int d = 0; d < g->nd; ++d) inv[d] = 1.0 / g->spacing[d];
  const int64_t nchunks = (g->size + CHUNK - 1) / CHUNK;
  double best = 0.0;
#pragma omp parallel num_threads(nthreads())
  {
    double lbest = 0.0;
#pragma omp for schedule(static)
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int64_t lo = ch * CHUNK;
      const int64_t hi = lo + CHUNK < g->size ? lo + CHUNK : g->size;
      const double r = update_range(g, m, db, inv, godunov, global_alpha, v, c, tg, out, dt, lo, hi);
      lbest = STD_MAX(lbest, r);
    }
#pragma omp critical
    best = STD_MAX(best, lbest);
  }
  return best;
}

int hjo_sweep(const hjb_grid* gi, const hjb_model* m, const hjb_dbounds* db, const double* v,
              const double* c, double dt, int32_t scheme, const double* global_alpha,
              double* out, double* max_dv) {
  grid_t g;
  int rc = check_ctx(gi, m, db, &g);
  if (rc) return rc;
  *max_dv = sweep(&g, m, db, v, c, NULL, dt, scheme == HJB_GODUNOV, global_alpha, out);
  return 0;
}

int hjo_sweep_planes(const hjb_grid* gi, const hjb_model* m, const hjb_dbounds* db,
                     const double* v, const double* c, double dt, int32_t scheme,
                     const double* global_alpha, int64_t pb, int64_t pe, double* out,
                     double* max_dv) {
  grid_t g;
  int rc = check_ctx(gi, m, db, &g);
  if (rc) return rc;
  if (pb < 0 || pe > g.n[0] || pb >= pe)
    return fail(HJB_ERR_INVALID_ARGUMENT, "sweep_planes: bad plane range");
  double inv[HJB_MAX_DIMS];
  for (int d = 0; d < g.nd; ++d) inv[d] = 1.0 / g.spacing[d];
  *max_dv = update_range(&g, m, db, inv, scheme == HJB_GODUNOV, global_alpha, v, c, NULL, out, dt,
                         pb * g.stride[0], pe * g.stride[0]);
  return 0;
}

/* vi_step, solver.cpp:284-308 */
int hjo_vi_step(const hjb_grid* gi, const hjb_model* m, const hjb_dbounds* db, const double* v,
                const double* c, double dt, const hjb_solve_config* cfg, double* out) {
  grid_t g;
  int rc = check_ctx(gi, m, db, &g);
  if (rc) return rc;
  hjo_scan s;
  scan_alpha(&g, m, db, &s);
  if (dt * s.max_speed_sum > 1.0 + 1e-12)
    return fail(HJB_ERR_INVALID_ARGUMENT, "vi_step: dt violates the CFL bound");
  if (cfg->scheme == HJB_GODUNOV && !s.separable)
    return fail(HJB_ERR_INVALID_ARGUMENT,
                "vi_step: model inputs are not row-separable, use the Lax-Friedrichs scheme");
  const double* ga = cfg->dissipation == HJB_GLOBAL ? s.max_alpha : NULL;
  sweep(&g, m, db, v, c, cfg->target, dt, cfg->scheme == HJB_GODUNOV, ga, out);
  return 0;
}

int hjo_ho_solve(const grid_t* g, const hjb_model* m, const hjb_dbounds* db, const double* init,
                 const double* c, const hjb_solve_config* cfg, const hjo_scan* s, double dt,
                 double* out, hjb_solve_result* res);

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* solve, solver.cpp:310-376 */
int hjo_solve(const hjb_grid* gi, const hjb_model* m, const hjb_dbounds* db, const double* init,
              const double* c, const hjb_solve_config* cfg, double* out, hjb_solve_result* res) {
  if (!(cfg->cfl_factor > 0.0) || cfg->cfl_factor > 1.0)
    return fail(HJB_ERR_INVALID_ARGUMENT, "SolveConfig: cfl_factor must be in (0,1]");
  if (!(cfg->tolerance > 0.0))
    return fail(HJB_ERR_INVALID_ARGUMENT, "SolveConfig: tolerance must be > 0");
  grid_t g;
  int rc = check_ctx(gi, m, db, &g);
  if (rc) return rc;
  hjo_scan s;
  scan_alpha(&g, m, db, &s);
  if (!(s.max_speed_sum > 0.0))
    return fail(HJB_ERR_RUNTIME, "solve: flow is identically zero on the grid");
  if (cfg->scheme == HJB_GODUNOV && !s.separable)
    return fail(HJB_ERR_INVALID_ARGUMENT,
                "solve: model inputs are not row-separable, use the Lax-Friedrichs scheme");
  const double dt = cfg->cfl_factor / s.max_speed_sum;
  res->dt = dt;
  res->nodes_per_sweep = g.size;
  res->converged = 0;
  res->iterations = 0;
  if (cfg->spatial_order > 1 || cfg->time_order > 1 || (cfg->flags & HJB_FLAG_FORCE_HO))
    return hjo_ho_solve(&g, m, db, init, c, cfg, &s, dt, out, res);
  const double* ga = cfg->dissipation == HJB_GLOBAL ? s.max_alpha : NULL;
  const int godunov = cfg->scheme == HJB_GODUNOV;

  const double t0 = now_ms();
  double* front = (double*)malloc(g.size * sizeof(double));
  double* back = (double*)malloc(g.size * sizeof(double));
  memcpy(front, init, g.size * sizeof(double));
  double min_residual = INFINITY, first = 0.0, residual = 0.0;
  int status = 0;
  for (int64_t iter = 1; iter <= cfg->max_iters; ++iter) {
    const double max_dv = sweep(&g, m, db, front, c, cfg->target, dt, godunov, ga, back);
    residual = max_dv / dt;
    double* t = front;
    front = back;
    back = t;
    res->iterations = iter;
    if (iter == 1) first = residual;
    if (res->residual_history && iter <= res->history_capacity)
      res->residual_history[iter - 1] = residual;
    if (res->wall_ms_history && iter <= res->history_capacity)
      res->wall_ms_history[iter - 1] = now_ms() - t0;
    if (residual < cfg->tolerance) {
      res->converged = 1;
      break;
    }
    min_residual = STD_MIN(min_residual, residual);
    if (!isfinite(residual) || residual > 10.0 * STD_MAX(min_residual, first)) {
      status = fail(HJB_ERR_DIVERGED, "solve: diverging (residual grew 10x above its minimum)");
      break;
    }
    if (cfg->time_horizon > 0.0 && (double)iter * dt >= cfg->time_horizon) break;
  }
  res->final_residual = residual;
  memcpy(out, front, g.size * sizeof(double));
  res->wall_seconds = (now_ms() - t0) * 1e-3;
  free(front);
  free(back);
  return status;
}

/* ------------------------------------------------------ interpolation */
/* locate + interp_ex, grid.cpp:84-135 */
static double interp_at(const grid_t* g, const double* f, const double* x, int* ood) {
  int64_t base[HJB_MAX_DIMS];
  double frac[HJB_MAX_DIMS];
  *ood = 0;
  for (int d = 0; d < g->nd; ++d) {
    double t = (x[d] - g->min[d]) / g->spacing[d];
    if (t < 0.0) {
      t = 0.0;
      *ood = 1;
    }
    const double tmax = (double)(g->n[d] - 1);
    if (t > tmax) {
      t = tmax;
      if (x[d] > g->max[d]) *ood = 1;
    }
    int64_t i0 = (int64_t)t;
    if (i0 > g->n[d] - 2) i0 = g->n[d] - 2;
    base[d] = i0;
    frac[d] = t - (double)i0;
  }
  double value = 0.0;
  const int64_t corners = (int64_t)1 << g->nd;
  for (int64_t corner = 0; corner < corners; ++corner) {
    double w = 1.0;
    int64_t lin = 0;
    for (int d = 0; d < g->nd; ++d) {
      const int hi = (corner >> d) & 1;
      w *= hi ? frac[d] : 1.0 - frac[d];
      lin += (base[d] + (hi ? 1 : 0)) * g->stride[d];
    }
    if (w != 0.0) value += w * f[lin];
  }
  return value;
}

int hjo_interp(const hjb_grid* gi, const double* field, const double* x, double* value,
               int32_t* out_of_domain) {
  grid_t g;
  int rc = grid_init(gi, &g);
  if (rc) return rc;
  for (int d = 0; d < g.nd; ++d)
    if (!isfinite(x[d])) return fail(HJB_ERR_INVALID_ARGUMENT, "interp: non-finite query");
  int ood;
  *value = interp_at(&g, field, x, &ood);
  *out_of_domain = ood;
  return 0;
}

/* ------------------------------------------------ safety-filter queries */
/* locate, grid.cpp:90-111 (base / frac only) */
static void locate_cell(const grid_t* g, const double* x, int64_t* base, double* frac, int* ood) {
  *ood = 0;
  for (int d = 0; d < g->nd; ++d) {
    double t = (x[d] - g->min[d]) / g->spacing[d];
    if (t < 0.0) {
      t = 0.0;
      *ood = 1;
    }
    const double tmax = (double)(g->n[d] - 1);
    if (t > tmax) {
      t = tmax;
      if (x[d] > g->max[d]) *ood = 1;
    }
    int64_t i0 = (int64_t)t;
    if (i0 > g->n[d] - 2) i0 = g->n[d] - 2;
    base[d] = i0;
    frac[d] = t - (double)i0;
  }
}

/* max_cell_jump, grid.cpp:177-195 */
static double max_cell_jump_at(const grid_t* g, const double* f, const int64_t* base) {
  double jump = 0.0;
  const int64_t corners = (int64_t)1 << g->nd;
  for (int64_t corner = 0; corner < corners; ++corner) {
    int64_t lin = 0;
    for (int d = 0; d < g->nd; ++d) lin += (base[d] + ((corner >> d) & 1)) * g->stride[d];
    for (int d = 0; d < g->nd; ++d) {
      if ((corner >> d) & 1) continue;
      const double dv = fabs(f[lin + g->stride[d]] - f[lin]);
      if (dv > jump) jump = dv;
    }
  }
  return jump;
}

/* gradient_at, grid.cpp:141-163 */
static void gradient_at(const grid_t* g, const double* f, int64_t lin, int d, double* left,
                        double* right) {
  const int64_t n = g->n[d];
  const int64_t stride = g->stride[d];
  const int64_t k = (lin / stride) % n;
  const double inv_dx = 1.0 / g->spacing[d];
  if (k > 0 && k < n - 1) {
    *left = (f[lin] - f[lin - stride]) * inv_dx;
    *right = (f[lin + stride] - f[lin]) * inv_dx;
  } else if (k == 0) {
    *right = (f[lin + stride] - f[lin]) * inv_dx;
    *left = *right;
  } else {
    *left = (f[lin] - f[lin - stride]) * inv_dx;
    *right = *left;
  }
}

/* SafetyFilter::optimal_control / filter, safety.cpp:86-127, with
 * interpolated_costate (safety.cpp:14-49), IntervalField::at
 * (interval_field.cpp:29-31) and extremal_inputs (dynamics.cpp:37-63). */
int hjo_filter_batch(const hjb_grid* gi, const hjb_model* m, const hjb_dbounds* db,
                     const double* value, int64_t nq, const double* x, const double* u_perf,
                     const hjb_filter_config* cfg, const hjb_filter_out* out) {
  grid_t g;
  int rc = grid_init(gi, &g);
  if (rc) return rc;
  if (m->state_dim != g.nd)
    return fail(HJB_ERR_INVALID_ARGUMENT, "SafetyFilter: grid rank does not match model");
  if (db->channels != m->disturbance_dim)
    return fail(HJB_ERR_INVALID_ARGUMENT, "filter: disturbance channel count mismatch");
  for (int64_t q = 0; q < nq; ++q)
    for (int d = 0; d < g.nd; ++d)
      if (!isfinite(x[q * g.nd + d])) return fail(HJB_ERR_INVALID_ARGUMENT, "interp: non-finite query");
  const int n = m->state_dim, nu = m->control_dim, np = m->disturbance_dim;
  for (int64_t q = 0; q < nq; ++q) {
    const double* xq = x + q * n;
    int64_t base[HJB_MAX_DIMS];
    double frac[HJB_MAX_DIMS];
    int ood;
    locate_cell(&g, xq, base, frac, &ood);
    const double v = interp_at(&g, value, xq, &ood);
    double band = 0.0;
    if (cfg->mode == HJB_FILTER_FILTER) {
      const double eta = STD_MAX(cfg->eta_floor, 0.5 * max_cell_jump_at(&g, value, base));
      band = eta;
      if (!ood && v <= -cfg->lambda - eta) {
        if (out->value) out->value[q] = v;
        if (out->band) out->band[q] = eta;
        if (out->control)
          for (int j = 0; j < nu; ++j) out->control[q * nu + j] = u_perf[q * nu + j];
        if (out->worst_disturbance)
          for (int k = 0; k < np; ++k) out->worst_disturbance[q * np + k] = 0.0;
        if (out->flags) out->flags[q] = 0;
        continue;
      }
    }
    /* interpolated_costate: std::clamp locate == locate's base/frac */
    double costate[HJB_MAX_STATE] = {0};
    double dlo[HJB_MAX_INPUT] = {0}, dhi[HJB_MAX_INPUT] = {0};
    const int64_t corners = (int64_t)1 << g.nd;
    for (int64_t corner = 0; corner < corners; ++corner) {
      double w = 1.0;
      int64_t lin = 0;
      for (int d = 0; d < g.nd; ++d) {
        const int hi = (corner >> d) & 1;
        w *= hi ? frac[d] : 1.0 - frac[d];
        lin += (base[d] + (hi ? 1 : 0)) * g.stride[d];
      }
      if (w == 0.0) continue;
      for (int d = 0; d < g.nd; ++d) {
        double left, right;
        gradient_at(&g, value, lin, d, &left, &right);
        costate[d] += w * 0.5 * (left + right);
      }
    }
    /* IntervalField::at: interp of each lo / hi field (skips w == 0) */
    for (int k = 0; k < np; ++k) {
      double lo = 0.0, hi = 0.0;
      for (int64_t corner = 0; corner < corners; ++corner) {
        double w = 1.0;
        int64_t lin = 0;
        for (int d = 0; d < g.nd; ++d) {
          const int b = (corner >> d) & 1;
          w *= b ? frac[d] : 1.0 - frac[d];
          lin += (base[d] + (b ? 1 : 0)) * g.stride[d];
        }
        if (w == 0.0) continue;
        lo += w * (db->per_node ? db->lo[k][lin] : db->constant[k].lo);
        hi += w * (db->per_node ? db->hi[k][lin] : db->constant[k].hi);
      }
      dlo[k] = lo;
      dhi[k] = hi;
    }
    /* extremal_inputs */
    int any_active = 0;
    for (int j = 0; j < nu; ++j) {
      double coeff = 0.0;
      for (int i = 0; i < n; ++i) coeff += costate[i] * m->control[i][j];
      const double u = coeff > 0.0 ? m->ubounds[j].lo
                                   : (coeff < 0.0 ? m->ubounds[j].hi : m->ubounds[j].lo);
      if (coeff != 0.0) any_active = 1;
      if (out->control) out->control[q * nu + j] = u;
    }
    for (int k = 0; k < np; ++k) {
      double coeff = 0.0;
      for (int i = 0; i < n; ++i) coeff += costate[i] * m->disturbance[i][k];
      const double dk = coeff > 0.0 ? dhi[k] : (coeff < 0.0 ? dlo[k] : dlo[k]);
      if (coeff != 0.0) any_active = 1;
      if (out->worst_disturbance) out->worst_disturbance[q * np + k] = dk;
    }
    const int degenerate = !any_active && (nu + np) > 0;
    if (out->value) out->value[q] = v;
    if (out->band) out->band[q] = band;
    if (out->flags)
      out->flags[q] = (uint8_t)(HJB_FILTER_OVERRIDE | (degenerate ? HJB_FILTER_DEGENERATE : 0) |
                                (ood ? HJB_FILTER_OOD : 0));
  }
  return 0;
}

/* resample, grid.cpp:215-231 */
int hjo_resample(const hjb_grid* sgi, const double* src, const hjb_grid* dgi, double* dst) {
  grid_t sg, dg;
  int rc = grid_init(sgi, &sg);
  if (rc) return rc;
  if ((rc = grid_init(dgi, &dg))) return rc;
  if (sg.nd != dg.nd) return fail(HJB_ERR_INVALID_ARGUMENT, "resample: dimension mismatch");
  const int64_t nchunks = (dg.size + CHUNK - 1) / CHUNK;
#pragma omp parallel for num_threads(nthreads()) schedule(static)
  for (int64_t ch = 0; ch < nchunks; ++ch) {
    const int64_t lo = ch * CHUNK;
    const int64_t hi = lo + CHUNK < dg.size ? lo + CHUNK : dg.size;
    int64_t idx[HJB_MAX_DIMS];
    double x[HJB_MAX_DIMS];
    unravel(&dg, lo, idx);
    for (int64_t lin = lo; lin < hi; ++lin) {
      for (int d = 0; d < dg.nd; ++d) x[d] = coord(&dg, d, idx[d]);
      int ood;
      dst[lin] = interp_at(&sg, src, x, &ood);
      odometer(&dg, idx);
    }
  }
  return 0;
}

/* max_adjacent_jump, grid.cpp:197-213 */
int hjo_max_adjacent_jump(const hjb_grid* gi, const double* f, double* out) {
  grid_t g;
  int rc = grid_init(gi, &g);
  if (rc) return rc;
  const int64_t nchunks = (g.size + CHUNK - 1) / CHUNK;
  double best = 0.0;
#pragma omp parallel num_threads(nthreads())
  {
    double lbest = 0.0;
#pragma omp for schedule(static)
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int64_t lo = ch * CHUNK;
      const int64_t hi = lo + CHUNK < g.size ? lo + CHUNK : g.size;
      int64_t idx[HJB_MAX_DIMS];
      unravel(&g, lo, idx);
      for (int64_t lin = lo; lin < hi; ++lin) {
        for (int d = 0; d < g.nd; ++d) {
          if (idx[d] + 1 >= g.n[d]) continue;
          const double dv = fabs(f[lin + g.stride[d]] - f[lin]);
          if (dv > lbest) lbest = dv;
        }
        odometer(&g, idx);
      }
    }
#pragma omp critical
    if (lbest > best) best = lbest;
  }
  *out = best;
  return 0;
}

/* seed_from lambda, solver.cpp:404-411 */
int hjo_seed_from(const hjb_grid* sgi, const double* src, const hjb_grid* dgi,
                  const double* c_dst, double* dst) {
  int rc = hjo_resample(sgi, src, dgi, dst);
  if (rc) return rc;
  double slack;
  if ((rc = hjo_max_adjacent_jump(sgi, src, &slack))) return rc;
  grid_t dg;
  grid_init(dgi, &dg);
  for (int64_t i = 0; i < dg.size; ++i) dst[i] = STD_MAX(dst[i] - slack, c_dst[i]);
  return 0;
}

/* solve_coarse_to_fine, solver.cpp:387-425 (constant dbounds: resampling a
 * constant IntervalField reproduces the constant, solver.cpp:378-385, since
 * the multilinear weights of every query sum to one... only when they do
 * exactly; per-node resampling is done explicitly below to stay faithful) */
int hjo_solve_coarse_to_fine(const hjb_grid* fine, const hjb_model* m, const hjb_dbounds* db,
                             const double* c_fine, const hjb_grid* coarse,
                             const hjb_solve_config* cfg, const double* warm_init_fine,
                             double* coarse_out, hjb_solve_result* coarse_res, double* fine_out,
                             hjb_solve_result* fine_res) {
  grid_t fg, cg;
  int rc = grid_init(fine, &fg);
  if (rc) return rc;
  if ((rc = grid_init(coarse, &cg))) return rc;
  if (cg.nd != fg.nd)
    return fail(HJB_ERR_INVALID_ARGUMENT, "solve_coarse_to_fine: grid rank mismatch");
  double* c_coarse = (double*)malloc(cg.size * sizeof(double));
  double* init_coarse = (double*)malloc(cg.size * sizeof(double));
  double* init_fine = (double*)malloc(fg.size * sizeof(double));
  double* dbuf = NULL;
  hjb_dbounds dbc = *db;
  hjo_resample(fine, c_fine, coarse, c_coarse);
  /* resample(IntervalField), solver.cpp:378-385: per channel lo/hi */
  if (db->channels > 0) {
    dbuf = (double*)malloc((size_t)2 * db->channels * fg.size * sizeof(double));
    double* cbuf = (double*)malloc((size_t)2 * db->channels * cg.size * sizeof(double));
    for (int ch = 0; ch < db->channels; ++ch) {
      double* flo = dbuf + (size_t)(2 * ch) * fg.size;
      double* fhi = dbuf + (size_t)(2 * ch + 1) * fg.size;
      for (int64_t i = 0; i < fg.size; ++i) {
        flo[i] = db->per_node ? db->lo[ch][i] : db->constant[ch].lo;
        fhi[i] = db->per_node ? db->hi[ch][i] : db->constant[ch].hi;
      }
      hjo_resample(fine, flo, coarse, cbuf + (size_t)(2 * ch) * cg.size);
      hjo_resample(fine, fhi, coarse, cbuf + (size_t)(2 * ch + 1) * cg.size);
      dbc.lo[ch] = cbuf + (size_t)(2 * ch) * cg.size;
      dbc.hi[ch] = cbuf + (size_t)(2 * ch + 1) * cg.size;
    }
    dbc.per_node = 1;
    free(dbuf);
    dbuf = cbuf;
  }
  if (warm_init_fine)
    hjo_seed_from(fine, warm_init_fine, coarse, c_coarse, init_coarse);
  else
    memcpy(init_coarse, c_coarse, cg.size * sizeof(double));
  rc = hjo_solve(coarse, m, &dbc, init_coarse, c_coarse, cfg, coarse_out, coarse_res);
  if (!rc) {
    hjo_seed_from(coarse, coarse_out, fine, c_fine, init_fine);
    rc = hjo_solve(fine, m, db, init_fine, c_fine, cfg, fine_out, fine_res);
  }
  free(c_coarse);
  free(init_coarse);
  free(init_fine);
  free(dbuf);
  return rc;
}

int hjo_solve_multilevel(int32_t nl, const hjb_grid* grids, const hjb_model* m,
                         const hjb_dbounds* db, const double* c_fine, const hjb_solve_config* cfg,
                         const double* warm, double* const* values_out,
                         hjb_solve_result* results) {
  if (nl < 1 || nl > HJB_MAX_LEVELS)
    return fail(HJB_ERR_INVALID_ARGUMENT, "solve_multilevel: 1..8 levels");
  grid_t g[HJB_MAX_LEVELS];
  int rc;
  for (int l = 0; l < nl; ++l)
    if ((rc = grid_init(&grids[l], &g[l]))) return rc;
  for (int l = 0; l < nl; ++l)
    if (g[l].nd != g[nl - 1].nd)
      return fail(HJB_ERR_INVALID_ARGUMENT, "solve_coarse_to_fine: grid rank mismatch");
  const int F = nl - 1;
  const int64_t nf = g[F].size;
  double* fine_db = NULL;  /* fine-level bounds as fields, for resampling */
  if (db->channels > 0 && nl > 1) {
    fine_db = (double*)malloc((size_t)2 * db->channels * nf * sizeof(double));
    for (int ch = 0; ch < db->channels; ++ch)
      for (int64_t i = 0; i < nf; ++i) {
        fine_db[(2 * ch) * nf + i] = db->per_node ? db->lo[ch][i] : db->constant[ch].lo;
        fine_db[(2 * ch + 1) * nf + i] = db->per_node ? db->hi[ch][i] : db->constant[ch].hi;
      }
  }
  double* own[HJB_MAX_LEVELS] = {0};
  double* cl[HJB_MAX_LEVELS] = {0};
  double* dbl[HJB_MAX_LEVELS] = {0};
  double* init = NULL;
  rc = 0;
  for (int l = 0; l < nl && !rc; ++l) {
    const int64_t n = g[l].size;
    double* out = (values_out && values_out[l]) ? values_out[l]
                                                : (own[l] = (double*)malloc(n * sizeof(double)));
    hjb_dbounds dbx = *db;
    const double* c = c_fine;
    if (l < F) {
      cl[l] = (double*)malloc(n * sizeof(double));
      hjo_resample(&grids[F], c_fine, &grids[l], cl[l]);
      c = cl[l];
      if (db->channels > 0) {
        dbl[l] = (double*)malloc((size_t)2 * db->channels * n * sizeof(double));
        for (int ch = 0; ch < db->channels; ++ch) {
          hjo_resample(&grids[F], fine_db + (2 * ch) * nf, &grids[l], dbl[l] + (2 * ch) * n);
          hjo_resample(&grids[F], fine_db + (2 * ch + 1) * nf, &grids[l], dbl[l] + (2 * ch + 1) * n);
          dbx.lo[ch] = dbl[l] + (2 * ch) * n;
          dbx.hi[ch] = dbl[l] + (2 * ch + 1) * n;
        }
        dbx.per_node = 1;
      }
    }
    free(init);
    init = (double*)malloc(n * sizeof(double));
    if (l == 0) {
      if (warm) hjo_seed_from(&grids[F], warm, &grids[0], c, init);
      else memcpy(init, c, n * sizeof(double));
    } else {
      const double* prev = (values_out && values_out[l - 1]) ? values_out[l - 1] : own[l - 1];
      hjo_seed_from(&grids[l - 1], prev, &grids[l], c, init);
    }
    rc = hjo_solve(&grids[l], m, &dbx, init, c, cfg, out, &results[l]);
  }
  free(init);
  free(fine_db);
  for (int l = 0; l < nl; ++l) {
    free(own[l]);
    free(cl[l]);
    free(dbl[l]);
  }
  return rc;
}

/* ------------------------------------------------------------ level sets */
/* signed_distance_band, levelset.cpp:54-66 */
int hjo_signed_distance_band(const hjb_grid* gi, int32_t dim, double lo, double hi, double* out) {
  grid_t g;
  int rc = grid_init(gi, &g);
  if (rc) return rc;
  if (dim < 0 || dim >= g.nd)
    return fail(HJB_ERR_INVALID_ARGUMENT, "signed_distance_band: dim out of range");
  if (!(lo < hi)) return fail(HJB_ERR_INVALID_ARGUMENT, "signed_distance_band: lo must be < hi");
  for (int64_t lin = 0; lin < g.size; ++lin) {
    const double x = coord(&g, dim, (lin / g.stride[dim]) % g.n[dim]);
    out[lin] = STD_MAX(lo - x, x - hi);
  }
  return 0;
}

/* signed_distance_box_at / signed_distance_box, levelset.cpp:11-52 */
int hjo_signed_distance_box(const hjb_grid* gi, const double* lo, const double* hi, double* out) {
  grid_t g;
  int rc = grid_init(gi, &g);
  if (rc) return rc;
  for (int d = 0; d < g.nd; ++d)
    if (!(lo[d] < hi[d]))
      return fail(HJB_ERR_INVALID_ARGUMENT, "signed_distance_box: lo must be < hi");
  int64_t idx[HJB_MAX_DIMS] = {0};
  for (int64_t lin = 0; lin < g.size; ++lin) {
    double inside = INFINITY, outside_sq = 0.0;
    int outside = 0;
    for (int d = 0; d < g.nd; ++d) {
      const double x = coord(&g, d, idx[d]);
      const double below = lo[d] - x;
      const double above = x - hi[d];
      const double excess = STD_MAX(below, above);
      if (excess > 0.0) {
        outside = 1;
        outside_sq += excess * excess;
      } else {
        inside = STD_MIN(inside, -excess);
      }
    }
    out[lin] = outside ? sqrt(outside_sq) : -inside;
    odometer(&g, idx);
  }
  return 0;
}

/* ------------------------------------------------------------- probes */
int hjo_hamiltonian(const hjb_model* m, const double* x, const double* p, const hjb_interval* db,
                    double* h) {
  int rc = model_check(m);
  if (rc) return rc;
  affine_t af;
  model_affine(m, x, NULL, &af);
  *h = hamiltonian(&af, p, m->ubounds, db);
  return 0;
}

int hjo_flow_bounds(const hjb_model* m, const double* x, const hjb_interval* db, double* alpha) {
  int rc = model_check(m);
  if (rc) return rc;
  affine_t af;
  model_affine(m, x, NULL, &af);
  flow_bounds(&af, m->ubounds, db, alpha);
  return 0;
}

/* ------------------------------------------- high order (no reference) */
/* ENO2/ENO3 spatial derivatives + TVD-RK2/RK3 (Shu-Osher) time stepping.
 * PARITY UNPINNED: the reference has no high-order scheme.
 * Definitions (shared bit for bit with the device kernel k_ho_stage):
 *  a(j) = (V[j+1] - V[j]) * inv_dx              (j = left node of the face)
 *  ghost faces (j < 0 or j > n-2): Godunov 0.0 (the reference's zero ghost
 *    difference, solver.cpp:141-147); LF the nearest interior face (the
 *    reference's replicated one-sided difference)
 *  d2(j) = a(j) - a(j-1);  d3(j) = d2(j+1) - d2(j);  minabs(x,y) = |x|<=|y| ? x : y
 *  ENO1: D- = a(k-1), D+ = a(k)
 *  ENO2: D- = a(k-1) + 0.5*minabs(d2(k-1), d2(k))
 *        D+ = a(k)  + (-0.5)*minabs(d2(k), d2(k+1))
 *  ENO3 (Osher & Fedkiw, Level Set Methods, sec. 3.3, base K = k-1 for D-,
 *        K = k for D+): pick c2 = minabs(d2(K), d2(K+1)) with ks = K-1 when
 *        d2(K) wins else K; c3 = minabs(d3(ks), d3(ks+1));
 *        D = (a(K) + s2*c2) + w(k-ks)*c3, s2 = +0.5 (D-) / -0.5 (D+),
 *        w(0) = w(2) = 1/3, w(1) = -1/6
 *  The numerical Hamiltonian is the reference's (Godunov or LF) applied to
 *  (D-, D+).  Stages: s = Vs + dt*Hhat(Vs); Euler/first stage V1 = max(c, s);
 *  RK2 final max(c, 0.5*V + 0.5*s); RK3 second max(c, 0.75*V + 0.25*s),
 *  final max(c, (1/3)*V + (2/3)*s): the VI clamp after every stage.
 *  Residual = max|V_{n+1} - V_n| / dt.  ENO1 + Euler reproduces the
 *  reference update bit for bit (tested). */

static const double kThird = 1.0 / 3.0;
static const double kTwoThirds = 2.0 / 3.0;
static const double kSixthNeg = -1.0 / 6.0;

static inline double minabs(double x, double y) { return fabs(x) <= fabs(y) ? x : y; }

/* face difference a(j) along axis d for the node at linear index lin whose
 * axis-d index is k */
static inline double face(const double* v, int64_t lin, int64_t stride, int64_t k, int64_t n,
                          int64_t j, double inv, int godunov) {
  if (j < 0 || j > n - 2) {
    if (godunov || n < 2) return 0.0;
    j = j < 0 ? 0 : n - 2;
  }
  const double* p = v + lin + (j - k) * stride;
  return (p[stride] - p[0]) * inv;
}

static inline void eno_pair(const double* v, int64_t lin, int64_t stride, int64_t k, int64_t n,
                            double inv, int godunov, int order, double* dm, double* dp) {
  if (order <= 1) {
    *dm = face(v, lin, stride, k, n, k - 1, inv, godunov);
    *dp = face(v, lin, stride, k, n, k, inv, godunov);
    return;
  }
  double a[6]; /* a(k-3) .. a(k+2) */
  for (int t = 0; t < 6; ++t) a[t] = face(v, lin, stride, k, n, k - 3 + t, inv, godunov);
#define A(j) a[(j) - (k - 3)]
#define D2(j) (A(j) - A((j) - 1))
  if (order == 2) {
    *dm = A(k - 1) + 0.5 * minabs(D2(k - 1), D2(k));
    *dp = A(k) + -0.5 * minabs(D2(k), D2(k + 1));
  } else {
    for (int side = 0; side < 2; ++side) {
      const int64_t K = side == 0 ? k - 1 : k;
      const double x = D2(K), y = D2(K + 1);
      const int left = fabs(x) <= fabs(y);
      const double c2 = left ? x : y;
      const int64_t ks = left ? K - 1 : K;
      const double c3 = minabs(D2(ks + 1) - D2(ks), D2(ks + 2) - D2(ks + 1));
      const int64_t mm = k - ks;
      const double w = mm == 1 ? kSixthNeg : kThird;
      const double s2 = side == 0 ? 0.5 : -0.5;
      const double d = (A(K) + s2 * c2) + w * c3;
      if (side == 0) *dm = d; else *dp = d;
    }
  }
#undef D2
#undef A
}

/* one RK stage over the whole grid; kind: 0 V1 = max(c, s), 1 RK2 final,
 * 2 RK3 second, 3 RK3 final.  Returns max|out - vn| (meaningful for the
 * final stage). */
/* nodes [begin, end) of one stage */
static double ho_stage_range(const grid_t* g, const hjb_model* m, const hjb_dbounds* db,
                             const double* inv, int godunov, const double* global_alpha,
                             int order, const double* vs, const double* vn, const double* c,
                             const double* tg, double dt, int kind, double* out, int64_t begin,
                             int64_t end) {
  const int nd = g->nd;
  const int64_t nchunks = (end - begin + CHUNK - 1) / CHUNK;
  double best = 0.0;
#pragma omp parallel num_threads(nthreads())
  {
    double lbest = 0.0;
#pragma omp for schedule(static)
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int64_t lo = begin + ch * CHUNK;
      const int64_t hi = lo + CHUNK < end ? lo + CHUNK : end;
      int64_t idx[HJB_MAX_DIMS];
      double x[HJB_MAX_STATE], dminus[HJB_MAX_STATE], dplus[HJB_MAX_STATE];
      double costate[HJB_MAX_STATE], alpha[HJB_MAX_STATE];
      slopes_t slopes[HJB_MAX_STATE];
      hjb_interval dbn[HJB_MAX_INPUT];
      affine_t af;
      unravel(g, lo, idx);
      for (int64_t lin = lo; lin < hi; ++lin) {
        for (int d = 0; d < nd; ++d) x[d] = coord(g, d, idx[d]);
        for (int d = 0; d < nd; ++d)
          eno_pair(vs, lin, g->stride[d], idx[d], g->n[d], inv[d], godunov, order, &dminus[d],
                   &dplus[d]);
        db_at(db, lin, dbn);
        model_affine(m, x, idx, &af);
        double hhat = 0.0;
        if (godunov) {
          dim_slopes(&af, m->ubounds, dbn, slopes);
          for (int d = 0; d < nd; ++d) hhat += godunov_flux(slopes[d], dminus[d], dplus[d]);
        } else {
          for (int d = 0; d < nd; ++d) costate[d] = 0.5 * (dminus[d] + dplus[d]);
          hhat = hamiltonian(&af, costate, m->ubounds, dbn);
          if (!global_alpha) {
            flow_bounds(&af, m->ubounds, dbn, alpha);
            for (int d = 0; d < nd; ++d) hhat += alpha[d] * 0.5 * (dplus[d] - dminus[d]);
          } else {
            for (int d = 0; d < nd; ++d) hhat += global_alpha[d] * 0.5 * (dplus[d] - dminus[d]);
          }
        }
        const double st = vs[lin] + dt * hhat;
        double val;
        switch (kind) {
          case 1: val = 0.5 * vn[lin] + 0.5 * st; break;
          case 2: val = 0.75 * vn[lin] + 0.25 * st; break;
          case 3: val = kThird * vn[lin] + kTwoThirds * st; break;
          default: val = st; break;
        }
        if (tg) val = tg[lin] < val ? tg[lin] : val; /* target: min(l, .) first */
        const double cl = val > c[lin] ? val : c[lin];
        out[lin] = cl;
        const double dv = fabs(cl - vn[lin]);
        if (dv > lbest) lbest = dv;
        odometer(g, idx);
      }
    }
#pragma omp critical
    if (lbest > best) best = lbest;
  }
  return best;
}

static double ho_stage(const grid_t* g, const hjb_model* m, const hjb_dbounds* db,
                       const double* inv, int godunov, const double* global_alpha, int order,
                       const double* vs, const double* vn, const double* c, const double* tg,
                       double dt, int kind, double* out) {
  return ho_stage_range(g, m, db, inv, godunov, global_alpha, order, vs, vn, c, tg, dt, kind, out,
                        0, g->size);
}

/* one ENO/TVD-RK stage restricted to axis-0 planes [pb, pe) of the full grid
 * (the slab computation of one rank of the sharded solve) */
int hjo_ho_stage_planes(const hjb_grid* gi, const hjb_model* m, const hjb_dbounds* db,
                        const double* vs, const double* vn, const double* c, double dt,
                        int32_t order, int32_t kind, int64_t pb, int64_t pe, double* out,
                        double* max_dv) {
  grid_t g;
  int rc = check_ctx(gi, m, db, &g);
  if (rc) return rc;
  if (pb < 0 || pe > g.n[0] || pb >= pe)
    return fail(HJB_ERR_INVALID_ARGUMENT, "ho_stage_planes: bad plane range");
  double inv[HJB_MAX_DIMS];
  for (int d = 0; d < g.nd; ++d) inv[d] = 1.0 / g.spacing[d];
  *max_dv = ho_stage_range(&g, m, db, inv, 1, NULL, order, vs, vn, c, NULL, dt, kind, out,
                           pb * g.stride[0], pe * g.stride[0]);
  return 0;
}

int hjo_ho_solve(const grid_t* g, const hjb_model* m, const hjb_dbounds* db, const double* init,
                 const double* c, const hjb_solve_config* cfg, const hjo_scan* s, double dt,
                 double* out, hjb_solve_result* res) {
  const int order = cfg->spatial_order < 1 ? 1 : cfg->spatial_order;
  const int rk = cfg->time_order < 1 ? 1 : cfg->time_order;
  if (order > 3 || rk > 3) return fail(HJB_ERR_INVALID_ARGUMENT, "SolveConfig: order must be 1..3");
  const double* ga = cfg->dissipation == HJB_GLOBAL ? s->max_alpha : NULL;
  const int godunov = cfg->scheme == HJB_GODUNOV;
  double inv[HJB_MAX_DIMS];
  for (int d = 0; d < g->nd; ++d) inv[d] = 1.0 / g->spacing[d];
  const size_t bytes = g->size * sizeof(double);
  double* front = (double*)malloc(bytes);
  double* back = (double*)malloc(bytes);
  double* s1 = (double*)malloc(bytes);
  double* s2 = (double*)malloc(bytes);
  memcpy(front, init, bytes);
  const double t0 = now_ms();
  double min_residual = INFINITY, first = 0.0, residual = 0.0;
  int status = 0;
  for (int64_t iter = 1; iter <= cfg->max_iters; ++iter) {
    double max_dv;
    if (rk == 1) {
      max_dv = ho_stage(g, m, db, inv, godunov, ga, order, front, front, c, cfg->target, dt, 0, back);
    } else if (rk == 2) {
      ho_stage(g, m, db, inv, godunov, ga, order, front, front, c, cfg->target, dt, 0, s1);
      max_dv = ho_stage(g, m, db, inv, godunov, ga, order, s1, front, c, cfg->target, dt, 1, back);
    } else {
      ho_stage(g, m, db, inv, godunov, ga, order, front, front, c, cfg->target, dt, 0, s1);
      ho_stage(g, m, db, inv, godunov, ga, order, s1, front, c, cfg->target, dt, 2, s2);
      max_dv = ho_stage(g, m, db, inv, godunov, ga, order, s2, front, c, cfg->target, dt, 3, back);
    }
    residual = max_dv / dt;
    double* t = front;
    front = back;
    back = t;
    res->iterations = iter;
    if (iter == 1) first = residual;
    if (res->residual_history && iter <= res->history_capacity)
      res->residual_history[iter - 1] = residual;
    if (res->wall_ms_history && iter <= res->history_capacity)
      res->wall_ms_history[iter - 1] = now_ms() - t0;
    if (residual < cfg->tolerance) {
      res->converged = 1;
      break;
    }
    min_residual = STD_MIN(min_residual, residual);
    if (!isfinite(residual) || residual > 10.0 * STD_MAX(min_residual, first)) {
      status = fail(HJB_ERR_DIVERGED, "solve: diverging (residual grew 10x above its minimum)");
      break;
    }
    if (cfg->time_horizon > 0.0 && (double)iter * dt >= cfg->time_horizon) break;
  }
  res->final_residual = residual;
  memcpy(out, front, bytes);
  res->wall_seconds = (now_ms() - t0) * 1e-3;
  free(front);
  free(back);
  free(s1);
  free(s2);
  return status;
}

/* ------------------------------------------------------------------- GP */
/* GpModel::kernel, gp.cpp:22-30 */
static double gp_kernel(const hjb_gp_model* m, const double* a, const double* b) {
  double q = 0.0;
  for (int d = 0; d < m->input_dim; ++d) {
    const double r = (a[d] - b[d]) / m->lengthscales[d];
    q += r * r;
  }
  return m->signal_var * exp(-0.5 * q);
}

/* GpModel::predict, gp.cpp:188-208 */
int hjo_gp_predict(const hjb_gp_model* m, const double* x, double* mean, double* variance) {
  const int64_t n = m->n_train;
  if (n == 0) {  /* prior, gp.cpp:190 */
    *mean = 0.0;
    *variance = m->signal_var;
    return 0;
  }
  double* v = (double*)malloc((size_t)n * sizeof(double));
  if (!v) return fail(HJB_ERR_RUNTIME, "GP predict: out of memory");
  for (int64_t i = 0; i < n; ++i) v[i] = gp_kernel(m, x, m->inputs + i * m->input_dim);
  double mu = 0.0;
  for (int64_t i = 0; i < n; ++i) mu += v[i] * m->alpha[i];
  /* v = L^-1 k*, forward substitution (gp.cpp:196-202) */
  for (int64_t i = 0; i < n; ++i) {
    double s = v[i];
    for (int64_t j = 0; j < i; ++j) s -= m->chol[i * n + j] * v[j];
    v[i] = s / m->chol[i * n + i];
  }
  double var = m->signal_var;
  for (int64_t i = 0; i < n; ++i) var -= v[i] * v[i];
  free(v);
  *mean = mu;
  *variance = STD_MAX(var, 0.0);
  return 0;
}

/* bounds_on_grid, gp.cpp:211-249 */
int hjo_gp_bounds_on_grid(const hjb_grid* gi, int32_t channels, const hjb_gp_model* models,
                          double confidence, double* const* lo, double* const* hi) {
  grid_t g;
  int rc = grid_init(gi, &g);
  if (rc) return rc;
  for (int ch = 0; ch < channels; ++ch) {
    const hjb_gp_model* m = &models[ch];
    if (m->n_dims != m->input_dim)
      return fail(HJB_ERR_INVALID_ARGUMENT, "bounds_on_grid: input-dim map does not match GP");
    for (int d = 0; d < m->n_dims; ++d)
      if (m->input_dims[d] < 0 || m->input_dims[d] >= g.nd)
        return fail(HJB_ERR_INVALID_ARGUMENT, "bounds_on_grid: input dim out of grid range");
  }
  for (int ch = 0; ch < channels; ++ch) {
    const hjb_gp_model* m = &models[ch];
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t lin = 0; lin < g.size; ++lin) {
      int64_t idx[HJB_MAX_DIMS];
      double x[HJB_MAX_DIMS];
      unravel(&g, lin, idx);
      for (int d = 0; d < m->n_dims; ++d)
        x[d] = coord(&g, m->input_dims[d], idx[m->input_dims[d]]);
      double mean, var;
      if (hjo_gp_predict(m, x, &mean, &var)) {
        bad = 1;
        continue;
      }
      const double band = confidence * sqrt(var + m->noise_var);
      lo[ch][lin] = mean - band;
      hi[ch][lin] = mean + band;
    }
    if (bad) return fail(HJB_ERR_RUNTIME, "GP predict: out of memory");
  }
  return 0;
}
