/*
 * ref_shim.h — TEST INFRASTRUCTURE ONLY.
 *
 * extern "C" harness over the UNMODIFIED reference sources
 * (/root/reference/proj/src/{grid,hjvf,levelset,dynamics,interval_field,
 * solver,safety,decomposition}.cpp), compiled by oracle/Makefile into oracle/_ref/libhjref.so.
 * It is the parity anchor for the C restatement (oracle/hj_oracle.c) and the
 * CPU arm of bench.py.  The product path never links or loads it.
 */
#ifndef HJ_REF_SHIM_H_
#define HJ_REF_SHIM_H_

#include <stdint.h>

#include "../include/hjb.h"

#ifdef __cplusplus
extern "C" {
#endif

enum hjr_model_kind {
  HJR_QUAD2D_VERT = 0,    /* Quad2DVert           dynamics.hpp:102-125 */
  HJR_PLANAR4D = 1,       /* NearHoverPlanar4D    dynamics.hpp:133-162 */
  HJR_VERTICAL2D = 2,     /* NearHoverVertical2D  dynamics.hpp:170-197 */
  HJR_DOUBLE_INT = 3,     /* DoubleIntegrator     dynamics.hpp:201-223 */
  HJR_TWIN_DI = 4,        /* TwinDoubleIntegrator dynamics.hpp:227-244 */
  HJR_ADVECTION = 5,      /* ConstantAdvection, test_solver.cpp:14-29  */
  HJR_NEAR_HOVER_10D = 6  /* NearHover10D         dynamics.hpp:250-271 */
};

/* Model by kind + parameters.
 *  QUAD2D_VERT: p = {k_thrust, k_offset, gravity}
 *  PLANAR4D:    p = {d0, d1, n0, gravity, max_angle_cmd}; d_row = 1 is the
 *               stock reference class, d_row = 0 the BASELINE variant (wind
 *               on the position row) as a harness-side DynamicsModel
 *               subclass, exactly like the reference's own test models.
 *  VERTICAL2D:  p = {gravity, thrust_gain, frac_lo, frac_hi}
 *  DOUBLE_INT / TWIN_DI: p = {a_min, a_max}
 *  ADVECTION:   d_row = number of dims, p = speeds
 *  NEAR_HOVER_10D: p = {planar d0,d1,n0,g,max_angle, vertical g,kT,lo,hi} */
typedef struct hjr_model_spec {
  int32_t kind;
  int32_t d_row;
  double p[10];
} hjr_model_spec;

typedef struct hjr_result {
  int64_t iterations;
  double dt;
  double wall_seconds;
  int32_t converged;
  int32_t reserved;
  int64_t nodes_per_sweep;
  double* residual_history;
  int64_t history_capacity;
  double* wall_ms_history; /* may be NULL; history_capacity entries */
} hjr_result;

/* All return 0 on success, 1 std::invalid_argument, 2 std::runtime_error,
 * 3 other; the message is copied into err (if non-NULL). */
int hjr_cfl_dt(const hjb_grid* g, const hjr_model_spec* m, const hjb_dbounds* db, double cfl,
               unsigned threads, double* dt, char* err, int errlen);
int hjr_vi_step(const hjb_grid* g, const hjr_model_spec* m, const hjb_dbounds* db,
                const double* v, const double* c, double dt, const hjb_solve_config* cfg,
                double* out, char* err, int errlen);
int hjr_solve(const hjb_grid* g, const hjr_model_spec* m, const hjb_dbounds* db,
              const double* init, const double* c, const hjb_solve_config* cfg, double* out,
              hjr_result* res, char* err, int errlen);
int hjr_solve_coarse_to_fine(const hjb_grid* fine, const hjr_model_spec* m,
                             const hjb_dbounds* db_fine, const double* c_fine,
                             const hjb_grid* coarse, const hjb_solve_config* cfg,
                             const double* warm_init_fine, double* coarse_out,
                             hjr_result* coarse_res, double* fine_out, hjr_result* fine_res,
                             char* err, int errlen);
/* solve_coarse_to_fine with the warm start on its OWN grid (the reference's
 * ScalarField carries its grid; seed_from resamples from it,
 * solver.cpp:404-414).  Used to compose the N-level chain from the
 * reference's own 2-level driver. warm_grid == NULL means the fine grid. */
int hjr_solve_coarse_to_fine_w(const hjb_grid* fine, const hjr_model_spec* m,
                               const hjb_dbounds* db_fine, const double* c_fine,
                               const hjb_grid* coarse, const hjb_solve_config* cfg,
                               const hjb_grid* warm_grid, const double* warm, double* coarse_out,
                               hjr_result* coarse_res, double* fine_out, hjr_result* fine_res,
                               char* err, int errlen);
int hjr_resample(const hjb_grid* src_g, const double* src, const hjb_grid* dst_g, double* dst,
                 char* err, int errlen);
int hjr_max_adjacent_jump(const hjb_grid* g, const double* v, double* out, char* err,
                          int errlen);
/* levelset.cpp:80-86 (the reference's own field_max / field_min) */
int hjr_field_max(const hjb_grid* g, const double* a, const double* b, double* out, char* err,
                  int errlen);
int hjr_field_min(const hjb_grid* g, const double* a, const double* b, double* out, char* err,
                  int errlen);
int hjr_signed_distance_band(const hjb_grid* g, int32_t dim, double lo, double hi, double* out,
                             char* err, int errlen);
int hjr_signed_distance_box(const hjb_grid* g, const double* lo, const double* hi, double* out,
                            char* err, int errlen);
/* dynamics probes (test_dynamics.cpp restatements) */
int hjr_hamiltonian(const hjr_model_spec* m, const double* x, const double* p,
                    const hjb_interval* db, double* h, char* err, int errlen);
int hjr_flow_bounds(const hjr_model_spec* m, const double* x, const hjb_interval* db,
                    double* alpha, char* err, int errlen);
int hjr_affine(const hjr_model_spec* m, const double* x, double* drift, double* control,
               double* disturbance, hjb_interval* ubounds, int32_t* dims, char* err,
               int errlen);
/* HJVF I/O (hjvf.cpp:46-95) for golden files */
/* SafetyFilter (safety.hpp:35-107) around V with Config::eta_floor; after
 * contract(violations) (viol_x: nviol states), answers nq queries with
 * filter (mode HJB_FILTER_FILTER, u_perf per query) or optimal_control;
 * reports the filter's lambda and emergency flag. */
int hjr_filter_batch(const hjb_grid* g, const hjr_model_spec* m, const hjb_dbounds* db,
                     const double* value, int64_t nq, const double* x, const double* u_perf,
                     int32_t mode, double eta_floor, int64_t nviol, const double* viol_x,
                     double* lambda_out, int32_t* emergency_out, const hjb_filter_out* out,
                     char* err, int errlen);
/* Decomposition (decomposition.hpp:33-80) of nsub subsystems, each with its
 * grid, model, bounds and converged V (values[i]); maps holds, per
 * subsystem, state_map, control_map and disturbance_map back to back.
 * After contract(violations) (viol_x: nviol full states), answers nq full
 * queries: combined_value -> cv_out, combined_control -> value / band /
 * control / flags (HJB_FILTER_OVERRIDE | HJB_FILTER_OOD). */
int hjr_decomposition_batch(int32_t nsub, const hjb_grid* grids, const hjr_model_spec* models,
                            const hjb_dbounds* dbs, const double* const* values,
                            const int32_t* maps, int32_t full_n, int32_t full_m, int32_t full_p,
                            double eta_floor, int64_t nviol, const double* viol_x, int64_t nq,
                            const double* x, const double* u_perf, double* lambda_out,
                            int32_t* emergency_out, double* cv_out, double* value_out,
                            double* band_out, double* control_out, uint8_t* flags_out, char* err,
                            int errlen);
int hjr_write_hjvf(const char* path, const hjb_grid* g, const double* v, char* err, int errlen);

#ifdef __cplusplus
}
#endif

#endif
