/*
 * hj_oracle.h — TEST INFRASTRUCTURE ONLY: plain-C CPU restatement of the
 * reference's hot path (hjsafe::solve and its helpers).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.  The product (libhjb.so) never
 * links or calls it.  Each function cites the reference file:line it
 * restates.  Parity of this restatement is pinned against the reference
 * itself (oracle/_ref/libhjref.so, built from the unmodified reference
 * sources) and against the golden fixtures under tests/golden/.
 *
 * The ENO2/ENO3 + TVD-RK2/RK3 extension (hjo_sweep_ho / hjo_solve with
 * spatial_order/time_order > 1) has NO reference implementation (reference
 * SPEC.md:324 lists high-order schemes as non-goals): that part is
 * "parity unpinned" and is validated by reduction to the first-order
 * reference, convergence-order tests and sign agreement.
 */
#ifndef HJ_ORACLE_H_
#define HJ_ORACLE_H_

#include <stdint.h>

#include "../include/hjb.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hjo_scan {
  double max_speed_sum;
  double max_alpha[HJB_MAX_STATE];
  int32_t separable;
} hjo_scan;

/* Status codes follow hjb_status.  Messages mirror the reference's. */
const char* hjo_last_error(void);
void hjo_set_threads(int threads);

/* scan_alpha, solver.cpp:221-268 */
int hjo_scan_alpha(const hjb_grid* g, const hjb_model* m, const hjb_dbounds* db, hjo_scan* out);
/* cfl_dt, solver.cpp:272-282 */
int hjo_cfl_dt(const hjb_grid* g, const hjb_model* m, const hjb_dbounds* db, double cfl,
               double* dt);
/* update_chunk over the whole grid, solver.cpp:106-190; returns max|dV|.
 * global_alpha == NULL selects per-node dissipation. */
int hjo_sweep(const hjb_grid* g, const hjb_model* m, const hjb_dbounds* db, const double* v,
              const double* c, double dt, int32_t scheme, const double* global_alpha,
              double* out, double* max_dv);
/* update_chunk over planes [plane_begin, plane_end) of axis 0 only: the slab
 * computation of one rank of the multi-GPU partition (neighbour planes are
 * read from v; the grid's own edges keep the reference edge rule). */
int hjo_sweep_planes(const hjb_grid* g, const hjb_model* m, const hjb_dbounds* db,
                     const double* v, const double* c, double dt, int32_t scheme,
                     const double* global_alpha, int64_t plane_begin, int64_t plane_end,
                     double* out, double* max_dv);
/* vi_step, solver.cpp:284-308 */
int hjo_vi_step(const hjb_grid* g, const hjb_model* m, const hjb_dbounds* db, const double* v,
                const double* c, double dt, const hjb_solve_config* cfg, double* out);
/* solve, solver.cpp:310-376 (+ ENO/TVD-RK extension when orders > 1) */
int hjo_solve(const hjb_grid* g, const hjb_model* m, const hjb_dbounds* db, const double* init,
              const double* c, const hjb_solve_config* cfg, double* out, hjb_solve_result* res);
/* interp_ex at a point, grid.cpp:84-135 (returns out_of_domain flag) */
int hjo_interp(const hjb_grid* g, const double* field, const double* x, double* value,
               int32_t* out_of_domain);
/* resample, grid.cpp:215-231 */
int hjo_resample(const hjb_grid* src_g, const double* src, const hjb_grid* dst_g, double* dst);
/* max_adjacent_jump, grid.cpp:197-213 */
int hjo_max_adjacent_jump(const hjb_grid* g, const double* v, double* out);
/* seed_from, solver.cpp:404-411 */
int hjo_seed_from(const hjb_grid* src_g, const double* src, const hjb_grid* dst_g,
                  const double* c_dst, double* dst);
/* solve_coarse_to_fine, solver.cpp:387-425 (dbounds must be constant) */
int hjo_solve_coarse_to_fine(const hjb_grid* fine, const hjb_model* m, const hjb_dbounds* db,
                             const double* c_fine, const hjb_grid* coarse,
                             const hjb_solve_config* cfg, const double* warm_init_fine,
                             double* coarse_out, hjb_solve_result* coarse_res, double* fine_out,
                             hjb_solve_result* fine_res);
/* N-level chain generalising solve_coarse_to_fine (solver.cpp:387-425),
 * composed from resample + max_adjacent_jump + clamp + solve (the reference's
 * seed_from is a private lambda, solver.cpp:404-411).  values_out[l] may be
 * NULL. */
int hjo_solve_multilevel(int32_t nlevels, const hjb_grid* grids, const hjb_model* m,
                         const hjb_dbounds* db, const double* c_fine, const hjb_solve_config* cfg,
                         const double* warm_init_fine, double* const* values_out,
                         hjb_solve_result* results);
/* signed_distance_band / signed_distance_box, levelset.cpp:11-66 */
int hjo_signed_distance_band(const hjb_grid* g, int32_t dim, double lo, double hi, double* out);
int hjo_signed_distance_box(const hjb_grid* g, const double* lo, const double* hi, double* out);
/* hamiltonian / flow_bounds at a point, dynamics.cpp:37-112 */
int hjo_hamiltonian(const hjb_model* m, const double* x, const double* p, const hjb_interval* db,
                    double* h);
int hjo_flow_bounds(const hjb_model* m, const double* x, const hjb_interval* db, double* alpha);

/* one Godunov ENO/TVD-RK stage on axis-0 planes [pb, pe) (high-order
 * extension, parity unpinned; kind: 0 Euler/first stage, 1 RK2 final,
 * 2 RK3 second, 3 RK3 final) */
int hjo_ho_stage_planes(const hjb_grid* g, const hjb_model* m, const hjb_dbounds* db,
                        const double* vs, const double* vn, const double* c, double dt,
                        int32_t order, int32_t kind, int64_t pb, int64_t pe, double* out,
                        double* max_dv);

/* SafetyFilter::optimal_control / filter batched (safety.cpp:86-127) */
int hjo_filter_batch(const hjb_grid* g, const hjb_model* m, const hjb_dbounds* db,
                     const double* value, int64_t nq, const double* x, const double* u_perf,
                     const hjb_filter_config* cfg, const hjb_filter_out* out);

/* GpModel::predict, gp.cpp:188-208 (kernel gp.cpp:22-30): mean and latent
 * variance at x[0 .. input_dim).  n_train == 0 is the prior. */
int hjo_gp_predict(const hjb_gp_model* m, const double* x, double* mean, double* variance);
/* bounds_on_grid, gp.cpp:211-249: predict at EVERY node (the reference's
 * per-node evaluation), band = confidence * sqrt(var + noise_var). */
int hjo_gp_bounds_on_grid(const hjb_grid* g, int32_t channels, const hjb_gp_model* models,
                          double confidence, double* const* lo, double* const* hi);

#ifdef __cplusplus
}
#endif

#endif
