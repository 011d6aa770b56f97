/*
 * hjb.h — C ABI of the B200-native Hamilton-Jacobi reachability solver.
 *
 * This is the drop-in boundary for the reference library's solver API
 * (hjsafe, `proj/include/hjsafe/solver.hpp:45-77`).  Every entry point below
 * replaces one reference function; the citation is given next to it.  All
 * signatures use plain C types: pointers, sizes and POD descriptors — no C++
 * or torch types cross this boundary.
 *
 * Conventions
 *  - Fields are fp64, row-major, last axis fastest (reference
 *    `proj/src/grid.cpp:27-30`).
 *  - Functions without a suffix take HOST pointers (the reference's
 *    `ScalarField` / `IntervalField` storage) and copy to/from the GPU inside
 *    the call.  Functions with the `_dev` suffix take DEVICE pointers so warm
 *    and adaptive chains stay resident in HBM.
 *  - Every call returns an `int` status (hjb_status).  The message of the
 *    last failure on the calling thread is returned by hjb_last_error().
 *    HJB_ERR_INVALID_ARGUMENT maps to the reference's std::invalid_argument,
 *    HJB_ERR_RUNTIME / HJB_ERR_DIVERGED to std::runtime_error
 *    (`proj/src/solver.cpp:14-17,194-199,279-280,291-295,318-322,367-369`).
 *  - A context (hjb_context) owns a CUDA stream and device workspaces.  A
 *    context must not be used by two threads at once; independent contexts
 *    may run concurrently (the reference's solve is re-entrant,
 *    `proj/src/sim.cpp:340-363`).
 *  - There is no CPU fallback: without a usable CUDA device every compute
 *    call fails with HJB_ERR_CUDA.
 */
#ifndef HJB_H_
#define HJB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HJB_MAX_DIMS 6   /* grid rank supported by the device kernels */
#define HJB_MAX_STATE 10 /* reference kMaxStateDim, dynamics.hpp:12 */
#define HJB_MAX_INPUT 3  /* reference kMaxInputDim, dynamics.hpp:13 */
#define HJB_MAX_LEVELS 8 /* hjb_solve_multilevel */

typedef enum hjb_status {
  HJB_OK = 0,
  HJB_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  HJB_ERR_RUNTIME = 2,          /* std::runtime_error (e.g. zero flow)     */
  HJB_ERR_CUDA = 3,             /* no device / CUDA failure                */
  HJB_ERR_UNSUPPORTED = 4,      /* valid for the reference, not on device  */
  HJB_ERR_DIVERGED = 5,         /* std::runtime_error "solve: diverging"   */
  HJB_ERR_NCCL = 6
} hjb_status;

/* ---------------------------------------------------------------- grid */
/* GridDim, reference grid.hpp:11-17 (same field order). */
typedef struct hjb_grid_dim {
  double min;
  double max;
  int64_t n;
} hjb_grid_dim;

/* Grid, reference grid.hpp:23-48.  spacing = (max-min)/(n-1)
 * (grid.cpp:24); coord(d,k) = k==n-1 ? max : min + k*spacing
 * (grid.cpp:33-38). */
typedef struct hjb_grid {
  int32_t ndims;
  int32_t reserved;
  hjb_grid_dim dims[HJB_MAX_DIMS];
} hjb_grid;

/* Interval, reference dynamics.hpp:16-19. */
typedef struct hjb_interval {
  double lo;
  double hi;
} hjb_interval;

/* ------------------------------------------------------------- dynamics */
/* Control-affine dynamics f(x,u,d) = drift(x) + B u + C d (reference
 * AffineFlow, dynamics.hpp:24-33) with an additively separable drift:
 *   drift_i(x) = term0_i(x) + term1_i(x)      (term1 optional)
 * Each term depends on one coordinate and is evaluated with the reference
 * model's own expression, so the device consumes identical bits:
 *   COORD: scale * x[axis]          e.g. x[1], -d1*theta   (dynamics.cpp:139)
 *   TAN:   scale * tan(x[axis])     g*tan(theta)           (dynamics.cpp:138)
 *   CONST: scale                    -g, gravity+k_offset   (dynamics.cpp:129,148)
 *   TABLE: table[k_axis]            user-tabulated f(x_axis), one entry per node
 * Every model of the reference (dynamics.cpp:126-198) has this form. */
typedef enum hjb_term_kind {
  HJB_TERM_NONE = 0,
  HJB_TERM_COORD = 1,
  HJB_TERM_TAN = 2,
  HJB_TERM_CONST = 3,
  HJB_TERM_TABLE = 4
} hjb_term_kind;

typedef struct hjb_drift_term {
  int32_t kind;
  int32_t axis;
  double scale;
  const double* table; /* host pointer, HJB_TERM_TABLE only */
} hjb_drift_term;

typedef struct hjb_model {
  int32_t state_dim;
  int32_t control_dim;
  int32_t disturbance_dim;
  int32_t reserved;
  hjb_drift_term drift[HJB_MAX_STATE][2];
  double control[HJB_MAX_STATE][HJB_MAX_INPUT];     /* B, row per state */
  double disturbance[HJB_MAX_STATE][HJB_MAX_INPUT]; /* C, row per state */
  hjb_interval ubounds[HJB_MAX_INPUT];              /* control_bounds() */
} hjb_model;

/* IntervalField, reference interval_field.hpp:11-42: per channel [lo,hi]
 * either constant (IntervalField::constant, interval_field.cpp:16-27) or one
 * value per node.  Per-node pointers live in the same memory space as the
 * field pointers of the call (host for plain calls, device for _dev). */
typedef struct hjb_dbounds {
  int32_t channels;
  int32_t per_node;
  hjb_interval constant[HJB_MAX_INPUT];
  const double* lo[HJB_MAX_INPUT];
  const double* hi[HJB_MAX_INPUT];
} hjb_dbounds;

/* --------------------------------------------------------------- solver */
typedef enum hjb_scheme { HJB_GODUNOV = 0, HJB_LAX_FRIEDRICHS = 1 } hjb_scheme;
typedef enum hjb_dissipation { HJB_PER_NODE = 0, HJB_GLOBAL = 1 } hjb_dissipation;

/* SolveConfig, reference solver.hpp:12-25, plus the B200 extensions
 * (spatial/time order, time horizon, target set). */
typedef struct hjb_solve_config {
  double cfl_factor;     /* (0,1], default 0.8 */
  double tolerance;      /* > 0, default 1e-3 */
  int64_t max_iters;     /* default 20000 */
  int32_t scheme;        /* hjb_scheme, default Godunov */
  int32_t dissipation;   /* hjb_dissipation, default per-node */
  int32_t spatial_order; /* 1 = reference first order; 2 = ENO2; 3 = ENO3 */
  int32_t time_order;    /* 1 = forward Euler (reference); 2/3 = TVD-RK */
  double time_horizon;   /* > 0: also stop once iterations*dt >= horizon */
  int32_t threads;       /* reference CPU knob; accepted and ignored */
  int32_t flags;         /* HJB_FLAG_* (0 by default) */
  /* Optional target set l(x) (B200 extension, no reference counterpart; the
   * reference clamps against the avoid set only, solver.cpp:178-179): a field
   * on the solve's grid, in the memory space of the call's other fields.
   * Every update (every RK stage) becomes the reach-avoid
   *   V' = max(c, min(l, stepped))      (std::min / std::max order)
   * NULL (default) = the reference update V' = max(c, stepped).  Supported
   * by hjb_solve / hjb_solve_dev / hjb_vi_step[_dev]; the sharded and
   * multilevel drivers reject it. */
  const double* target;
} hjb_solve_config;

/* run the ENO/TVD-RK stage machinery even for order 1 / Euler (verification:
 * it must reproduce the reference update bit for bit) */
#define HJB_FLAG_FORCE_HO 1

/* hjb_solve_result.kernel: which kernel family ran the iterations (a model
 * or bound field outside the 4D fast path's shapes runs the generic kernel,
 * ~3.5x slower per cell at 51^4; this reports it instead of falling back
 * silently) */
#define HJB_KERNEL_NONE 0          /* max_iters == 0 */
#define HJB_KERNEL_GENERIC 1       /* k_step, any rank 1..6 */
#define HJB_KERNEL_FAST4D 2        /* k_fast4d, one launch per sweep */
#define HJB_KERNEL_FAST4D_MULTI 3  /* k_fast4d multi-sweep persistent launch */
#define HJB_KERNEL_SMALL2D 4       /* k_small2d, whole loop in one cluster launch */
#define HJB_KERNEL_HO_GENERIC 5    /* k_ho_stage (ENO / TVD-RK, rank 1..4) */
#define HJB_KERNEL_HO4D 6          /* k_ho4t / k_eno3g / k_ho4d */
#define HJB_KERNEL_SMALL2D_HO 7    /* k_small2d_ho */
#define HJB_KERNEL_FAST4D_GEN 8    /* k_fast4d<ShapeGen>: run-time row shapes, one launch per sweep */

/* SolveResult, reference solver.hpp:27-36.  The value field is written to
 * the caller's buffer; histories are written to caller buffers of
 * `history_capacity` entries (may be NULL / 0). */
typedef struct hjb_solve_result {
  int64_t iterations;
  double dt;
  double wall_seconds;  /* device time of the iteration loop */
  int32_t converged;
  int32_t kernel;       /* HJB_KERNEL_*: the sweep kernel the solve ran */
  int64_t nodes_per_sweep;
  double final_residual;
  double* residual_history; /* max|dV|/dt per iteration */
  double* wall_ms_history;  /* cumulative device ms per iteration */
  int64_t history_capacity;
} hjb_solve_result;

typedef struct hjb_context hjb_context;

/* ------------------------------------------------------------ lifecycle */
const char* hjb_version(void);
const char* hjb_last_error(void);
void hjb_solve_config_default(hjb_solve_config* cfg);
int hjb_context_create(int device, hjb_context** out);
int hjb_context_destroy(hjb_context* ctx);
int hjb_device_count(int* out);

/* ------------------------------------------------------------ solver API */
/* cfl_dt, reference solver.hpp:48-49 / solver.cpp:272-282. */
int hjb_cfl_dt(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
               const hjb_dbounds* dbounds, double cfl_factor, double* dt_out);

/* vi_step, reference solver.hpp:55-57 / solver.cpp:284-308. */
int hjb_vi_step(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
                const hjb_dbounds* dbounds, const double* value, const double* constraint,
                double dt, const hjb_solve_config* cfg, double* out);

/* solve, reference solver.hpp:63-65 / solver.cpp:310-376.  init may be the
 * constraint pointer itself (the reference's cold solve, solve(c, c, ...),
 * sim.cpp:282): the field is then copied to the device once. */
int hjb_solve(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
              const hjb_dbounds* dbounds, const double* init, const double* constraint,
              const hjb_solve_config* cfg, double* value_out, hjb_solve_result* result);

/* solve_coarse_to_fine, reference solver.hpp:70-74 / solver.cpp:387-425.
 * warm_init_fine may be NULL (cold coarse stage). */
int hjb_solve_coarse_to_fine(hjb_context* ctx, const hjb_grid* fine_grid,
                             const hjb_model* model, const hjb_dbounds* dbounds_fine,
                             const double* constraint_fine, const hjb_grid* coarse_grid,
                             const hjb_solve_config* cfg, const double* warm_init_fine,
                             double* coarse_value_out, hjb_solve_result* coarse_result,
                             double* fine_value_out, hjb_solve_result* fine_result,
                             double* wall_seconds);

/* Multi-level adaptive solve, the N-level generalisation of
 * solve_coarse_to_fine (reference solver.cpp:387-425; with nlevels == 2 it is
 * that function exactly).  grids[0..nlevels-1] run coarse to fine; the last
 * is the fine grid of c_fine / dbounds_fine.  For every coarser level l:
 * c_l = resample(c_fine, grid_l), db_l = resample(db_fine, grid_l)
 * (solver.cpp:396-397); level 0 starts from c_0, or from
 * seed_from(warm_init_fine, grid_0, c_0) when warm_init_fine != NULL
 * (solver.cpp:413-414); level l > 0 starts from
 * seed_from(V*_{l-1}, grid_l, c_l) (solver.cpp:404-411,419-420).  A level
 * that does not converge still seeds the next (the reference has no
 * converged-check between stages).  values_out[l] (may be NULL) receives V*_l,
 * results[l] its SolveResult. */
int hjb_solve_multilevel(hjb_context* ctx, int32_t nlevels, const hjb_grid* grids,
                         const hjb_model* model, const hjb_dbounds* dbounds_fine,
                         const double* c_fine, const hjb_solve_config* cfg,
                         const double* warm_init_fine, double* const* values_out,
                         hjb_solve_result* results, double* wall_seconds);
/* Same with device pointers (c_fine, warm_init_fine, values_out[l] and the
 * per-node bounds of dbounds_fine). */
int hjb_solve_multilevel_dev(hjb_context* ctx, int32_t nlevels, const hjb_grid* grids,
                             const hjb_model* model, const hjb_dbounds* dbounds_fine,
                             const double* c_fine, const hjb_solve_config* cfg,
                             const double* warm_init_fine, double* const* values_out,
                             hjb_solve_result* results, double* wall_seconds);

/* ------------------------------------------------ grid / level-set helpers */
/* resample (multilinear), reference grid.hpp:108-109 / grid.cpp:215-231. */
int hjb_resample(hjb_context* ctx, const hjb_grid* src_grid, const double* src,
                 const hjb_grid* dst_grid, double* dst);

/* max_adjacent_jump, reference grid.hpp:104 / grid.cpp:197-213. */
int hjb_max_adjacent_jump(hjb_context* ctx, const hjb_grid* grid, const double* field,
                          double* out);

/* seed_from lambda, reference solver.cpp:404-411:
 *   dst = max(resample(src) - max_adjacent_jump(src), constraint_dst). */
int hjb_seed_from(hjb_context* ctx, const hjb_grid* src_grid, const double* src,
                  const hjb_grid* dst_grid, const double* constraint_dst, double* dst);

/* signed_distance_band, reference levelset.hpp:31 / levelset.cpp:54-66. */
int hjb_signed_distance_band(hjb_context* ctx, const hjb_grid* grid, int32_t dim, double lo,
                             double hi, double* out);

/* ------------------------------------------- device-resident (_dev) API */
int hjb_vi_step_dev(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
                    const hjb_dbounds* dbounds, const double* value, const double* constraint,
                    double dt, const hjb_solve_config* cfg, double* out);

int hjb_solve_dev(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
                  const hjb_dbounds* dbounds, const double* init, const double* constraint,
                  const hjb_solve_config* cfg, double* value_out, hjb_solve_result* result);

int hjb_resample_dev(hjb_context* ctx, const hjb_grid* src_grid, const double* src,
                     const hjb_grid* dst_grid, double* dst);

int hjb_max_adjacent_jump_dev(hjb_context* ctx, const hjb_grid* grid, const double* field,
                              double* out);

int hjb_seed_from_dev(hjb_context* ctx, const hjb_grid* src_grid, const double* src,
                      const hjb_grid* dst_grid, const double* constraint_dst, double* dst);

int hjb_signed_distance_band_dev(hjb_context* ctx, const hjb_grid* grid, int32_t dim,
                                 double lo, double hi, double* out);

/* Elementwise max/min (field_max/field_min, levelset.cpp:81-95). */
int hjb_field_max_dev(hjb_context* ctx, int64_t n, const double* a, const double* b,
                      double* out);
int hjb_field_min_dev(hjb_context* ctx, int64_t n, const double* a, const double* b,
                      double* out);
/* out = -a: the complement {x : -f(x) <= 0} of a level-set field (an
 * obstacle band turned into an avoid set, config 5); no reference function
 * (the reference composes sets by field_max / field_min only). */
int hjb_field_negate_dev(hjb_context* ctx, int64_t n, const double* a, double* out);

/* ------------------------------------------- multi-GPU slab partition */
/* Axis-0 slab partition across ranks: one process per GPU,
 * balanced slabs (the first n0 % nranks ranks own one extra plane). */
typedef struct hjb_comm hjb_comm;
int hjb_slab_partition(int64_t n0, int32_t nranks, int32_t rank, int64_t* begin, int64_t* end);
/* The plan one rank runs (host only, no device needed): local geometry and
 * the halo protocol, in LOCAL plane numbers of the rank's buffers.
 * out[0..14] = {owned, nloc, cbeg, cend, global_begin,
 *               send_lo, recv_lo, send_hi, recv_hi, halo_planes (R),
 *               b0, e0, b1, e1 (boundary planes, swept first; b1 == e1: one
 *               range), i0, i1 (interior)} -- 16 entries; halo entries are
 * -1 on a side without a neighbour. */
int hjb_slab_plan(int64_t n0, int32_t nranks, int32_t rank, int32_t halo, int64_t* out16);
/* NCCL unique id (128 bytes) created on rank 0 and broadcast by the caller
 * (e.g. over torch.distributed); NCCL is loaded with dlopen. */
int hjb_nccl_unique_id(void* out128);
int hjb_comm_create(hjb_context* ctx, int32_t nranks, int32_t rank, const void* unique_id128,
                    hjb_comm** out);
int hjb_comm_destroy(hjb_comm* comm);
/* Peer-store communicator without NCCL (one process per GPU of one node,
 * NVLink peer memory): every per-sweep exchange of the slab solve runs on
 * the devices — the sweep kernels store their boundary planes into the
 * neighbours' halos and the residual all-reduce goes through system-scope
 * atomics into every rank's mailbox; the CFL scan all-reduce, the V_0 halos
 * and the per-solve buffer handles also go through peer memory.  Set up:
 * create, export this rank's control-block IPC handle (64 bytes), all-gather
 * the handles on the host (e.g. torch.distributed with gloo), open them.
 * First order and ENO / TVD-RK stages.  (The NCCL communicator takes the
 * same transport for its sweeps with HJB_SHARD_P2P=1.) */
int hjb_p2p_comm_create(hjb_context* ctx, int32_t nranks, int32_t rank, hjb_comm** out);
int hjb_comm_ctl_handle(hjb_comm* comm, void* out64);
int hjb_comm_open_peers(hjb_comm* comm, const void* handles64xN);
/* solve() over a slab-partitioned 4D grid: init/c/value_out hold this rank's
 * owned planes [begin, end) of `global_grid` (reference layout, device
 * pointers).  Per sweep / RK stage: one launch with the boundary planes
 * first; with an NCCL communicator the halos then travel by NCCL send/recv on
 * a second stream while the interior planes sweep (HJB_SHARD_P2P=1: stored
 * by the kernel into the neighbours, as below); with a peer-store
 * communicator (hjb_p2p_comm_create) the kernel itself stores the boundary
 * planes into the neighbours' halos and the all-reduces run on the devices.
 * Then the all-reduce(max) of max|dV| and the device epilogue; bitwise
 * identical to hjb_solve_dev.  4D fast-path models with constant bounds,
 * first order or ENO/TVD-RK (halo = ENO order), Godunov or Lax-Friedrichs. */
int hjb_solve_sharded_dev(hjb_context* ctx, hjb_comm* comm, const hjb_grid* global_grid,
                          const hjb_model* model, const hjb_dbounds* dbounds,
                          const double* init_slab, const double* c_slab,
                          const hjb_solve_config* cfg, double* value_slab_out,
                          hjb_solve_result* result);
/* The same slab-partitioned solve with `nranks` IN-PROCESS ranks on this
 * context's device: every rank has its own slab buffers, halo planes and
 * loop state, and runs exactly the per-rank plan of hjb_solve_sharded_dev
 * (boundary planes first, interior while the halos travel); halo planes move
 * by device copies on a second stream, the residual all-reduce is a kernel.
 * init/c/value_out are FULL-grid device arrays (reference layout).  Bitwise
 * identical to hjb_solve_dev; verifies and times the multi-rank protocol on
 * one GPU.  1 <= nranks <= 16. */
int hjb_solve_sharded_local_dev(hjb_context* ctx, int32_t nranks, const hjb_grid* grid,
                                const hjb_model* model, const hjb_dbounds* dbounds,
                                const double* init, const double* c,
                                const hjb_solve_config* cfg, double* value_out,
                                hjb_solve_result* result);
/* One sweep restricted to planes [plane_begin, plane_end) of a full grid
 * (device pointers): the slab computation of one rank, for single-device
 * verification of the partition.  Planes of `out` outside the range receive
 * a copy of `value`. */
int hjb_sweep_planes_dev(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
                         const hjb_dbounds* dbounds, const double* value,
                         const double* constraint, int64_t plane_begin, int64_t plane_end,
                         double dt, double* out, double* max_dv);

/* ------------------------------------------- safety-filter queries */
/* SafetyFilter queries (reference safety.hpp:35-107 / safety.cpp:86-127),
 * batched: nq states x[q*nd .. q*nd+nd-1] (nd = grid rank = model state
 * dim) against a value function V on `grid` and the disturbance bounds
 * `dbounds` (constant, or per node on the same grid).
 *  HJB_FILTER_OPTIMAL: SafetyFilter::optimal_control (safety.cpp:86-106):
 *    value = interp_ex(V, x) (grid.cpp:113-131), costate = the multilinear
 *    interpolation of central node gradients (safety.cpp:14-49 with
 *    gradient_at, grid.cpp:141-163), bounds = IntervalField::at (multilinear
 *    per channel, interval_field.cpp:29-31), control / worst disturbance /
 *    degenerate by extremal_inputs (dynamics.cpp:37-63); override = 1,
 *    band = 0.
 *  HJB_FILTER_FILTER: SafetyFilter::filter (safety.cpp:108-127): eta =
 *    max(eta_floor, 0.5 * max_cell_jump(V, x)) (grid.cpp:177-195); when
 *    !out_of_domain and value <= -lambda - eta the performance control
 *    u_perf[q*m ..] passes through (override 0, worst disturbance and
 *    flags 0), otherwise the optimal_control decision; band = eta.
 * A non-finite query is HJB_ERR_INVALID_ARGUMENT ("interp: non-finite
 * query", grid.cpp:95) and no output is defined. */
typedef enum hjb_filter_mode { HJB_FILTER_OPTIMAL = 0, HJB_FILTER_FILTER = 1 } hjb_filter_mode;

typedef struct hjb_filter_config {
  int32_t mode;      /* hjb_filter_mode */
  int32_t reserved;
  double eta_floor;  /* SafetyFilter::Config::eta_floor, default 1e-5 */
  double lambda;     /* contraction level of the filter state */
} hjb_filter_config;

#define HJB_FILTER_OVERRIDE 1   /* FilterDecision::override_active */
#define HJB_FILTER_DEGENERATE 2 /* FilterDecision::degenerate */
#define HJB_FILTER_OOD 4        /* FilterDecision::out_of_domain */

/* Output arrays (any may be NULL): value[nq], band[nq],
 * control[nq][control_dim], worst_disturbance[nq][disturbance_dim],
 * flags[nq] (HJB_FILTER_* bits).  FilterDecision, safety.hpp:14-22. */
typedef struct hjb_filter_out {
  double* value;
  double* band;
  double* control;
  double* worst_disturbance;
  uint8_t* flags;
} hjb_filter_out;

/* Host pointers (V, per-node bounds, x, u_perf and the outputs). */
int hjb_filter_batch(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
                     const hjb_dbounds* dbounds, const double* value, int64_t nq,
                     const double* x, const double* u_perf, const hjb_filter_config* cfg,
                     const hjb_filter_out* out);
/* Device pointers for everything (a value function kept resident in HBM). */
int hjb_filter_batch_dev(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
                         const hjb_dbounds* dbounds, const double* value, int64_t nq,
                         const double* x, const double* u_perf, const hjb_filter_config* cfg,
                         const hjb_filter_out* out);

/* interp_ex batched (reference grid.cpp:113-131): value[q] and
 * out_of_domain[q] (may be NULL) of `field` at x[q*nd ..]; device pointers.
 * A non-finite query is HJB_ERR_INVALID_ARGUMENT. */
int hjb_interp_batch_dev(hjb_context* ctx, const hjb_grid* grid, const double* field,
                         int64_t nq, const double* x, double* value, uint8_t* out_of_domain);

/* min / max over a device field (either output may be NULL): the
 * SafetyFilter's min V* (safety.cpp:60, std::min_element) without a host
 * round trip.  Values are compared as IEEE doubles (NaN-free input). */
int hjb_field_reduce_dev(hjb_context* ctx, int64_t n, const double* field, double* min_out,
                         double* max_out);

/* ---------------------------------------------- device memory helpers */
/* For FFI callers of the _dev entry points (no CUDA runtime of their own):
 * device allocations and copies ordered on the context's stream. */
int hjb_malloc_dev(hjb_context* ctx, uint64_t bytes, void** out);
int hjb_free_dev(hjb_context* ctx, void* ptr);
int hjb_copy_h2d(hjb_context* ctx, void* dst_dev, const void* src_host, uint64_t bytes);
int hjb_copy_d2h(hjb_context* ctx, void* dst_host, const void* src_dev, uint64_t bytes);
int hjb_copy_d2d(hjb_context* ctx, void* dst_dev, const void* src_dev, uint64_t bytes);

/* One Godunov ENO/TVD-RK stage (order 1..3; kind 0 Euler / first stage,
 * 1 RK2 final, 2 RK3 second, 3 RK3 final) restricted to axis-0 planes
 * [plane_begin, plane_end) of a full grid (device pointers): the per-stage
 * slab computation of the sharded high-order solve, for single-device
 * verification.  Planes of `out` outside the range receive a copy of
 * `stage_in`; max_dv = max |out - value_n| over the range.  4D fast-path
 * models. */
int hjb_ho_stage_planes_dev(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
                            const hjb_dbounds* dbounds, const double* stage_in,
                            const double* value_n, const double* constraint, double dt,
                            int32_t order, int32_t kind, int64_t plane_begin, int64_t plane_end,
                            double* out, double* max_dv);

/* ------------------------------------------- GP disturbance bounds */
/* A fitted GpModel (reference gp.hpp:41-75) over one disturbance channel:
 * squared-exponential kernel k(a,b) = signal_var * exp(-0.5 * sum_d
 * ((a_d - b_d) / lengthscales[d])^2) (gp.cpp:22-30) conditioned on n_train
 * inputs (row-major n_train x input_dim), alpha = (K + noise I)^-1 y and the
 * lower Cholesky factor chol (row-major n_train x n_train; only the lower
 * triangle is read) as GpModel::fit stores them (gp.cpp:172-183).
 * n_train = 0 is GpModel::prior (mean 0, variance signal_var).
 * input_dims[0 .. n_dims) are the grid axes the channel's GP conditions on
 * (bounds_on_grid's input_dims[ch]); n_dims must equal input_dim.  All
 * pointers are host memory. */
typedef struct hjb_gp_model {
  int32_t input_dim;
  int32_t n_dims;
  int32_t input_dims[HJB_MAX_DIMS];
  int64_t n_train;
  double signal_var;
  double noise_var;
  double lengthscales[HJB_MAX_DIMS];
  const double* inputs;
  const double* alpha;
  const double* chol;
} hjb_gp_model;

/* bounds_on_grid (reference gp.cpp:211-249): for every channel and node,
 * (mean, latent variance) = GpModel::predict at the node's coordinates
 * along input_dims (gp.cpp:188-208), band = confidence * sqrt(variance +
 * noise_var), lo = mean - band, hi = mean + band.  lo_out[ch] / hi_out[ch]
 * are grid.size doubles each: device pointers (_dev) or host pointers.
 * Errors: "bounds_on_grid: input-dim map does not match GP",
 * "bounds_on_grid: input dim out of grid range" (gp.cpp:219-227), the GP
 * hyperparameter checks of GpHyperparams::validate (gp.cpp:14-21). */
int hjb_gp_bounds_on_grid_dev(hjb_context* ctx, const hjb_grid* grid, int32_t channels,
                              const hjb_gp_model* models, double confidence,
                              double* const* lo_out, double* const* hi_out);
int hjb_gp_bounds_on_grid(hjb_context* ctx, const hjb_grid* grid, int32_t channels,
                          const hjb_gp_model* models, double confidence, double* const* lo_out,
                          double* const* hi_out);
/* GpModel::predict (gp.cpp:188-208) at nq points x[q*input_dim ..] (host):
 * mean[q] and latent variance[q] (host). */
int hjb_gp_predict_batch(hjb_context* ctx, const hjb_gp_model* model, int64_t nq,
                         const double* x, double* mean, double* variance);

/* GpModel::fit (gp.cpp:124-186), host only (O(n^3) once per model update):
 * uniform subsample to max_training, hyperparameters by log-marginal-
 * likelihood search over the reference's 48-candidate grid on a
 * search_subsample subset (HJB_GP_SEARCH) or the prior as given
 * (HJB_GP_FIXED), jitter 1e-8 signal_var, Cholesky, alpha, LML.
 * Caller buffers hold min(n, max_training) training points: inputs_out
 * (x input_dim), alpha_out, chol_out (squared); model_out points at them
 * (input_dims = 0..input_dim-1; set them for bounds_on_grid).  The
 * factorisation is a plain LLT, not Eigen's blocked one: factors match the
 * reference's to rounding, not bitwise. */
typedef enum hjb_gp_policy { HJB_GP_FIXED = 0, HJB_GP_SEARCH = 1 } hjb_gp_policy;
typedef struct hjb_gp_fit_config {
  int32_t policy;               /* hjb_gp_policy, default HJB_GP_SEARCH */
  int32_t prior_n_lengthscales;
  int64_t max_training;         /* 500 */
  int64_t search_subsample;     /* 250 */
  double prior_signal_var;      /* 0.01 */
  double prior_noise_var;       /* 0 */
  double prior_lengthscales[HJB_MAX_DIMS];
} hjb_gp_fit_config;
int hjb_gp_fit(int64_t n, int32_t input_dim, const double* x, const double* y,
               const hjb_gp_fit_config* cfg, double* inputs_out, double* alpha_out,
               double* chol_out, hjb_gp_model* model_out, double* lml_out);

/* Stream of the context (cudaStream_t as void*) and synchronisation. */
void* hjb_context_stream(hjb_context* ctx);
int hjb_context_synchronize(hjb_context* ctx);

/* Number of kernels this context launched since creation (bench evidence). */
int64_t hjb_context_launch_count(hjb_context* ctx);

#ifdef __cplusplus
}
#endif

#endif /* HJB_H_ */
