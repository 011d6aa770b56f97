// hjb_fast4d.cuh — launch interface of the specialised 4D sweep (hjb_fast4d.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "hjb_device.cuh"

namespace hjb {

// Lax-Friedrichs parameters of the 4D model shapes (one input term per
// row): drift, input coefficients and bounds, dissipation (k_fast4d, k_ho4t)
struct LfParams {
  double galpha[4];     // global alpha per axis (scan_alpha)
  int dr_off[4];        // drift table offset of each row (-1: constant drift)
  double dr_const[4];
  double ucoef[4];      // B coefficient of the row's control (shape U(d))
  double dcoef[4];      // C coefficient of the row's disturbance (shape D(d))
  double ulo[3], uhi[3], dlo[3], dhi[3];
  int off_alpha[4];     // LF per-node alpha tables (-1: |drift|)
  // the row's input products with each bound, formed on the host exactly as
  // the Hamiltonian forms them (B u* / C d*: ucoef * ulo[ch] etc.)
  double uprod_lo[4], uprod_hi[4], dprod_lo[4], dprod_hi[4];
  // run-time-shape variant: the control / disturbance channel of each row
  // (-1 none; one input term per row) and whether every channel enters at
  // most one row (its input then follows that row's product sign alone)
  int uch[4], dch[4];
  int single;
};

struct Fast4dArgs {
  CUtensorMap map0;  // V buffer 0 (padded), box = tile + halo rows
  CUtensorMap map1;  // V buffer 1
  CUtensorMap mapc;  // constraint (padded), box = tile rows
  uint32_t vslot_bytes, cslot_bytes, vbox_bytes, cbox_bytes;
  uint32_t n[4];
  uint32_t n3p;  // padded contiguous extent (even)
  double inv[4];
  uint32_t kcells;      // cells per thread along the contiguous axis (2 or 4)
  uint32_t maxthreads;  // CTA thread bound of the variant: (2, 576), (2, 448), (4, 384)
  uint32_t T1, T2, tiles1, tiles2, L, nchunks, items, blocks, threads, consumers, smem;
  // bal = 1: static balanced schedule — CTA b marches the tile-planes
  // [b U / G, (b+1) U / G) of the U = tiles x planes units (at most a few
  // tile pieces each); 0: dynamic items (tile x chunk) off the work counter
  uint32_t bal;
  uint32_t cbeg, cend;  // planes updated (0, 0 = the whole axis-0 extent)
  // sharded slabs: nb (0..2) BOUNDARY chunks [b0, e0), [b1, e1) come first
  // in the item order (bitems = tiles x nb items), then the interior
  // [cbeg, cend) in chunks of L planes.  signal: every consumer warp that
  // finishes a boundary item counts it in st->bnd_done; the count that
  // reaches bnd_target raises st->bnd_flag (the halo transfer waits for it
  // on the stream: cuStreamWaitValue32); an early exit raises it too
  uint32_t nb, b0, e0, b1, e1, bitems, bnd_target;
  int signal;
  // peer-store halos (sharded first order, HJB_SHARD_P2P): a boundary plane
  // i0 in [p2p_src0[s], p2p_src0[s] + p2p_R) is also stored into neighbour
  // s's output buffer (s = 0 lower, 1 upper; NVLink P2P stores, or a
  // same-device pointer for in-process ranks) at its plane i0 - p2p_src0[s] +
  // p2p_dst0[s]; the warp that completes the boundary count then publishes
  // p2p_epoch to the neighbours' flags (system-scope release), which their
  // next stage waits on.  Null p2p_dst[s]: no neighbour on that side.
  double* p2p_dst[2];
  uint32_t p2p_src0[2], p2p_dst0[2], p2p_R;
  unsigned int* p2p_flag[2];
  unsigned int p2p_epoch;
  // max|dV| accumulator of the launch (null: st->maxdv_bits)
  unsigned long long* mdv;
  // padded target set l (TG variant): out = max(c, min(l, stepped))
  const double* target;
  // 1: multi-sweep persistent launch (k_fast4d MS): one cooperative launch
  // runs every sweep of the solve with a grid barrier + device epilogue
  // between sweeps (Godunov, kcells 2 / 576 threads, constant or per-node
  // bounds)
  int ms;
  const double* tab;    // slope tables (staged into shared memory per CTA)
  uint32_t tab_len;     // doubles in tab
  uint32_t tab_off;     // shared-memory byte offset of the staged copy
  int tab_staged;       // 1: tables staged in shared memory, 0: read from global
  int off_pos[4], off_neg[4], off_a[4], off_b[4];
  // rows of the run-time-shape variant (ShapeGen): drift-table axes of each
  // row (gbx < 0: one-axis row, slopes from off_pos / off_neg; else an
  // input-free two-term row, slope = tab[off_a + k_a] + tab[off_b + k_b])
  int gax[4], gbx[4];
  // glin: bit d set when row d has no input (pos == neg == s everywhere):
  // its Godunov flux is s * D+ (s >= 0) or s * D- (the compiled shapes' LIN)
  int glin;
  // gx0: bit d set when row d's slopes vary along x0 (re-formed every plane)
  int gx0;
  // run-time shapes with per-node / plane-varying bounds (pv 1 / 2): the rows
  // with a disturbance term, at most two (slot s -> row gdrow[s], -1 none)
  int gdrow[2];
  const double* c;  // padded constraint
  // constraint that varies along axis 0 only (signed distance to a set in
  // x0, every BASELINE 4D config): c[i0] per plane, the padded field unused
  const double* cplane;
  double* buf0;
  double* buf1;
  const double* src;
  double* dst;
  LoopState* st;
  double dt;
  int loop;  // 0 single step, 1 device loop (fused epilogue), 2 sharded slab sweep
  cudaGraphConditionalHandle handle;
  int use_handle;
  // L2 residency of the constraint (read every sweep, never written): an
  // access-policy window attached to each launch; l2_bytes == 0 disables
  const void* l2_base;
  size_t l2_bytes;
  float l2_hit;
  // programmatic dependent launch (device loop): the kernel waits on
  // griddepcontrol before touching the loop state or V
  int pdl;
  // numerical Hamiltonian: 0 Godunov, 1 Lax-Friedrichs with per-node alpha,
  // 2 Lax-Friedrichs with global alpha (galpha)
  int lf;
  // per-node disturbance bounds that vary along axis 0 only (e.g. GP bounds
  // over x, gp.cpp:211-249): rows with a disturbance term take
  // pos = tab[off_pos] + tab[pv_pt + i0], neg = tab[off_neg] + tab[pv_nt + i0]
  // per plane (Godunov only)
  int pv;  // 1: plane-varying bounds (pv_pt / pv_nt tables); 2: per-node bounds
  int pv_pt[4], pv_nt[4];
  // per-node bounds (pv == 2): padded [n0][n1][n2][n3p] lo / hi of each
  // disturbance row's channel and the row's coefficient; pos / neg =
  // tab[off_pos / off_neg] (drift + controls) + max / min(coef*lo, coef*hi)
  const double* pn_lo[4];
  const double* pn_hi[4];
  double pn_coef[4];
  LfParams lp;
};

// One ENO/TVD-RK stage over a padded 4D grid (k_ho4d, hjb_fast4d.cu): the
// 4D Godunov fast-path models with constant bounds.  Buffers use the padded
// layout of Fast4dArgs; roles follow StepArgs (src_sel / dst_sel / kind).
struct Ho4dArgs {
  uint32_t n[4];
  uint32_t n3p;
  double inv[4];
  uint32_t T1, T2, tiles1, tiles2, L, nchunks, blocks, threads;
  const double* tab;
  int off_pos[4], off_neg[4], off_a[4], off_b[4];
  const double* c;
  const double* cplane;  // as Fast4dArgs::cplane (k_eno3g); null = per-node c
  double* buf0;  // V_n ping-pong (parity = st->iter)
  double* buf1;
  double* stage1;
  double* stage2;
  int src_sel, dst_sel, kind, final_stage, order;
  // 1: solve loop (buffer parity from st, fused epilogue on the final stage);
  // 2: sharded slab (parity from st, the caller all-reduces and runs the
  //    epilogue); 0: one stage on explicit buffers (xsrc, xvn -> xdst)
  int loop;
  uint32_t cbeg, cend;  // planes updated (0, 0 = all)
  uint32_t nb, b0, e0, b1, e1, bitems, bnd_target;  // boundary chunks first (as Fast4dArgs)
  int signal;
  unsigned long long* mdv;       // max|dV| accumulator (null: st->maxdv_bits)
  // pmode 1: the V_n buffer parity is `parity` (sharded loop: the loop
  // state's iteration count advances concurrently on the comm stream)
  int pmode, parity;
  const double* xsrc;
  const double* xvn;
  double* xdst;
  LoopState* st;
  double dt;
  cudaGraphConditionalHandle handle;
  int use_handle;
  // TMA-staged variant (k_ho4t): tensor maps of the four possible stage
  // inputs (buf0, buf1, stage1, stage2) with a box of tile + R-row halo in
  // i1 and i2, the shared-memory ring of those boxes, its depth
  CUtensorMap mapv[4];
  uint32_t vbox_bytes, vslot_bytes, ring, smem, tma;
  uint32_t T3, H3, segs;  // axis-3 segment per tile (even), its box halo (even >= R), segments per row
  uint32_t kc;            // cells per thread along axis 3 (1 or 2)
  // numerical Hamiltonian (k_ho4t): 0 Godunov, 1 / 2 Lax-Friedrichs per-node /
  // global alpha, ghost faces replicated from the nearest interior face
  int lf;
  LfParams lp;
  // 1: ENO3 Godunov stage in k_eno3g (face-shared choices, patched boxes,
  //    three barriers per ring slot); 0: k_ho4t
  int eno3g;
  // set before ho4d_config: keep k_eno3g's 512-thread tiling (the slab
  // solves, whose peer-store instantiations have that bound only)
  int tb_fixed;
  // run-time row shapes (k_ho4t<ShapeGen>, set before ho4d_config, which
  // then keeps k_eno3g off): the rows' table axes (no row on x0) and the
  // input-free rows, as Fast4dArgs::gax / gbx / glin
  int gen;
  int gax[4], gbx[4], glin;
  // peer-store halos of the sharded stages (as Fast4dArgs::p2p_*): a
  // boundary plane's stores (ghost cells included) also go into the
  // neighbour's same stage buffer
  double* p2p_dst[2];
  uint32_t p2p_src0[2], p2p_dst0[2], p2p_R;
  unsigned int* p2p_flag[2];
  unsigned int p2p_epoch;
  // ghost widths of the stage-buffer layout [n0][n1 + 2gh][n2 + 2gh][n3p + 2g3]
  // (k_eno3g: 3 and 4; k_ho4t / k_ho4d: 0, the plain padded layout)
  uint32_t gh, g3;
  // k_eno3g: tile-only boxes (T1 x T2 x T3, no halo) of the four stage buffers
  // (loop == 0: [0] the stage input, [1] V_n) and of c; each ring slot holds
  // the V box of plane q, c and V_n of plane q and the stage input of plane
  // q + 4 (the axis-0 window's next plane), tbox_slot bytes apart
  CUtensorMap mapt[4];
  CUtensorMap mapc;
  uint32_t tbox_bytes, tbox_slot;
};
void ho4d_config(const DevGrid& g, int sms, Ho4dArgs& a);
// fill mapv[] for the current buffers (k_ho4t); returns cudaErrorNotSupported
// when the driver entry point is unavailable
cudaError_t ho4d_make_maps(Ho4dArgs& a);
cudaError_t launch_ho4d(const Ho4dArgs& a, int shape, cudaStream_t s);
// elements per axis-0 plane of the stage buffers (ghost layout of `a`), and
// reference layout (planes of n1 * n2 * n3) <-> stage-buffer layout
uint64_t ho4d_plane(const Ho4dArgs& a);
cudaError_t ho4d_pad(const double* in, double* out, uint32_t planes, const Ho4dArgs& a,
                     cudaStream_t s);
cudaError_t ho4d_unpad(const double* in, double* out, uint32_t planes, const Ho4dArgs& a,
                       cudaStream_t s);

// Model shape id for the fast path (0..2 compiled shapes, kShapeGen run-time
// rows), or -1 when the generic kernel must run (rank != 4, per-node bounds,
// a two-term row with inputs, inputs not matching the shape under LF, ...).
// scheme: 0 Godunov, 1 LF per-node alpha, 2 LF global alpha.
int fast4d_shape(const DevGrid& g, const DevModel& m, int scheme);
// Shape id of the run-time-shape Godunov variant (k_fast4d<ShapeGen>): a
// model whose rows are admissible for the fast path (one-axis rows with any
// inputs, input-free two-term rows, on any axes; rows on x0 re-form their
// slopes every plane) but match none of the compiled shapes.  First order, Godunov, constant bounds, no target set;
// the high-order and Lax-Friedrichs paths treat it as -1 (generic kernel).
constexpr int kShapeGen = 3;
// Fast4dArgs::gax / gbx of the run-time-shape variant from the model rows
void fast4d_gen_rows(const DevModel& m, Fast4dArgs& a);
// Godunov fast-path shape for PER-NODE bounds (rows not folded); -1 if none.
// Rows with a disturbance term must be exactly the shape's D rows, one
// term each.  Bounds varying along axis 0 only run the plane-table variant
// (pv == 1), any other per-node field the per-node variant (pv == 2); the
// caller checks which on the device.
int fast4d_shape_pv(const DevGrid& g, const DevModel& m);
void fast4d_config(const DevGrid& g, int sms, Fast4dArgs& a);
// Configure a launch (fast4d_config / ho4d_config done) for a slab: the
// boundary planes [b0, e0) and, when b1 < e1, [b1, e1) as the FIRST items
// (one chunk per range and tile), then the interior [i0, i1) chunked as
// fast4d_chunks / ho4d_chunks would (i0 == i1: boundary only).
void fast4d_bfirst(Fast4dArgs& a, int sms, uint32_t b0, uint32_t e0, uint32_t b1, uint32_t e1,
                   uint32_t i0, uint32_t i1);
void ho4d_bfirst(Ho4dArgs& a, int sms, uint32_t b0, uint32_t e0, uint32_t b1, uint32_t e1,
                 uint32_t i0, uint32_t i1);
// Re-chunk a configured launch over its plane range [cbeg, cend) (the
// chunking fast4d_config / ho4d_config apply)
void fast4d_chunks(Fast4dArgs& a, int sms);
void ho4d_chunks(Ho4dArgs& a, int sms);
cudaError_t launch_fast4d(const Fast4dArgs& a, int shape, cudaStream_t s);
// Encode the three TMA tensor maps for the padded buffers (driver entry point
// fetched through the runtime; no libcuda link dependency).
cudaError_t fast4d_make_maps(Fast4dArgs& a, double* buf0, double* buf1, const double* c);
// Persisting-L2 carve-out for the constraint of a solve: sets the device
// limit and fills a.l2_*; l2_release() undoes it.  No-op (returns false)
// when the constraint does not fit the carve-out or HJB_L2PIN=0.
bool l2_pin(int device, Fast4dArgs& a, const void* base, size_t bytes);
void l2_release(Fast4dArgs& a);
cudaError_t launch_epilogue(LoopState* st, cudaGraphConditionalHandle handle, int use_handle,
                            cudaStream_t s, unsigned long long* slot = nullptr);
cudaError_t launch_pad4(const double* in, double* out, uint64_t rows, uint32_t n3, uint32_t n3p,
                        cudaStream_t s);
cudaError_t launch_unpad4(const double* in, double* out, uint64_t rows, uint32_t n3,
                          uint32_t n3p, cudaStream_t s);

}  // namespace hjb
