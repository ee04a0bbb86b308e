// hsde_kernels.cuh -- sm_100a fp64 kernels of the HSDE-ADMM hot path.
//
// One ADMM iteration (reference: chordalsdp/solver.py:375-395) on the
// compressed layout [x n_c | s n_d | y m | v n_d | tau] is, in launch order:
//
//   k_rhs      per covered coordinate l: pull-scatter of the clique slots
//              covering l (graphs.py:249-252, atomic-free) and
//              t0 = P^{-1} (r - A' rho_y)  (solver.py:222-231 without the A' term)
//   k_spmv_seg row-split CSR SpMV q0 = A t0 (solver.py:232 `dp.A @ t`)
//   k_schur    g = S^{-1} (q0 - rho_y) with the cached inverse
//   k_ua       ua = t0 - P^{-1} A' g + block partials of c.ua
//
//   With S = I + A P^{-1} A' this is the reference's block elimination
//   (t = t0 + P^{-1} A' rho_y, q' = S^{-1} A t, ua = t - P^{-1} A' q',
//   solver.py:231-235) rearranged: q' = g + rho_y, ua = t0 - P^{-1} A' g and
//   uy = rho_y - A ua = rho_y - q' = -g.  Two passes over A instead of three.
//   k_scalars  one CTA: zeta.u12, shift, tau/kappa, y update (solver.py:315-317,
//              388-394), next iteration's rho_y
//   k_cone     per clique: ub, uv, relaxation, PSD projection (symmat.py:153-165)
//              by team-parallel cyclic Jacobi in shared memory, s/z/v update
//   k_xupd     per covered coordinate: x / w_x update (solver.py:388-394)
//
// All reductions are fixed-order (block partials + ordered final sum), so
// runs are bitwise reproducible.  No atomics on the data path.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <type_traits>

namespace hsde {

constexpr int kBlock = 256;          // threads per CTA for streaming kernels
constexpr int kMaxParts = 4096;      // block partials for dot products
constexpr int kSegNnz = 2048;        // nnz per CSR segment (row-split SpMV)
constexpr int kMaxSweeps = 40;       // Jacobi sweep cap

// scalar slots in the device scalar buffer
enum Scal {
  S_ATAU = 0,   // a_tau = tau + kappa at the start of the iteration
  S_SHIFT = 1,  // rank-one shift (solver.py:315)
  S_ZU = 2,     // zeta . u12 before the shift
  S_UTAU = 3,   // u_hat tau (affine)
  S_COUNT = 16
};

struct DevProblem {
  int m, n_c, p;
  int64_t n_d, nnz, total;
  // A: CSR (rows = constraints) and CSC (= CSR of A') over covered columns
  const int64_t *a_rp;
  const int *a_col;
  const double *a_val;
  const int64_t *at_cp;
  const int *at_row;
  const double *at_val;
  // row-split segments of the CSR
  int nseg;
  const int *seg_row;
  const int64_t *seg_beg;
  const int *row_seg;  // [m+1] first segment of each row
  // cover lists: covered -> slots (ascending slot = bincount order)
  const int *cov_ptr;  // [n_c+1]
  const int *cov_slot; // [n_d]
  const int *slot_cov; // [n_d]
  int n_heavy;         // covered coordinates with > kHeavy slots
  const int *heavy;    // [n_heavy]
  // sharding; single GPU: n_sep = 0, owned = null
  int n_sep;           // global separator count |S|
  int n_sep_local;     // separator coordinates this shard touches
  const int *sep_of;   // [n_c] position in S or -1 (null when n_sep == 0)
  const int *sep_local;// [n_sep_local] local covered index
  const int *sep_pos;  // [n_sep_local] position in S
  const unsigned char *owned;  // [n_c] 1 if this shard owns the coordinate (null: all)
  int lead;            // 1 on the shard that contributes replicated terms (y, tau)
  const int64_t *cl_off;
  const int *cl_size;
  // symmetric half passes: when every column of A equals its
  // mirror's (A_ij = A_ji, the symmetric constraint matrices of an SDP), the
  // two A passes run over one column per mirror pair {l, mirror(l)}:
  //   A t = sum_pairs A_l (t_l + t_mirror),   (A' g)_l = (A' g)_mirror
  int half;              // 1: enabled
  int n_pair;
  const int *pair_l, *pair_m;  // [n_pair] representative (l <= mirror) and mirror
  int n_slice;           // SELL-32 slices of 32 pairs (A' g), pairs sorted by length
  const int64_t *sl_beg; // within windows of kSellSigma; [n_slice + 1]; element k of
  const uint16_t *sl_row;// lane j at sl_beg[s] + 32 k + j
  const double *sl_val;
  const int *sl_pl, *sl_pm;  // [n_pair] the pair (l, mirror) of SELL position q
  int rt_tile, rt_split;  // pairs per row-SELL tile (<= kRowTile), CTAs per tile
  int rt_ntile, rt_G;    // row-SELL tiles of rt_tile pairs x groups of 32 rows (A t),
  const int64_t *rt_beg; // owned pairs only, rows sorted by length within a tile;
  const uint16_t *rt_col;// [rt_ntile * rt_G + 1]; column within the tile
  const double *rt_val;
  const int *rt_row;     // [rt_ntile * m] row of tile position g * 32 + j
  // data of the iterated (normalised) problem
  const double *c, *b, *p_inv;
  // Schur inverse: dense m x m (row-major, symmetric) or diagonal m
  int schur_diag;
  const double *sinv;
  // M^{-1} zeta, layout [x n_c | s n_d | y m | v n_d]
  const double *mz;
  double zeta_scale, zmz, alpha;
};

struct DevState {
  double *u, *w;  // [total]
};

struct DevWork {
  double *t, *ua;      // [n_c]
  double *rtpart;      // [m * rt_ntile] tile partials of A t (half passes)
  double *xq;          // [n_pair] t_l + t_mirror (half passes)
  double *ry;          // [m] rho_y of the current iteration
  double *qseg;        // [nseg]
  double *qp;          // [m]
  double *uy;          // [m]
  double *part;        // [kMaxParts]
  double *scal;        // [S_COUNT]
  int *err;            // [1] bit 0: non-finite eigenvalue
  double *vstore;      // [n_d] eigenvectors of the last projection (warm start)
  int *vvalid;         // [p]   vstore holds a valid basis for clique k
  int *sweeps;         // [p]   Jacobi sweeps of the last projection (stats)
  double *sepbuf;      // [n_sep] separator partials (all-reduced)
  double *qbuf;        // [m]     partial A t (all-reduced)
  double *red;         // [8]     scalar partials (all-reduced)
  int *handoff;        // [p]     1: stage-1 Jacobi handed the clique to the refinement kernel
  int *cstate;         // [p]     k_cone_split outcome (SplitState), read by k_cone_block
  int *ckey;           // [p]     predicted cost of the clique's next projection (schedule key)
  int *corder;         // [p]     CTA-plan clique ids, refresh candidates first (k_scalars)
  const int *cta_ids;  // CTA-plan clique ids (plan order) to be scheduled into corder, or null
  int cta_n;
  double *xarg;        // [n_d]   k_cone_split -> k_cone_block hand-off (B = Vt X Vt'); cold path: raw X
  int *ccur, *cnext;   // [p]     CTA cliques: 1 = cold path this / next iteration (k_scalars copies next -> cur)
  double *dbg;         // [64]    Jacobi off-norm history of one clique (diagnostics)
  int dbg_clique;
};

__device__ __forceinline__ bool owns(const DevProblem &P, int l) {
  return P.owned == nullptr || P.owned[l];
}

// ---------------------------------------------------------------------------
// helpers

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Programmatic dependent launch (the hot chain k_rhs -> ... -> k_scalars of one
// stream): a kernel launched with programmatic stream serialisation may be
// scheduled while its predecessor drains; pdl_wait() returns once the
// predecessor grid has completed and its writes are visible (a no-op for a
// normal launch), pdl_trigger() lets the successor's launch begin.  Every
// thread calls pdl_wait() first, on every path, so completion stays transitive
// along the chain.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Fixed-order block sum; result valid in thread 0.  `sh` holds >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double *sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    r = lane < nw ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

__device__ __forceinline__ double relax(double uhat, double uold, double alpha) {
  // solver.py:388-390: u_hat *= alpha; u_hat += (1 - alpha) * u
  return alpha != 1.0 ? alpha * uhat + (1.0 - alpha) * uold : uhat;
}

// ---------------------------------------------------------------------------
// k_rhs: r0 = 0.5 H'(rho_s - rho_v) + H' rho_v + rho_x ; t0 = P^{-1} r0
// (solver.py:222-231 less the A' rho_y term, folded into k_schur).  FROM_STATE: rho comes from the state u + w and a_tau
// (affine_project :300-301 fused); otherwise from explicit vectors.

// Covered coordinates with more than kHeavy covering slots (e.g. the arrow
// head of a block-arrow pattern: 400 cliques share it) get a warp each;
// the rest a thread each.  Grid = [light blocks | heavy blocks].
constexpr int kHeavy = 32;

template <bool FROM_STATE>
__device__ __forceinline__ void rhs_slot(const DevProblem &P, const DevState &S, const double *rs,
                                         const double *rv, int j, double &sg, double &sv) {
  const int64_t so = P.n_c, vo = P.n_c + P.n_d + P.m;
  double as, av;
  if (FROM_STATE) {
    as = S.u[so + j] + S.w[so + j];
    av = S.u[vo + j] + S.w[vo + j];
  } else {
    as = rs[j];
    av = rv[j];
  }
  sg += as - av;
  sv += av;
}

template <bool FROM_STATE>
__device__ __forceinline__ void rhs_finish(const DevProblem &P, const DevState &S, const DevWork &W,
                                           const double *rx, double atau, int l, double sg, double sv) {
  if (P.n_sep && P.sep_of[l] >= 0) {  // separator: partial, finished after the all-reduce
    W.sepbuf[P.sep_of[l]] = sg * 0.5 + sv;
    return;
  }
  const double rx_l = FROM_STATE ? (S.u[l] + S.w[l]) - atau * P.c[l] : rx[l];
  const double r = (sg * 0.5 + sv) + rx_l;
  W.t[l] = r * P.p_inv[l];
}

// Grid = [heavy blocks | light blocks]: the few heavy warps start first.  Light
// threads take two coordinates per step with their dependent loads (cover
// range -> slot -> slot values) interleaved.
template <bool FROM_STATE>
__global__ void __launch_bounds__(kBlock) k_rhs(DevProblem P, DevState S, DevWork W,
                                                const double *rx, const double *rs,
                                                const double *rv, int nb_heavy) {
  pdl_wait();
  double atau = 0.0;
  if (FROM_STATE) atau = S.u[P.total - 1] + S.w[P.total - 1];
  if ((int)blockIdx.x >= nb_heavy) {
    const int stride = ((int)gridDim.x - nb_heavy) * blockDim.x;
    for (int l = ((int)blockIdx.x - nb_heavy) * blockDim.x + threadIdx.x; l < P.n_c; l += 2 * stride) {
      int lq[2], jb[2], je[2];
      lq[0] = l;
      lq[1] = l + stride < P.n_c ? l + stride : -1;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        jb[q] = lq[q] >= 0 ? P.cov_ptr[lq[q]] : 0;
        je[q] = lq[q] >= 0 ? P.cov_ptr[lq[q] + 1] : 0;
      }
      int j0[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) j0[q] = (je[q] > jb[q] && je[q] - jb[q] <= kHeavy) ? P.cov_slot[jb[q]] : -1;
      double sg[2] = {0.0, 0.0}, sv[2] = {0.0, 0.0};
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (j0[q] >= 0) rhs_slot<FROM_STATE>(P, S, rs, rv, j0[q], sg[q], sv[q]);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (lq[q] < 0 || je[q] - jb[q] > kHeavy) continue;
        for (int e = jb[q] + 1; e < je[q]; ++e) rhs_slot<FROM_STATE>(P, S, rs, rv, P.cov_slot[e], sg[q], sv[q]);
        rhs_finish<FROM_STATE>(P, S, W, rx, atau, lq[q], sg[q], sv[q]);
      }
    }
    pdl_trigger();
    return;
  }
  // heavy coordinates: one warp each, lanes stride the slot list
  const int lane = threadIdx.x & 31;
  const int hw = (int)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (hw >= P.n_heavy) {
    pdl_trigger();
    return;
  }
  const int l = P.heavy[hw];
  double sg = 0.0, sv = 0.0;
  for (int e = P.cov_ptr[l] + lane; e < P.cov_ptr[l + 1]; e += 32)
    rhs_slot<FROM_STATE>(P, S, rs, rv, P.cov_slot[e], sg, sv);
  sg = warp_sum(sg);
  sv = warp_sum(sv);
  if (lane == 0) rhs_finish<FROM_STATE>(P, S, W, rx, atau, l, sg, sv);
  pdl_trigger();
}

// t of the separator coordinates once their pull-scatter partials are all-reduced
template <bool FROM_STATE>
__global__ void k_sep_finish(DevProblem P, DevState S, DevWork W, const double *rx) {
  double atau = 0.0;
  if (FROM_STATE) atau = S.u[P.total - 1] + S.w[P.total - 1];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n_sep_local; i += gridDim.x * blockDim.x) {
    const int l = P.sep_local[i];
    const double rx_l = FROM_STATE ? (S.u[l] + S.w[l]) - atau * P.c[l] : rx[l];
    W.t[l] = (W.sepbuf[P.sep_pos[i]] + rx_l) * P.p_inv[l];
  }
}

__global__ void k_zero(double *x, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    x[k] = 0.0;
}

// rho_y for the first iteration after a state change: (u_y + w_y) + a_tau b
__global__ void k_prep_ry(DevProblem P, DevState S, DevWork W) {
  const double atau = S.u[P.total - 1] + S.w[P.total - 1];
  const int64_t yo = P.n_c + P.n_d;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m; i += gridDim.x * blockDim.x)
    W.ry[i] = (S.u[yo + i] + S.w[yo + i]) + atau * P.b[i];
}

// ---------------------------------------------------------------------------
// Row-split CSR SpMV: one warp per segment of <= kSegNnz nonzeros of one row.

__global__ void __launch_bounds__(kBlock) k_spmv_seg(DevProblem P, const double *__restrict__ x,
                                                      double *__restrict__ qseg) {
  const int lane = threadIdx.x & 31;
  const int seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (seg >= P.nseg) return;
  const int row = P.seg_row[seg];
  const int64_t b = P.seg_beg[seg];
  const int64_t e = min(b + (int64_t)kSegNnz, P.a_rp[row + 1]);
  double acc = 0.0;
  for (int64_t k = b + lane; k < e; k += 32) acc += P.a_val[k] * __ldg(x + P.a_col[k]);
  acc = warp_sum(acc);
  if (lane == 0) qseg[seg] = acc;
}

// g = S^{-1} (q0 - rho_y).  Every CTA rebuilds q0 - rho_y from the segment
// partials (ordered) into shared memory, then one warp per output row of the
// symmetric inverse.
constexpr int kSchurSplit = 4;  // warps per row of the dense S^-1 apply

__global__ void __launch_bounds__(kBlock) k_schur(DevProblem P, const double *__restrict__ qseg,
                                                   const double *__restrict__ qfull,
                                                   const double *__restrict__ ry,
                                                   double *__restrict__ g) {
  extern __shared__ double qs[];
  pdl_wait();
  for (int i = threadIdx.x; i < P.m; i += blockDim.x) {
    double q = 0.0;
    if (qfull) {
      q = qfull[i];  // already reduced (sharded)
    } else {
      for (int s = P.row_seg[i]; s < P.row_seg[i + 1]; ++s) q += qseg[s];
    }
    qs[i] = q - ry[i];
  }
  __syncthreads();
  if (P.schur_diag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m; i += gridDim.x * blockDim.x)
      g[i] = qs[i] * P.sinv[i];
    pdl_trigger();
    return;
  }
  // kSchurSplit warps per row (contiguous column segments), rows in pairs per
  // CTA: enough warps in flight for a latency-bound m x m apply; partials
  // summed in fixed order
  __shared__ double part[kBlock / 32];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int rows_per_cta = (kBlock / 32) / kSchurSplit, seg = wq % kSchurSplit;
  const int seg_len = (P.m + kSchurSplit - 1) / kSchurSplit;
  const int j0 = seg * seg_len, j1 = min(P.m, j0 + seg_len);
  for (int base = blockIdx.x * rows_per_cta; base < P.m; base += gridDim.x * rows_per_cta) {
    const int i = base + wq / kSchurSplit;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    if (i < P.m) {
      // S^-1 (m^2 doubles) is read with cached loads: it stays in L2 across
      // iterations while the A passes stream with evict-first loads
      const double *row = P.sinv + (int64_t)i * P.m;
      int j = j0 + lane;
      for (; j + 96 < j1; j += 128) {
        double r4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) r4[u] = __ldg(row + j + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] += r4[u] * qs[j + 32 * u];
      }
      for (; j < j1; j += 32) a[0] += __ldg(row + j) * qs[j];
    }
    const double acc = warp_sum((a[0] + a[1]) + (a[2] + a[3]));
    if (lane == 0) part[wq] = acc;
    __syncthreads();
    if (seg == 0 && lane == 0 && i < P.m) {
      double t = 0.0;
      for (int q = 0; q < kSchurSplit; ++q) t += part[wq + q];
      g[i] = t;
    }
    __syncthreads();
  }
  pdl_trigger();
}

// ua = t0 - P^{-1} (A' g)  (solver.py:232-235, see the header); WITH_DOT: block
// partials of c.ua
template <bool WITH_DOT>
__global__ void __launch_bounds__(kBlock) k_ua(DevProblem P, DevWork W, const double *__restrict__ qp) {
  __shared__ double sh[32];
  double dot = 0.0;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < P.n_c; l += gridDim.x * blockDim.x) {
    double atq = 0.0;
    const int64_t cb = P.at_cp[l], ce = P.at_cp[l + 1];
    for (int64_t e = cb; e < ce; ++e) atq += P.at_val[e] * __ldg(qp + P.at_row[e]);
    const double ua = W.t[l] - atq * P.p_inv[l];
    W.ua[l] = ua;
    if (WITH_DOT && owns(P, l)) dot += P.c[l] * ua;
  }
  if (WITH_DOT) {
    dot = block_sum(dot, sh);
    if (threadIdx.x == 0) W.part[blockIdx.x] = dot;
  }
}

// ---------------------------------------------------------------------------
// Half passes over mirror pairs (P.half).  Both stream A in 16-bit-index
// SELL layouts: every load is a coalesced 32-lane access.

// One lane's dot product over a SELL-32 slice: entries k, k+32, ... < e of
// (val, 16-bit index into the shared vector xs), two accumulators.  (Issuing
// four entries' loads before any use, four accumulators, measured slower:
// k_ua_half 76 -> 100 us, k_spmv_half 74 -> 85 us on config 4.)
__device__ __forceinline__ double sell_dot(const double *__restrict__ val, const uint16_t *__restrict__ idx,
                                           const double *xs, int64_t k, int64_t e) {
  double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
  for (; k + 32 < e; k += 64) {
    a0 += __ldcs(val + k) * xs[__ldcs(idx + k)];
    a1 += __ldcs(val + k + 32) * xs[__ldcs(idx + k + 32)];
  }
  if (k < e) a0 += __ldcs(val + k) * xs[__ldcs(idx + k)];
  return a0 + a1;
}

constexpr int kRowTile = 4096;  // pairs per row-SELL tile (16-bit column index)
constexpr int kSellSigma = 1024;  // SELL-32 sorting window (pairs)
constexpr int kRowTileDefault = 2048;  // default P.rt_tile
constexpr int kRowTileSplit = 2;  // default P.rt_split: CTAs per tile (row groups split among them)
// (config 4, m = 1000: 4096 x 4 -> 2048 x 2 took k_spmv_half from 74 to 67 us; 16 KB of
// staged pair values per CTA lets 2x more CTAs reside, 1024 x 4 / 2048 x 4 / x 8 measured 67-70 us)

// pair values x_q = t_l + t_mirror (t_l on the diagonal)
__global__ void k_pair_sum(DevProblem P, const double *__restrict__ t, double *__restrict__ xq) {
  pdl_wait();
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < P.n_pair; q += gridDim.x * blockDim.x) {
    const int l = P.pair_l[q], mm = P.pair_m[q];
    xq[q] = mm != l ? t[l] + t[mm] : t[l];
  }
  pdl_trigger();
}

// q0 partials: part[r * ntile + tile] = sum over the tile's owned pairs of
// A_r,pair x_pair; the tile's pair values are staged in shared memory.
// PAIRS: x_pair = t_l + t_mirror formed while staging (no separate pair-sum pass)
// (8 CTAs per SM: 32 registers; three more cost a quarter of the occupancy and
// 19 us of this HBM-bound pass)
template <bool PAIRS>
__global__ void __launch_bounds__(kBlock, 8) k_spmv_half(DevProblem P, const double *__restrict__ xq,
                                                       double *__restrict__ part) {
  extern __shared__ double xs[];  // [P.rt_tile]
  pdl_wait();
  const int tile = blockIdx.x / P.rt_split, rr = blockIdx.x - tile * P.rt_split;
  const int q0 = tile * P.rt_tile, wn = min(P.rt_tile, P.n_pair - q0);
  if (PAIRS) {
    for (int i0 = threadIdx.x; i0 < wn; i0 += 4 * blockDim.x) {  // 4 pairs in flight per thread
      int l[4], mm[4];
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = min(i0 + u * (int)blockDim.x, wn - 1);
        l[u] = P.pair_l[q0 + i];
        mm[u] = P.pair_m[q0 + i];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = xq[l[u]];
        b[u] = mm[u] != l[u] ? xq[mm[u]] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u * (int)blockDim.x < wn) xs[i0 + u * blockDim.x] = a[u] + b[u];
    }
  } else {
    for (int i = threadIdx.x; i < wn; i += blockDim.x) xs[i] = xq[q0 + i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int G = P.rt_G;
  for (int gr = rr * nw + (threadIdx.x >> 5); gr < G; gr += P.rt_split * nw) {
    const int64_t b = P.rt_beg[(int64_t)tile * G + gr], e = P.rt_beg[(int64_t)tile * G + gr + 1];
    const double acc = sell_dot(P.rt_val, P.rt_col, xs, b + lane, e);
    const int rq = gr * 32 + lane;
    if (rq < P.m) part[(int64_t)P.rt_row[(int64_t)tile * P.m + rq] * P.rt_ntile + tile] = acc;
  }
  pdl_trigger();
}

// q0_r = ordered sum of the row's tile partials (one warp per row)
__global__ void k_rowsum_tiles(DevProblem P, const double *__restrict__ part, double *__restrict__ q) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < P.m; r += warps) {
    double a = 0.0;
    for (int t = lane; t < P.rt_ntile; t += 32) a += part[(int64_t)r * P.rt_ntile + t];
    a = warp_sum(a);
    if (lane == 0) q[r] = a;
  }
  pdl_trigger();
}

// ua = t0 - P^{-1} A' g over mirror pairs (one warp per SELL slice, lane =
// pair), g staged in shared memory; WITH_DOT: block partials of c.ua (owned)
template <bool WITH_DOT>
__global__ void __launch_bounds__(kBlock) k_ua_half(DevProblem P, DevWork W, const double *__restrict__ g) {
  extern __shared__ double sg[];
  __shared__ double sh[32];
  pdl_wait();
  for (int i = threadIdx.x; i < P.m; i += blockDim.x) sg[i] = g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  double dot = 0.0;
  for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < P.n_slice; sl += warps) {
    const int64_t b = P.sl_beg[sl], e = P.sl_beg[sl + 1];
    const double atg = sell_dot(P.sl_val, P.sl_row, sg, b + lane, e);
    const int q = sl * 32 + lane;
    if (q < P.n_pair) {
      const int l = P.sl_pl[q], mm = P.sl_pm[q];
      const double ul = W.t[l] - atg * P.p_inv[l];
      W.ua[l] = ul;
      if (WITH_DOT && owns(P, l)) dot += P.c[l] * ul;
      if (mm != l) {
        const double um = W.t[mm] - atg * P.p_inv[mm];
        W.ua[mm] = um;
        if (WITH_DOT && owns(P, mm)) dot += P.c[mm] * um;
      }
    }
  }
  if (WITH_DOT) {
    dot = block_sum(dot, sh);
    if (threadIdx.x == 0) W.part[blockIdx.x] = dot;
  }
  pdl_trigger();
}

// ---------------------------------------------------------------------------
// k_scalars: one CTA.  zeta.u12 = c.ua - b.uy (zeta = (c, 0, -b, 0),
// solver.py:264), shift (:315), u_hat tau (:317), relaxation (:388-390), tau/kappa
// projection and dual update (:391-394), y update, next rho_y.

__global__ void __launch_bounds__(1024) k_scalars(DevProblem P, DevState S, DevWork W, int nparts,
                                                  int exact_uy, const double *__restrict__ auy,
                                                  const double *__restrict__ cua_red) {
  __shared__ double sh[32];
  __shared__ double bc[4];
  pdl_wait();
  const int64_t yo = P.n_c + P.n_d;
  // k_cone_split schedule (hsde_split.cuh): ids and keys loaded first, the
  // partition done at the end (their latency hides behind the sums)
  const bool sched = W.cta_ids != nullptr;
  int my_id = 0, my_key = 0;
  if (sched && (int)threadIdx.x < W.cta_n) {
    my_id = W.cta_ids[threadIdx.x];
    my_key = W.ckey[my_id];
  }
  double a = 0.0;
  if (!cua_red)
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) a += W.part[i];
  double cua = block_sum(a, sh);
  if (cua_red) cua = cua_red[0];  // all-reduced over shards (thread 0 uses it)
  double bu = 0.0;
  for (int i = threadIdx.x; i < P.m; i += blockDim.x) {
    // uy = rho_y - A ua (solver.py:240-241); identity rho_y - A ua = -g unless exact
    const double uy = exact_uy ? W.ry[i] - auy[i] : -W.qp[i];
    W.uy[i] = uy;
    bu += P.b[i] * uy;
  }
  const double buy = block_sum(bu, sh);
  if (threadIdx.x == 0) {
    const double tau = S.u[P.total - 1], kappa = S.w[P.total - 1];
    const double atau = tau + kappa;
    const double zu = cua - buy;
    const double shift = zu / P.zeta_scale;
    const double utau = atau + (zu - shift * P.zmz);
    const double utr = relax(utau, tau, P.alpha);
    const double arg = utr - kappa;
    const double tnew = arg > 0.0 ? arg : 0.0;
    const double knew = (kappa - utr) + tnew;
    S.u[P.total - 1] = tnew;
    S.w[P.total - 1] = knew;
    W.scal[S_SHIFT] = shift;
    W.scal[S_ZU] = zu;
    W.scal[S_UTAU] = utau;
    bc[0] = shift;
    bc[1] = tnew + knew;
  }
  __syncthreads();
  const double shift = bc[0], atau_next = bc[1];
  for (int i = threadIdx.x; i < P.m; i += blockDim.x) {
    const double uh = W.uy[i] - shift * P.mz[yo + i];
    const double yold = S.u[yo + i], wy = S.w[yo + i];
    const double ur = relax(uh, yold, P.alpha);
    const double yn = ur - wy;
    const double wn = (wy - ur) + yn;
    S.u[yo + i] = yn;
    S.w[yo + i] = wn;
    W.ry[i] = (yn + wn) + atau_next * P.b[i];
  }
  if (sched && W.ccur)  // this iteration's split / cold decision (hsde_cold.cuh)
    for (int i = threadIdx.x; i < W.cta_n; i += blockDim.x) {
      const int id = W.cta_ids[i];
      W.ccur[id] = W.cnext[id];
    }
  if (sched) {
    // the cliques with key 1 (likely to need a Jacobi refresh) first, plan order
    // otherwise: a stable partition by ballots, blockDim.x ids per chunk
    __shared__ int cnt[32];
    int base1 = 0, base0 = 0;
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5, nwq = blockDim.x >> 5;
    if (W.cta_n > (int)blockDim.x) {  // multi-chunk plans: count the key-1 ids first
      int n1 = 0;
      for (int i = threadIdx.x; i < W.cta_n; i += blockDim.x) n1 += W.ckey[W.cta_ids[i]] != 0;
      base0 = (int)block_sum((double)n1, sh);
      if (threadIdx.x == 0) bc[2] = base0;
      __syncthreads();
      base0 = (int)bc[2];
    }
    for (int c0 = 0; c0 < W.cta_n; c0 += blockDim.x) {
      const int i = c0 + threadIdx.x;
      const bool in = i < W.cta_n;
      int id = my_id, key = my_key;
      if (c0 > 0 && in) {
        id = W.cta_ids[i];
        key = W.ckey[id];
      }
      const bool k1 = in && key != 0;
      const unsigned b1 = __ballot_sync(0xffffffffu, k1), b0 = __ballot_sync(0xffffffffu, in && !k1);
      if (lane == 0) cnt[wq] = __popc(b1) | (__popc(b0) << 16);
      __syncthreads();
      int p1 = 0, p0 = 0, t1 = 0, t0 = 0;
      for (int q = 0; q < nwq; ++q) {
        const int c1 = cnt[q] & 0xffff, c0n = cnt[q] >> 16;
        if (q < wq) {
          p1 += c1;
          p0 += c0n;
        }
        t1 += c1;
        t0 += c0n;
      }
      if (W.cta_n <= (int)blockDim.x) base0 = t1;  // single chunk: the key-1 count is t1
      const unsigned below = (1u << lane) - 1u;
      if (k1) W.corder[base1 + p1 + __popc(b1 & below)] = id;
      else if (in) W.corder[base0 + p0 + __popc(b0 & below)] = id;
      base1 += t1;
      base0 += t0;
      __syncthreads();
    }
  }
}

// x / w_x update (solver.py:388-394 on the free x block)
__global__ void __launch_bounds__(kBlock) k_xupd(DevProblem P, DevState S, DevWork W) {
  const double shift = W.scal[S_SHIFT];
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < P.n_c; l += gridDim.x * blockDim.x) {
    const double uh = W.ua[l] - shift * P.mz[l];
    const double ur = relax(uh, S.u[l], P.alpha);
    const double wx = S.w[l];
    const double xn = ur - wx;
    S.u[l] = xn;
    S.w[l] = (wx - ur) + xn;
  }
}

#include "hsde_eig.cuh"
#include "hsde_split.cuh"
#include "hsde_cold.cuh"

// ---------------------------------------------------------------------------
// generic small kernels for the unit-level API path

// out[k] = w[k] - w3 * zeta[k] over the T-1 entries (solver.py:301)
__global__ void k_rho(DevProblem P, const double *w, double *rho) {
  const double w3 = w[P.total - 1];
  const int64_t n = P.total - 1, so = P.n_c, yo = P.n_c + P.n_d, vo = yo + P.m;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    double z = 0.0;
    if (k < so) z = P.c[k];
    else if (k >= yo && k < vo) z = -P.b[k - yo];
    rho[k] = w[k] - w3 * z;
  }
}

// slot outputs of _solve_inner_parts: ub, uv from rho_s, rho_v and ua
__global__ void k_slot_out(DevProblem P, const double *rs, const double *rv, const double *ua,
                           double *ub, double *uv) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P.n_d;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double gb = rs[j] - rv[j];
    const double hua = ua[P.slot_cov[j]];
    const double b = (gb + hua) * 0.5;
    ub[j] = b;
    uv[j] = (b - hua) + rv[j];
  }
}

// uy = wy - A ua (solver.py:240-241): A ua reduced from row segments, or the
// identity uy = -g when g (k_schur's output) is given
__global__ void k_uy_from_seg(DevProblem P, const double *qseg, const double *g,
                              const double *wy, double *uy) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m; i += gridDim.x * blockDim.x) {
    if (g) {
      uy[i] = -g[i];
      continue;
    }
    double q = 0.0;
    for (int s = P.row_seg[i]; s < P.row_seg[i + 1]; ++s) q += qseg[s];
    uy[i] = wy[i] - q;
  }
}

// out_i = sum of the row's segment partials (A x)_i
__global__ void k_rowsum_seg(DevProblem P, const double *qseg, double *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m; i += gridDim.x * blockDim.x) {
    double q = 0.0;
    for (int s = P.row_seg[i]; s < P.row_seg[i + 1]; ++s) q += qseg[s];
    out[i] = q;
  }
}

// block partials of sum_k a[k] * b[k]
__global__ void __launch_bounds__(kBlock) k_dot_part(const double *a, const double *b, int64_t n,
                                                     double *part) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    acc += a[k] * b[k];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}


// ordered sum of nparts partials -> out[0]
__global__ void __launch_bounds__(1024) k_sum_parts(const double *part, int nparts, double *out) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) a += part[i];
  a = block_sum(a, sh);
  if (threadIdx.x == 0) out[0] = a;
}

// u12 -= shift * mz ; u_tau = w3 + zeta . u12' computed by the caller
__global__ void k_shift_apply(DevProblem P, double *u12, const double *scal_zu) {
  const double shift = scal_zu[0] / P.zeta_scale;
  const int64_t n = P.total - 1;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    u12[k] -= shift * P.mz[k];
}

// residual pieces (solver.py:398-429, :455-505) on explicit vectors.
// hv = H' v (pull scatter over the covering slots); separator coordinates
// leave a partial in W.sepbuf for the all-reduce (then k_sep_store).
__global__ void __launch_bounds__(kBlock) k_pull(DevProblem P, DevWork W, const double *v,
                                                 double *hv, int nb_light) {
  if ((int)blockIdx.x < nb_light) {
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < P.n_c; l += nb_light * blockDim.x) {
      const int jb = P.cov_ptr[l], je = P.cov_ptr[l + 1];
      if (je - jb > kHeavy) continue;
      double acc = 0.0;
      for (int e = jb; e < je; ++e) acc += v[P.cov_slot[e]];
      if (P.n_sep && P.sep_of[l] >= 0) W.sepbuf[P.sep_of[l]] = acc;
      else hv[l] = acc;
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const int hw = ((int)blockIdx.x - nb_light) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (hw >= P.n_heavy) return;
  const int l = P.heavy[hw];
  double acc = 0.0;
  for (int e = P.cov_ptr[l] + lane; e < P.cov_ptr[l + 1]; e += 32) acc += v[P.cov_slot[e]];
  acc = warp_sum(acc);
  if (lane == 0) {
    if (P.n_sep && P.sep_of[l] >= 0) W.sepbuf[P.sep_of[l]] = acc;
    else hv[l] = acc;
  }
}

__global__ void k_sep_store(DevProblem P, DevWork W, double *hv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n_sep_local; i += gridDim.x * blockDim.x)
    hv[P.sep_local[i]] = W.sepbuf[P.sep_pos[i]];
}

// per owned covered l: (A' y + hv - c)_l^2   (c optional)
__global__ void __launch_bounds__(kBlock) k_dres_part(DevProblem P, const double *y, const double *hv,
                                                      const double *c, double *part) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < P.n_c; l += gridDim.x * blockDim.x) {
    if (!owns(P, l)) continue;
    double aty = 0.0;
    for (int64_t e = P.at_cp[l]; e < P.at_cp[l + 1]; ++e) aty += P.at_val[e] * y[P.at_row[e]];
    const double r = c ? (aty + hv[l]) - c[l] : aty + hv[l];
    acc += r * r;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// block partials of sum over owned l of a[l] * b[l]
__global__ void __launch_bounds__(kBlock) k_dot_owned_part(DevProblem P, const double *a,
                                                           const double *b, double *part) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < P.n_c; l += gridDim.x * blockDim.x)
    if (owns(P, l)) acc += a[l] * b[l];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// merit pieces |u - prev|^2 over the stacked vector: x owned, s/v local,
// y / tau only on the lead shard (replicated there)
__global__ void __launch_bounds__(kBlock) k_merit_part(DevProblem P, const double *a,
                                                       const double *b, double *part) {
  __shared__ double sh[32];
  double acc = 0.0;
  const int64_t yo = P.n_c + P.n_d, vo = yo + P.m;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < P.total;
       k += (int64_t)gridDim.x * blockDim.x) {
    bool use;
    if (k < P.n_c) use = owns(P, (int)k);
    else if (k >= yo && k < vo) use = P.lead;
    else if (k == P.total - 1) use = P.lead;
    else use = true;
    if (use) {
      const double d = a[k] - b[k];
      acc += d * d;
    }
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// per slot: (x[cov(j)] - s[j])^2 and s[j]^2
__global__ void __launch_bounds__(kBlock) k_cons_part(DevProblem P, const double *x, const double *s,
                                                      double *part_a, double *part_b) {
  __shared__ double sh[32];
  double acc = 0.0, ss = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P.n_d;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double d = x[P.slot_cov[j]] - s[j];
    acc += d * d;
    ss += s[j] * s[j];
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part_a[blockIdx.x] = acc;
  ss = block_sum(ss, sh);
  if (threadIdx.x == 0) part_b[blockIdx.x] = ss;
}

// out[k] = in[k] / den   (x / tau, y / b.y, ... as the reference divides)
__global__ void k_div_copy(const double *in, const double *den, double den_mul, int64_t n,
                           double *out) {
  const double dv = den[0] * den_mul;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = in[k] / dv;
}

// out[j] = x[slot_cov[j]]   (gather, graphs.py:245-247)
__global__ void k_gather(DevProblem P, const double *x, double *out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P.n_d;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = x[P.slot_cov[j]];
}

// row residual (A x)_i - b_i with A x from segments; b may be null
__global__ void __launch_bounds__(kBlock) k_rowres_part(DevProblem P, const double *qseg,
                                                        const double *qfull, const double *bvec,
                                                        double *part) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m; i += gridDim.x * blockDim.x) {
    double q = 0.0;
    if (qfull) q = qfull[i];
    else
      for (int s = P.row_seg[i]; s < P.row_seg[i + 1]; ++s) q += qseg[s];
    const double r = bvec ? q - bvec[i] : q;
    acc += r * r;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// block partials of sum (a[k] - b[k])^2
__global__ void __launch_bounds__(kBlock) k_diff2_part(const double *a, const double *b, int64_t n,
                                                       double *part) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double d = a[k] - b[k];
    acc += d * d;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// u_tau of affine_project: out = w3 + zeta . u12'  (solver.py:317)
__global__ void k_tau_out(const double *w, int64_t total, const double *dot, double *u) {
  if (threadIdx.x == 0 && blockIdx.x == 0) u[total - 1] = w[total - 1] + dot[0];
}

// tau clamp of project_cone (solver.py:353-354)
__global__ void k_tau_clamp(const double *in, int64_t total, double *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double t = in[total - 1];
    out[total - 1] = t > 0.0 ? t : 0.0;
  }
}

}  // namespace hsde
