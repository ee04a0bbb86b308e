// hsde_kernels.cuh -- sm_100a fp64 kernels of the HSDE-ADMM hot path.
//
// One ADMM iteration (reference: chordalsdp/solver.py:375-395) on the
// compressed layout [x n_c | s n_d | y m | v n_d | tau] is, in launch order:
//
//   k_rhs      per covered coordinate l: pull-scatter of the clique slots
//              covering l (graphs.py:249-252, atomic-free), CSC column of A'
//              (solver.py:226), r and t = P^{-1} r (solver.py:222-231)
//   k_spmv_seg row-split CSR SpMV q = A t (solver.py:232 `dp.A @ t`)
//   k_schur    q' = S^{-1} q with the cached inverse (solver.py:232 cho_solve)
//   k_ua       ua = t - P^{-1} A' q' (solver.py:232-235) + block partials of c.ua
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
  const int64_t *cl_off;
  const int *cl_size;
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
  double *ry;          // [m] rho_y of the current iteration
  double *qseg;        // [nseg]
  double *qp;          // [m]
  double *uy;          // [m]
  double *part;        // [kMaxParts]
  double *scal;        // [S_COUNT]
  int *err;            // [1] bit 0: non-finite eigenvalue
};

// ---------------------------------------------------------------------------
// helpers

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

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
// k_rhs: r = 0.5 H'(rho_s - rho_v) + H' rho_v + A' rho_y + rho_x ; t = P^{-1} r
// (solver.py:222-231).  FROM_STATE: rho comes from the state u + w and a_tau
// (affine_project :300-301 fused); otherwise from explicit vectors.

template <bool FROM_STATE>
__global__ void __launch_bounds__(kBlock) k_rhs(DevProblem P, DevState S, DevWork W,
                                                const double *rx, const double *rs,
                                                const double *ry, const double *rv) {
  const int64_t xo = 0, so = P.n_c, vo = P.n_c + P.n_d + P.m;
  double atau = 0.0;
  if (FROM_STATE) {
    atau = S.u[P.total - 1] + S.w[P.total - 1];
    ry = W.ry;
  }
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < P.n_c; l += gridDim.x * blockDim.x) {
    double sg = 0.0, sv = 0.0;
    const int jb = P.cov_ptr[l], je = P.cov_ptr[l + 1];
    for (int e = jb; e < je; ++e) {
      const int j = P.cov_slot[e];
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
    double aty = 0.0;
    const int64_t cb = P.at_cp[l], ce = P.at_cp[l + 1];
    for (int64_t e = cb; e < ce; ++e) aty += P.at_val[e] * __ldg(ry + P.at_row[e]);
    double rx_l;
    if (FROM_STATE)
      rx_l = (S.u[xo + l] + S.w[xo + l]) - atau * P.c[l];
    else
      rx_l = rx[l];
    const double r = ((sg * 0.5 + sv) + aty) + rx_l;
    W.t[l] = r * P.p_inv[l];
  }
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

// q' = S^{-1} q.  Every CTA rebuilds q from the segment partials (ordered),
// then one warp per output row of the symmetric inverse.
__global__ void __launch_bounds__(kBlock) k_schur(DevProblem P, const double *__restrict__ qseg,
                                                   double *__restrict__ qp) {
  extern __shared__ double qs[];
  for (int i = threadIdx.x; i < P.m; i += blockDim.x) {
    double q = 0.0;
    for (int s = P.row_seg[i]; s < P.row_seg[i + 1]; ++s) q += qseg[s];
    qs[i] = q;
  }
  __syncthreads();
  if (P.schur_diag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m; i += gridDim.x * blockDim.x)
      qp[i] = qs[i] * P.sinv[i];
    return;
  }
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < P.m; i += warps) {
    const double *row = P.sinv + (int64_t)i * P.m;
    double acc = 0.0;
    for (int j = lane; j < P.m; j += 32) acc += row[j] * qs[j];
    acc = warp_sum(acc);
    if (lane == 0) qp[i] = acc;
  }
}

// ua = t - P^{-1} (A' q')  (solver.py:232-235); WITH_DOT: block partials of c.ua
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
    if (WITH_DOT) dot += P.c[l] * ua;
  }
  if (WITH_DOT) {
    dot = block_sum(dot, sh);
    if (threadIdx.x == 0) W.part[blockIdx.x] = dot;
  }
}

// ---------------------------------------------------------------------------
// k_scalars: one CTA.  zeta.u12 = c.ua - b.uy (zeta = (c, 0, -b, 0),
// solver.py:264), shift (:315), u_hat tau (:317), relaxation (:388-390), tau/kappa
// projection and dual update (:391-394), y update, next rho_y.

__global__ void __launch_bounds__(1024) k_scalars(DevProblem P, DevState S, DevWork W, int nparts,
                                                  int exact_uy, const double *__restrict__ auy) {
  __shared__ double sh[32];
  __shared__ double bc[4];
  const int64_t yo = P.n_c + P.n_d;
  double a = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) a += W.part[i];
  const double cua = block_sum(a, sh);
  double bu = 0.0;
  for (int i = threadIdx.x; i < P.m; i += blockDim.x) {
    // uy = rho_y - A ua (solver.py:240-241); identity A ua = q' unless exact
    const double uy = W.ry[i] - (exact_uy ? auy[i] : W.qp[i]);
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

// ---------------------------------------------------------------------------
// Team-parallel cyclic Jacobi for the PSD projection (symmat.py:153-165).
//
// The symmetric matrix lives in shared memory with an even leading dimension
// dp (a zero row/column pads odd d).  One round of the round-robin tournament
// rotates dp/2 disjoint pairs at once: rotation parameters first (one thread
// per pair), then every 2x2 block (pair k rows) x (pair l cols) is transformed
// independently, A <- J' A J, and the eigenvector rows Vt[p], Vt[q] are
// rotated.  Two team barriers per round; sweeps until no pair exceeds the
// absolute threshold 2^-60 |A|_F (projection error is absolute).

struct WarpTeam {
  int rank;
  __device__ static constexpr int size() { return 32; }
  __device__ void sync() const { __syncwarp(); }
};
struct BlockTeam {
  int rank, n;
  __device__ int size() const { return n; }
  __device__ void sync() const { __syncthreads(); }
};

template <class Team>
__device__ double team_sum(const Team &tm, double v, double *red) {
  v = warp_sum(v);
  v = __shfl_sync(0xffffffffu, v, 0);
  if (tm.size() <= 32) return v;
  const int lane = tm.rank & 31, wid = tm.rank >> 5;
  tm.sync();
  if (lane == 0) red[wid] = v;
  tm.sync();
  double r = 0.0;
  const int nw = (tm.size() + 31) >> 5;
  for (int i = 0; i < nw; ++i) r += red[i];
  tm.sync();
  return r;
}

__device__ __forceinline__ int tour_player(int pos, int r, int dp) {
  return pos == 0 ? 0 : 1 + ((pos - 1 + r) % (dp - 1));
}

// Scratch layout for one team (doubles): A[dp*dp] Vt[dp*dp] cs[dp] (c,s interleaved)
// tt[dp/2] ; ints: pq[dp/2] ; flags[2] ; red[32]
struct JacobiScratch {
  double *A, *Vt, *cs, *tt, *red;
  int *pq, *flag, *pos;
};

__host__ __device__ inline int64_t jacobi_scratch_doubles(int dp) {
  return 2LL * dp * dp + dp + dp / 2 + 32 + (dp / 2 + 2 + dp + 1) / 2 + 2;
}

__device__ inline JacobiScratch jacobi_carve(double *base, int dp) {
  JacobiScratch s;
  s.A = base;
  s.Vt = s.A + dp * dp;
  s.cs = s.Vt + dp * dp;
  s.tt = s.cs + dp;
  s.red = s.tt + dp / 2;
  s.pq = reinterpret_cast<int *>(s.red + 32);
  s.flag = s.pq + dp / 2;
  s.pos = s.flag + 2;
  return s;
}

// Returns number of sweeps; eigenvalues on diag(A) (positions < d), vectors in Vt rows.
template <class Team>
__device__ int jacobi_eigh(const Team &tm, JacobiScratch &js, int d, int dp) {
  double *A = js.A, *Vt = js.Vt;
  const int half = dp / 2;
  // Vt = I
  for (int e = tm.rank; e < dp * dp; e += tm.size()) Vt[e] = (e / dp == e % dp) ? 1.0 : 0.0;
  double loc = 0.0;
  for (int e = tm.rank; e < dp * dp; e += tm.size()) loc += A[e] * A[e];
  const double nrm2 = team_sum(tm, loc, js.red);
  const double thr = sqrt(nrm2) * 8.673617379884035e-19;  // 2^-60 |A|_F
  int sweep = 0;
  const int noff = half * (half - 1) / 2;
  for (; sweep < kMaxSweeps; ++sweep) {
    if (tm.rank == 0) js.flag[0] = 0;
    tm.sync();
    for (int r = 0; r < dp - 1; ++r) {
      // step 1: rotation parameters of the dp/2 disjoint pairs
      for (int k = tm.rank; k < half; k += tm.size()) {
        const int p = tour_player(k, r, dp), q = tour_player(dp - 1 - k, r, dp);
        const double apq = A[p * dp + q];
        double c = 1.0, s = 0.0, t = 0.0;
        if (fabs(apq) > thr) {
          const double app = A[p * dp + p], aqq = A[q * dp + q];
          const double th = (aqq - app) / (2.0 * apq);
          const double ath = fabs(th);
          t = ath > 1e150 ? 0.5 / th : (th >= 0.0 ? 1.0 : -1.0) / (ath + sqrt(1.0 + th * th));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
          js.flag[0] = 1;
        }
        js.cs[2 * k] = c;
        js.cs[2 * k + 1] = s;
        js.tt[k] = t;
        js.pq[k] = p | (q << 16);
      }
      tm.sync();
      // step 2: all 2x2 blocks, diagonal blocks, eigenvector rows
      const int nv = half * dp;
      const int items = noff + half + nv;
      for (int it = tm.rank; it < items; it += tm.size()) {
        if (it < noff) {
          // unrank (k, l), k < l
          int k = 0, rem = it;
          while (rem >= half - 1 - k) { rem -= half - 1 - k; ++k; }
          const int l = k + 1 + rem;
          const double ck = js.cs[2 * k], sk = js.cs[2 * k + 1];
          const double cl = js.cs[2 * l], sl = js.cs[2 * l + 1];
          if (sk == 0.0 && sl == 0.0) continue;
          const int pk = js.pq[k] & 0xffff, qk = js.pq[k] >> 16;
          const int pl = js.pq[l] & 0xffff, ql = js.pq[l] >> 16;
          const double a = A[pk * dp + pl], bb = A[pk * dp + ql];
          const double cc = A[qk * dp + pl], ee = A[qk * dp + ql];
          const double r_pp = ck * a - sk * cc, r_pq = ck * bb - sk * ee;
          const double r_qp = sk * a + ck * cc, r_qq = sk * bb + ck * ee;
          const double n_pp = cl * r_pp - sl * r_pq, n_pq = sl * r_pp + cl * r_pq;
          const double n_qp = cl * r_qp - sl * r_qq, n_qq = sl * r_qp + cl * r_qq;
          A[pk * dp + pl] = n_pp; A[pl * dp + pk] = n_pp;
          A[pk * dp + ql] = n_pq; A[ql * dp + pk] = n_pq;
          A[qk * dp + pl] = n_qp; A[pl * dp + qk] = n_qp;
          A[qk * dp + ql] = n_qq; A[ql * dp + qk] = n_qq;
        } else if (it < noff + half) {
          const int k = it - noff;
          const double t = js.tt[k];
          if (t == 0.0 && js.cs[2 * k + 1] == 0.0) continue;
          const int p = js.pq[k] & 0xffff, q = js.pq[k] >> 16;
          const double apq = A[p * dp + q];
          A[p * dp + p] -= t * apq;
          A[q * dp + q] += t * apq;
          A[p * dp + q] = 0.0;
          A[q * dp + p] = 0.0;
        } else {
          const int v = it - noff - half;
          const int k = v / dp, i = v - k * dp;
          const double c = js.cs[2 * k], s = js.cs[2 * k + 1];
          if (s == 0.0) continue;
          const int p = js.pq[k] & 0xffff, q = js.pq[k] >> 16;
          const double vp = Vt[p * dp + i], vq = Vt[q * dp + i];
          Vt[p * dp + i] = c * vp - s * vq;
          Vt[q * dp + i] = s * vp + c * vq;
        }
      }
      tm.sync();
    }
    const int rotated = js.flag[0];
    tm.sync();
    if (!rotated) break;
  }
  return sweep;
}

// P = sum_{lambda_i > 0} lambda_i v_i v_i'  written through `emit(a, b, value)`
// for a <= b (caller mirrors).  Uses A's off-diagonal storage as scratch for the
// scaled vectors; js.pos holds the compacted positive positions.
template <class Team, class Emit>
__device__ void psd_rebuild(const Team &tm, JacobiScratch &js, int d, int dp, Emit emit) {
  double *A = js.A, *Vt = js.Vt;
  // compact positive eigenvalues (warp 0 ballot, ascending position order)
  if (tm.rank < 32) {
    int base = 0;
    for (int i0 = 0; i0 < d; i0 += 32) {
      const int i = i0 + tm.rank;
      const bool pos = i < d && A[i * dp + i] > 0.0;
      const unsigned mask = __ballot_sync(0xffffffffu, pos);
      if (pos) js.pos[base + __popc(mask & ((1u << tm.rank) - 1u))] = i;
      base += __popc(mask);
    }
    if (tm.rank == 0) js.pos[dp] = base;
  }
  tm.sync();
  const int r = js.pos[dp];
  const int nout = d * (d + 1) / 2;
  for (int o = tm.rank; o < nout; o += tm.size()) {
    int a = 0, rem = o;
    while (rem >= d - a) { rem -= d - a; ++a; }
    const int b = a + rem;
    double acc = 0.0;
    for (int k = 0; k < r; ++k) {
      const int pi = js.pos[k];
      const double lam = A[pi * dp + pi];
      acc += (Vt[pi * dp + a] * lam) * Vt[pi * dp + b];
    }
    emit(a, b, acc);
  }
}

// Cone kernel modes
enum ConeMode { CONE_HOT = 0, CONE_PLAIN = 1, CONE_MINEIG = 2 };

struct ConeArgs {
  const int *ids;     // clique ids of this launch
  int count;
  int dpmax;          // scratch leading dimension bound
  const double *in;   // PLAIN/MINEIG: stacked s-segment input [n_d]
  double *out;        // PLAIN: stacked s-segment output; MINEIG: per-clique min eig [p]
  double in_scale;    // MINEIG: multiply input by this
};

// Load phase of the hot path for one slot j of a clique: builds arg_s and
// performs the v / w_v update and the first half of the w_s update in place.
__device__ __forceinline__ double hot_slot_load(const DevProblem &P, const DevState &S,
                                                const DevWork &W, int64_t j, double shift) {
  const int64_t so = P.n_c, vo = P.n_c + P.n_d + P.m;
  const double us = S.u[so + j], ws = S.w[so + j];
  const double uv0 = S.u[vo + j], wv = S.w[vo + j];
  const double as = us + ws, av = uv0 + wv;                  // a = u + w
  const double gb = as - av;                                 // solver.py:222
  const double hua = W.ua[P.slot_cov[j]];                    // :236
  const double ub = (gb + hua) * 0.5;                        // :237-239
  const double uv = (ub - hua) + av;                         // :242-244
  const double mzs = P.mz[P.n_c + j], mzv = P.mz[P.n_c + P.n_d + P.m + j];
  const double us_h = relax(ub - shift * mzs, us, P.alpha);  // :316, :388-390
  const double uv_h = relax(uv - shift * mzv, uv0, P.alpha);
  const double arg_s = us_h - ws;                            // :391
  const double vn = uv_h - wv;                               // free block: projection = identity
  S.u[vo + j] = vn;
  S.w[vo + j] = (wv - uv_h) + vn;                            // :393-394
  S.w[so + j] = ws - us_h;                                   // completed after projection
  return arg_s;
}

template <int MODE, class Team>
__device__ void cone_one(const Team &tm, const DevProblem &P, const DevState &S, const DevWork &W,
                         const ConeArgs &ca, int k, double *scratch) {
  const int d = P.cl_size[k];
  const int64_t off = P.cl_off[k];
  const int64_t so = P.n_c;
  const double shift = (MODE == CONE_HOT) ? W.scal[S_SHIFT] : 0.0;
  if (d == 1) {
    if (tm.rank == 0) {
      double a;
      if (MODE == CONE_HOT) a = hot_slot_load(P, S, W, off, shift);
      else a = ca.in[off] * (MODE == CONE_MINEIG ? ca.in_scale : 1.0);
      const double pr = (a != a) ? a : (a > 0.0 ? a : 0.0);  // np.maximum(b, 0.0)
      if (MODE == CONE_HOT) {
        S.u[so + off] = pr;
        S.w[so + off] += pr;
      } else if (MODE == CONE_PLAIN) {
        ca.out[off] = pr;
      } else {
        ca.out[k] = a;
      }
    }
    return;
  }
  const int dp = d + (d & 1);
  JacobiScratch js = jacobi_carve(scratch, dp);
  double *A = js.A;
  // load (raw), then symmetrise sym = 0.5 (B + B')  (symmat.py:157)
  for (int e = tm.rank; e < d * d; e += tm.size()) {
    const int a = e / d, bcol = e - a * d;
    double v;
    if (MODE == CONE_HOT) v = hot_slot_load(P, S, W, off + e, shift);
    else v = ca.in[off + e] * (MODE == CONE_MINEIG ? ca.in_scale : 1.0);
    A[a * dp + bcol] = v;
  }
  if (d & 1) {
    for (int e = tm.rank; e < dp; e += tm.size()) {
      A[d * dp + e] = 0.0;
      A[e * dp + d] = 0.0;
    }
  }
  tm.sync();
  for (int e = tm.rank; e < d * d; e += tm.size()) {
    const int a = e / d, bcol = e - a * d;
    if (a < bcol) {
      const double s = 0.5 * (A[a * dp + bcol] + A[bcol * dp + a]);
      A[a * dp + bcol] = s;
      A[bcol * dp + a] = s;
    } else if (a == bcol) {
      A[a * dp + a] = 0.5 * (A[a * dp + a] + A[a * dp + a]);
    }
  }
  tm.sync();
  jacobi_eigh(tm, js, d, dp);
  // non-finite eigenvalue -> EigenFailure (symmat.py:162-163)
  bool bad = false;
  for (int i = tm.rank; i < d; i += tm.size()) bad |= !isfinite(A[i * dp + i]);
  if (bad) atomicOr(W.err, 1);
  if (MODE == CONE_MINEIG) {
    double mn = CUDART_INF;
    for (int i = 0; i < d; ++i) mn = fmin(mn, A[i * dp + i]);
    if (tm.rank == 0) ca.out[k] = mn;
    tm.sync();
    return;
  }
  if (MODE == CONE_HOT) {
    psd_rebuild(tm, js, d, dp, [&](int a, int bcol, double v) {
      const int64_t j1 = so + off + (int64_t)a * d + bcol, j2 = so + off + (int64_t)bcol * d + a;
      S.u[j1] = v;
      S.w[j1] += v;
      if (j2 != j1) {
        S.u[j2] = v;
        S.w[j2] += v;
      }
    });
  } else {
    psd_rebuild(tm, js, d, dp, [&](int a, int bcol, double v) {
      ca.out[off + (int64_t)a * d + bcol] = v;
      ca.out[off + (int64_t)bcol * d + a] = v;
    });
  }
  tm.sync();
}

// one warp per clique (d <= 32); dynamic smem = warps * scratch(dpmax)
template <int MODE>
__global__ void __launch_bounds__(kBlock) k_cone_warp(DevProblem P, DevState S, DevWork W, ConeArgs ca) {
  extern __shared__ double smem[];
  const int wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + wid;
  if (gw >= ca.count) return;
  double *scratch = smem + (int64_t)wid * jacobi_scratch_doubles(ca.dpmax);
  WarpTeam tm{(int)(threadIdx.x & 31)};
  cone_one<MODE>(tm, P, S, W, ca, ca.ids[gw], scratch);
}

// one CTA per clique (d > 32)
template <int MODE>
__global__ void __launch_bounds__(kBlock) k_cone_block(DevProblem P, DevState S, DevWork W, ConeArgs ca) {
  extern __shared__ double smem[];
  if ((int)blockIdx.x >= ca.count) return;
  BlockTeam tm{(int)threadIdx.x, (int)blockDim.x};
  cone_one<MODE>(tm, P, S, W, ca, ca.ids[blockIdx.x], smem);
}

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

// uy = wy - A ua, rows reduced from segments (solver.py:240-241)
__global__ void k_uy_from_seg(DevProblem P, const double *qseg, const double *wy, double *uy) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m; i += gridDim.x * blockDim.x) {
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

// residual pieces (solver.py:398-429, :455-505) on explicit vectors:
//   per covered l: (A' y + H' v - c)_l  (c optional)
__global__ void __launch_bounds__(kBlock) k_dres_part(DevProblem P, const double *y, const double *v,
                                                      const double *c, double *part) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < P.n_c; l += gridDim.x * blockDim.x) {
    double aty = 0.0;
    for (int64_t e = P.at_cp[l]; e < P.at_cp[l + 1]; ++e) aty += P.at_val[e] * y[P.at_row[e]];
    double hv = 0.0;
    for (int e = P.cov_ptr[l]; e < P.cov_ptr[l + 1]; ++e) hv += v[P.cov_slot[e]];
    const double r = c ? (aty + hv) - c[l] : aty + hv;
    acc += r * r;
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
                                                        const double *bvec, double *part) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m; i += gridDim.x * blockDim.x) {
    double q = 0.0;
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
