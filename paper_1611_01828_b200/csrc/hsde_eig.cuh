// hsde_eig.cuh -- batched PSD-cone projection of the clique blocks
// (reference: chordalsdp/symmat.py:153-165 `project_psd_batch`, called per
// clique-size group from solver.py:335-342).
//
//   sym = 0.5 (B + B')            eigendecomposition (LAPACK dsyevd there,
//   lambda+ = max(lambda, 0)      cyclic Jacobi here)
//   P = Q diag(lambda+) Q'
//
// One *team* per clique: a warp for d <= 32 (several cliques per CTA), a CTA
// for d > 32.  The symmetric block and its eigenvector rows live in shared
// memory with an odd leading dimension ld = dp + 1 (dp = d rounded up to even;
// a zero row/column pads odd d), which keeps row-strided accesses free of
// bank conflicts.
//
// Cyclic Jacobi, round-robin (tournament) ordering: each round rotates the
// dp/2 disjoint pairs at once -- parameters first (one thread per pair), then
// every 2x2 block (pair k rows) x (pair l columns) transforms independently,
// A <- J' A J, and the eigenvector rows Vt[p], Vt[q] rotate.  Two team
// barriers per round.  Rotations below 2^-60 |A|_F are skipped; sweeps stop
// when the off-diagonal mass falls below 2^-56 |A|_F or a sweep rotates
// nothing (absolute accuracy is what the projection needs: |P - P_exact| is
// bounded by the remaining off-diagonal mass).
//
// Warm start (CTA teams, hot path): ADMM iterates move slowly, so the
// previous iteration's eigenvectors V nearly diagonalise the new block.  The
// kernel forms B = V X V' with two register-tiled shared-memory GEMMs and runs
// Jacobi on B starting from V: typically a few sweeps instead of ~10.
#pragma once
// (included inside namespace hsde by hsde_kernels.cuh)

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

// sum over the team, returned to every member
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

struct JacobiScratch {
  double *A, *Vt, *cs, *tt, *lam, *red;
  int *pq, *offtab, *pos, *flag;
  int ld;
};

__host__ __device__ inline int64_t jacobi_scratch_doubles(int dp) {
  const int64_t ld = dp + 1, half = dp / 2;
  const int64_t noff = half * (half - 1) / 2;
  const int64_t ints = half + noff + dp + 1 + 2;
  return 2 * dp * ld + dp + half + dp + 32 + (ints + 1) / 2 + 1;
}

__device__ inline JacobiScratch jacobi_carve(double *base, int dp) {
  JacobiScratch s;
  const int half = dp / 2;
  s.ld = dp + 1;
  s.A = base;
  s.Vt = s.A + dp * s.ld;
  s.cs = s.Vt + dp * s.ld;
  s.tt = s.cs + dp;
  s.lam = s.tt + half;
  s.red = s.lam + dp;
  s.pq = reinterpret_cast<int *>(s.red + 32);
  s.offtab = s.pq + half;
  s.pos = s.offtab + half * (half - 1) / 2;
  s.flag = s.pos + dp + 1;
  return s;
}

// off-block table (k, l), k < l, and Vt = I (unless warm)
template <class Team>
__device__ void jacobi_prepare(const Team &tm, JacobiScratch &js, int dp, bool init_identity) {
  const int half = dp / 2, ld = js.ld;
  for (int k = tm.rank; k < half; k += tm.size()) {
    const int base = k * (half - 1) - k * (k - 1) / 2;
    for (int l = k + 1; l < half; ++l) js.offtab[base + (l - k - 1)] = k | (l << 16);
  }
  if (init_identity)
    for (int e = tm.rank; e < dp * dp; e += tm.size()) {
      const int i = e / dp, j = e - i * dp;
      js.Vt[i * ld + j] = (i == j) ? 1.0 : 0.0;
    }
}

template <class Team>
__device__ void jacobi_norms(const Team &tm, const JacobiScratch &js, int dp, double &norm2,
                             double &off2) {
  double a2 = 0.0, o2 = 0.0;
  for (int e = tm.rank; e < dp * dp; e += tm.size()) {
    const int i = e / dp, j = e - i * dp;
    const double a = js.A[i * js.ld + j];
    a2 += a * a;
    if (i != j) o2 += a * a;
  }
  norm2 = team_sum(tm, a2, js.red);
  off2 = team_sum(tm, o2, js.red);
}

// Cyclic Jacobi on the symmetric A (dp x dp, padded); rotations accumulate
// into the rows of Vt.  Returns the number of sweeps performed.
template <class Team>
__device__ int jacobi_sweeps(const Team &tm, JacobiScratch &js, int d, int dp) {
  double *A = js.A, *Vt = js.Vt;
  const int ld = js.ld, half = dp / 2, noff = half * (half - 1) / 2;
  double norm2, off2;
  jacobi_norms(tm, js, dp, norm2, off2);
  const double thr = sqrt(norm2) * 8.673617379884035e-19;   // 2^-60 |A|_F
  const double stop2 = norm2 * 1.925929944387236e-34;       // (2^-56 |A|_F)^2
  const int T = tm.size();
  const int vdk = T / d, vdi = T - (T / d) * d;
  int sweep = 0;
  for (; sweep < kMaxSweeps; ++sweep) {
    if (!(off2 > stop2)) break;  // also stops on NaN
    if (tm.rank == 0) js.flag[0] = 0;
    tm.sync();
    for (int r = 0; r < dp - 1; ++r) {
      for (int k = tm.rank; k < half; k += T) {
        const int p = tour_player(k, r, dp), q = tour_player(dp - 1 - k, r, dp);
        const double apq = A[p * ld + q];
        double c = 1.0, s = 0.0, t = 0.0;
        if (fabs(apq) > thr) {
          const double diff = A[q * ld + q] - A[p * ld + p];
          const double rr = sqrt(diff * diff + 4.0 * apq * apq);
          t = (2.0 * apq) / (fabs(diff) + rr);
          if (diff < 0.0) t = -t;
          c = rsqrt(1.0 + t * t);
          s = t * c;
          js.flag[0] = 1;
        }
        js.cs[2 * k] = c;
        js.cs[2 * k + 1] = s;
        js.tt[k] = t;
        js.pq[k] = p | (q << 16);
      }
      tm.sync();
      // off-diagonal 2x2 blocks
      for (int it = tm.rank; it < noff; it += T) {
        const int kl = js.offtab[it];
        const int k = kl & 0xffff, l = kl >> 16;
        const double sk = js.cs[2 * k + 1], sl = js.cs[2 * l + 1];
        if (sk == 0.0 && sl == 0.0) continue;
        const double ck = js.cs[2 * k], cl = js.cs[2 * l];
        const int pk = js.pq[k] & 0xffff, qk = js.pq[k] >> 16;
        const int pl = js.pq[l] & 0xffff, ql = js.pq[l] >> 16;
        const double a = A[pk * ld + pl], bb = A[pk * ld + ql];
        const double cc = A[qk * ld + pl], ee = A[qk * ld + ql];
        const double r_pp = ck * a - sk * cc, r_pq = ck * bb - sk * ee;
        const double r_qp = sk * a + ck * cc, r_qq = sk * bb + ck * ee;
        const double n_pp = cl * r_pp - sl * r_pq, n_pq = sl * r_pp + cl * r_pq;
        const double n_qp = cl * r_qp - sl * r_qq, n_qq = sl * r_qp + cl * r_qq;
        A[pk * ld + pl] = n_pp; A[pl * ld + pk] = n_pp;
        A[pk * ld + ql] = n_pq; A[ql * ld + pk] = n_pq;
        A[qk * ld + pl] = n_qp; A[pl * ld + qk] = n_qp;
        A[qk * ld + ql] = n_qq; A[ql * ld + qk] = n_qq;
      }
      // diagonal 2x2 blocks: closed form
      for (int k = tm.rank; k < half; k += T) {
        const double t = js.tt[k];
        if (t == 0.0) continue;
        const int p = js.pq[k] & 0xffff, q = js.pq[k] >> 16;
        const double apq = A[p * ld + q];
        A[p * ld + p] -= t * apq;
        A[q * ld + q] += t * apq;
        A[p * ld + q] = 0.0;
        A[q * ld + p] = 0.0;
      }
      // eigenvector rows (columns < d only; the pad column stays zero)
      {
        int k = tm.rank / d, i = tm.rank - (tm.rank / d) * d;
        while (k < half) {
          const double s = js.cs[2 * k + 1];
          if (s != 0.0) {
            const double c = js.cs[2 * k];
            const int p = js.pq[k] & 0xffff, q = js.pq[k] >> 16;
            const double vp = Vt[p * ld + i], vq = Vt[q * ld + i];
            Vt[p * ld + i] = c * vp - s * vq;
            Vt[q * ld + i] = s * vp + c * vq;
          }
          k += vdk;
          i += vdi;
          if (i >= d) {
            i -= d;
            ++k;
          }
        }
      }
      tm.sync();
    }
    const int rotated = js.flag[0];
    double n2;
    jacobi_norms(tm, js, dp, n2, off2);  // (team barriers inside)
    if (!rotated) {
      ++sweep;
      break;  // every pair below the rotation threshold
    }
  }
  return sweep;
}

// ---------------------------------------------------------------------------
// register-tiled team GEMMs on d x d shared-memory operands (ld-strided).
// Thread t owns the interleaved 4x4 tile rows {u + nt a}, cols {v + nt b},
// u = t / nt, v = t % nt, nt = ceil(d / 4): consecutive threads read
// consecutive rows / columns, so the odd ld keeps them conflict free.
// Requires nt * nt <= team size.

// out = L * R'   (out[i][j] = sum_k L[i][k] R[j][k]); out may alias L or R.
template <class Team>
__device__ void team_gemm_nt(const Team &tm, const double *L, const double *R, double *out,
                             int d, int ld) {
  const int nt = (d + 3) >> 2;
  const int t = tm.rank;
  const bool active = t < nt * nt;
  const int u = active ? t / nt : 0, v = active ? t - u * nt : 0;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  if (active) {
    int ri[4], rj[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      ri[a] = min(u + nt * a, d - 1) * ld;
      rj[a] = min(v + nt * a, d - 1) * ld;
    }
    for (int k = 0; k < d; ++k) {
      double l[4], r[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        l[a] = L[ri[a] + k];
        r[a] = R[rj[a] + k];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(l[a], r[b], acc[a][b]);
    }
  }
  tm.sync();
  if (active) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = u + nt * a, j = v + nt * b;
        if (i < d && j < d) out[i * ld + j] = acc[a][b];
      }
  }
  tm.sync();
}

// P = W' V over the first r rows (P[i][j] = sum_k W[k][i] V[k][j]), symmetric
// output: tiles with u <= v compute, each value emitted for (i, j) and (j, i).
template <class Team, class Emit>
__device__ void team_gemm_tn_sym(const Team &tm, const double *W, const double *V, const int *vrow,
                                 int r, int d, int ld, Emit emit) {
  const int nt = (d + 3) >> 2;
  const int t = tm.rank;
  if (t >= nt * nt) return;
  const int u = t / nt, v = t - u * nt;
  if (u > v) return;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  int ci[4], cj[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    ci[a] = min(u + nt * a, d - 1);
    cj[a] = min(v + nt * a, d - 1);
  }
  for (int k = 0; k < r; ++k) {
    double w[4], x[4];
#pragma unroll
    const int vk = vrow[k] * ld;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      w[a] = W[k * ld + ci[a]];
      x[a] = V[vk + cj[a]];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(w[a], x[b], acc[a][b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = u + nt * a, j = v + nt * b;
      if (i < d && j < d && (u < v || i <= j)) emit(i, j, acc[a][b]);
    }
}

// compacted positive eigenvalues (warp 0 ballot, ascending position order)
template <class Team>
__device__ int compact_positive(const Team &tm, JacobiScratch &js, int d) {
  const int ld = js.ld;
  if (tm.rank < 32) {
    int base = 0;
    for (int i0 = 0; i0 < d; i0 += 32) {
      const int i = i0 + tm.rank;
      const double lam = i < d ? js.A[i * ld + i] : 0.0;
      const bool pos = i < d && lam > 0.0;
      const unsigned mask = __ballot_sync(0xffffffffu, pos);
      if (pos) {
        const int slot = base + __popc(mask & ((1u << tm.rank) - 1u));
        js.pos[slot] = i;
        js.lam[slot] = lam;
      }
      base += __popc(mask);
    }
    if (tm.rank == 0) js.pos[d] = base;
  }
  tm.sync();
  return js.pos[d];
}

// P = sum_{lambda > 0} lambda v v' -> emit(a, b, value) for all a, b (both triangles)
template <class Team, class Emit>
__device__ void psd_rebuild(const Team &tm, JacobiScratch &js, int d, Emit emit) {
  const int ld = js.ld;
  const int r = compact_positive(tm, js, d);
  const int nt = (d + 3) >> 2;
  if (tm.size() <= 32 || nt * nt > tm.size()) {
    // small (warp teams) or too large for one tile per thread: direct sums
    const int nout = d * (d + 1) / 2;
    for (int o = tm.rank; o < nout; o += tm.size()) {
      int a = 0, rem = o;
      while (rem >= d - a) {
        rem -= d - a;
        ++a;
      }
      const int b = a + rem;
      double acc = 0.0;
      for (int k = 0; k < r; ++k) {
        const int pi = js.pos[k];
        acc += (js.lam[k] * js.Vt[pi * ld + a]) * js.Vt[pi * ld + b];
      }
      emit(a, b, acc);
      if (a != b) emit(b, a, acc);
    }
    tm.sync();
    return;
  }
  // CTA: W[k] = lambda_k Vt[pos[k]] into A's storage (A no longer needed)
  double *W = js.A;
  for (int e = tm.rank; e < r * d; e += tm.size()) {
    const int k = e / d, i = e - k * d;
    W[k * ld + i] = js.lam[k] * js.Vt[js.pos[k] * ld + i];
  }
  tm.sync();
  team_gemm_tn_sym(tm, W, js.Vt, js.pos, r, d, ld, [&](int i, int j, double v) {
    emit(i, j, v);
    if (i != j) emit(j, i, v);
  });
  tm.sync();
}

// ---------------------------------------------------------------------------
// cone kernels

enum ConeMode { CONE_HOT = 0, CONE_PLAIN = 1, CONE_MINEIG = 2 };

struct ConeArgs {
  const int *ids;   // clique ids of this launch
  int count;
  int dpmax;        // scratch leading dimension bound
  const double *in; // PLAIN/MINEIG: stacked s-segment input [n_d]
  double *out;      // PLAIN: stacked output; MINEIG: per-clique min eigenvalue [p]
  double in_scale;
  int warm;         // HOT: use / refresh the per-clique eigenvector store
};

// Hot-path load of slot j: builds arg_s and performs the v / w_v update and
// the first half of the w_s update in place (solver.py:222-244 slot part,
// :316, :388-394).
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
  const double vn = uv_h - wv;                               // free block: identity
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
      else a = ca.in[off] * ca.in_scale;
      const double pr = (a != a) ? a : (a > 0.0 ? a : 0.0);  // np.maximum(b, 0.0)
      if (MODE == CONE_HOT) {
        S.u[so + off] = pr;
        S.w[so + off] += pr;
        if (W.sweeps) W.sweeps[k] = 0;
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
  const int ld = js.ld;
  double *A = js.A;
  const bool warm = (MODE == CONE_HOT) && ca.warm && W.vvalid[k] &&
                    ((d + 3) >> 2) * ((d + 3) >> 2) <= tm.size();
  // load (raw), then symmetrise sym = 0.5 (B + B')  (symmat.py:157)
  for (int e = tm.rank; e < d * d; e += tm.size()) {
    const int a = e / d, bcol = e - a * d;
    double v;
    if (MODE == CONE_HOT) v = hot_slot_load(P, S, W, off + e, shift);
    else v = ca.in[off + e] * ca.in_scale;
    A[a * ld + bcol] = v;
    if (warm) js.Vt[a * ld + bcol] = W.vstore[off + e];
  }
  if (d & 1) {
    for (int e = tm.rank; e < dp; e += tm.size()) {
      A[d * ld + e] = 0.0;
      A[e * ld + d] = 0.0;
      js.Vt[d * ld + e] = (e == d) ? 1.0 : 0.0;
      js.Vt[e * ld + d] = (e == d) ? 1.0 : 0.0;
    }
  }
  jacobi_prepare(tm, js, dp, !warm);
  tm.sync();
  for (int e = tm.rank; e < d * d; e += tm.size()) {
    const int a = e / d, bcol = e - a * d;
    if (a < bcol) {
      const double s = 0.5 * (A[a * ld + bcol] + A[bcol * ld + a]);
      A[a * ld + bcol] = s;
      A[bcol * ld + a] = s;
    }
  }
  tm.sync();
  if (warm) {
    // B = V X V' (rows of Vt are the previous eigenvectors)
    team_gemm_nt(tm, js.Vt, A, A, d, ld);   // T1 = Vt X   (X symmetric)
    team_gemm_nt(tm, A, js.Vt, A, d, ld);   // B = T1 Vt'
    for (int e = tm.rank; e < d * d; e += tm.size()) {
      const int a = e / d, bcol = e - a * d;
      if (a < bcol) {
        const double s = 0.5 * (A[a * ld + bcol] + A[bcol * ld + a]);
        A[a * ld + bcol] = s;
        A[bcol * ld + a] = s;
      }
    }
    tm.sync();
  }
  const int sw = jacobi_sweeps(tm, js, d, dp);
  if (MODE == CONE_HOT && tm.rank == 0 && W.sweeps) W.sweeps[k] = sw;
  // non-finite eigenvalue -> EigenFailure (symmat.py:162-163)
  double nb = 0.0;
  for (int i = tm.rank; i < d; i += tm.size()) nb += isfinite(A[i * ld + i]) ? 0.0 : 1.0;
  const bool bad = team_sum(tm, nb, js.red) > 0.0;
  if (bad && tm.rank == 0) atomicOr(W.err, 1);
  if (MODE == CONE_MINEIG) {
    double mn = CUDART_INF;
    for (int i = 0; i < d; ++i) mn = fmin(mn, A[i * ld + i]);
    if (tm.rank == 0) ca.out[k] = mn;
    tm.sync();
    return;
  }
  if (MODE == CONE_HOT && ca.warm) {
    for (int e = tm.rank; e < d * d; e += tm.size()) {
      const int a = e / d, bcol = e - a * d;
      W.vstore[off + e] = js.Vt[a * ld + bcol];
    }
    if (tm.rank == 0) W.vvalid[k] = bad ? 0 : 1;
  }
  if (MODE == CONE_HOT) {
    psd_rebuild(tm, js, d, [&](int a, int bcol, double v) {
      const int64_t j = so + off + (int64_t)a * d + bcol;
      S.u[j] = v;
      S.w[j] += v;
    });
  } else {
    psd_rebuild(tm, js, d, [&](int a, int bcol, double v) {
      ca.out[off + (int64_t)a * d + bcol] = v;
    });
  }
}

constexpr int kConeBlock = 512;  // threads per CTA team (d > 32)

// one warp per clique (d <= 32); dynamic smem = warps * scratch(dpmax)
template <int MODE>
__global__ void __launch_bounds__(kBlock) k_cone_warp(DevProblem P, DevState S, DevWork W, ConeArgs ca) {
  extern __shared__ double smem[];
  const int wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + wid;
  if (gw >= ca.count) return;
  double *scratch = smem + (int64_t)wid * jacobi_scratch_doubles(ca.dpmax);
  WarpTeam tm{(int)(threadIdx.x & 31)};
  ConeArgs c2 = ca;
  c2.warm = 0;
  cone_one<MODE>(tm, P, S, W, c2, ca.ids[gw], scratch);
}

// one CTA per clique (d > 32)
template <int MODE>
__global__ void __launch_bounds__(kConeBlock, 2) k_cone_block(DevProblem P, DevState S, DevWork W, ConeArgs ca) {
  extern __shared__ double smem[];
  if ((int)blockIdx.x >= ca.count) return;
  BlockTeam tm{(int)threadIdx.x, (int)blockDim.x};
  cone_one<MODE>(tm, P, S, W, ca, ca.ids[blockIdx.x], smem);
}
