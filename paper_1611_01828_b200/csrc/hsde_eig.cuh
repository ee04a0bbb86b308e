// hsde_eig.cuh -- batched PSD-cone projection of the clique blocks
// (reference: chordalsdp/symmat.py:153-165 `project_psd_batch`, called per
// clique-size group from solver.py:335-342).
//
//   sym = 0.5 (B + B')            eigendecomposition (LAPACK dsyevd there,
//   lambda+ = max(lambda, 0)      cyclic Jacobi here)
//   P = Q diag(lambda+) Q'
//
// One *team* per clique: a warp for d <= 32 (several cliques per CTA), a CTA
// for d > 32.  The symmetric block lives in shared memory with an odd leading
// dimension (lda = dp + 1, dp = d rounded up to even; a zero row/column pads
// odd d) so that row- and column-strided accesses are conflict free; the
// eigenvector rows Vt use a leading dimension that is a multiple of 4 so they
// are updated with 16-byte vector accesses.
//
// Cyclic Jacobi, round-robin (tournament) ordering: each round rotates the
// dp/2 disjoint pairs at once.  Per round:
//   phase P  -- rotation parameters of round r (one thread per pair, into a
//               double-buffered table) while the other threads apply round
//               r-1's rotations to the eigenvector rows;
//   phase A  -- every 2x2 block (pair k rows) x (pair l columns) transforms
//               independently, A <- J' A J, plus the closed-form diagonal.
// Two team barriers per round.  Rotations below 2^-60 |A|_F are skipped;
// sweeps stop when the off-diagonal mass falls below 2^-56 |A|_F or a sweep
// rotates nothing (absolute accuracy is what the projection needs: the
// error of P is bounded by the remaining off-diagonal mass).
//
// Warm start (hot path): ADMM iterates move slowly, so the
// previous iteration's eigenvectors V nearly diagonalise the new block.  The
// kernel forms B = V X V' with two register-tiled shared-memory GEMMs and runs
// Jacobi on B starting from V: ~3 sweeps instead of ~10.  V is refreshed by
// a cold solve every kWarmMaxAge iterations to bound its orthogonality drift.
#pragma once
// (included inside namespace hsde by hsde_kernels.cuh)

constexpr int kWarmMaxAge = 64;

// k_cone_split -> k_cone_block hand-off states (DevWork::cstate, hsde_split.cuh)
// (SPLIT_HANDOFF + 0/1/2: off(B) > g / 10 / r > n / the fixed point stalled)
enum SplitState { SPLIT_DONE = 0, SPLIT_UNTOUCHED = 1, SPLIT_HANDOFF = 2 };
// vvalid bit: the fast path asks for a refreshed V (the next projection of the
// clique runs in k_cone_block, warm, which rotates V)
constexpr int kVRefresh = 1 << 30;

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
// GEMM tiles per thread: a warp covers d <= 32 (8 x 8 tiles of 4 x 4) with two
template <class Team> struct TeamTiles { static constexpr int value = 1; };
template <> struct TeamTiles<WarpTeam> { static constexpr int value = 2; };

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

// player at tournament position `pos` in round r (0 <= r < dp - 1): position 0
// is fixed, the others rotate (no integer division: pos - 1 + r < 2 (dp - 1)).
// Pair k of round r is (tour_player(k), tour_player(dp - 1 - k)).
__device__ __forceinline__ int tour_player(int pos, int r, int dp) {
  int x = pos - 1 + r;
  if (x >= dp - 1) x -= dp - 1;
  return pos == 0 ? 0 : 1 + x;
}

// Leading dimensions.  A: lda = 1 (mod 16), so the 8-byte bank of entry
// (i, j) is (i + j) mod 16 for either orientation -- the 2x2-block updates of
// one row pair k over consecutive column pairs l touch consecutive players
// and hit distinct banks.  Vt: ldv = 2 (mod 16), so the rows of consecutive
// players start in consecutive 16-byte bank groups (16-byte row alignment).
__host__ __device__ inline int jacobi_lda(int dp) { return ((dp + 15) & ~15) + 1; }
__host__ __device__ inline int jacobi_ldv(int dp) { return ((dp + 13) & ~15) + 2; }

// upper-triangle position of the symmetric entry {i, j}: during the sweeps only
// i <= j is stored (the strict lower triangle is refreshed on exit)
__device__ __forceinline__ int sym_at(int i, int j, int lda) {
  return i < j ? i * lda + j : j * lda + i;
}

struct JacobiScratch {
  double *A, *Vt;
  double *rc, *rs;  // [2][half] rotation cosines / sines (double buffered)
  int2 *pq;         // [2][half] players (p, q) of each pair (double buffered)
  double *tt, *lam, *red;
  int *offtab, *pos, *flag;
  int lda, ldv;
  double *dbg;  // optional off-norm history (diagnostics)
};

__host__ __device__ inline int64_t jacobi_scratch_doubles(int dp) {
  const int64_t lda = jacobi_lda(dp), ldv = jacobi_ldv(dp), half = dp / 2;
  const int64_t noff = half * (half - 1) / 2;
  const int64_t ints = noff + dp + 1 + 2;
  const int64_t n = dp * lda + dp * ldv + 4 * half + 2 * half + half + dp + 32 + (ints + 1) / 2 + 2;
  return (n + 1) & ~int64_t(1);  // keep per-warp slices 16-byte aligned
}

__device__ inline JacobiScratch jacobi_carve(double *base, int dp) {
  JacobiScratch s;
  const int half = dp / 2;
  s.lda = jacobi_lda(dp);
  s.ldv = jacobi_ldv(dp);
  s.A = base;
  s.Vt = s.A + dp * s.lda;  // dp even -> 16-byte aligned
  s.rc = s.Vt + dp * s.ldv;
  s.rs = s.rc + 2 * half;
  s.pq = reinterpret_cast<int2 *>(s.rs + 2 * half);
  s.tt = reinterpret_cast<double *>(s.pq + 2 * half);
  s.lam = s.tt + half;
  s.red = s.lam + dp;
  s.offtab = reinterpret_cast<int *>(s.red + 32);
  s.pos = s.offtab + half * (half - 1) / 2;
  s.flag = s.pos + dp + 1;
  s.dbg = nullptr;
  return s;
}

// off-block table (k, l), k < l; Vt = I (cold) with zero padding columns
template <class Team>
__device__ void jacobi_prepare(const Team &tm, JacobiScratch &js, int dp, bool init_identity) {
  const int half = dp / 2;
  for (int k = tm.rank; k < half; k += tm.size()) {
    const int base = k * (half - 1) - k * (k - 1) / 2;
    for (int l = k + 1; l < half; ++l) js.offtab[base + (l - k - 1)] = k | (l << 16);
  }
  if (init_identity)
    for (int e = tm.rank; e < dp * js.ldv; e += tm.size()) {
      const int i = e / js.ldv, j = e - i * js.ldv;
      js.Vt[e] = (i == j) ? 1.0 : 0.0;
    }
}

// min over the team, returned to every member
template <class Team>
__device__ double team_min(const Team &tm, double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (tm.size() <= 32) return v;
  const int lane = tm.rank & 31, wid = tm.rank >> 5;
  tm.sync();
  if (lane == 0) red[wid] = v;
  tm.sync();
  double r = red[0];
  const int nw = (tm.size() + 31) >> 5;
  for (int i = 1; i < nw; ++i) r = fmin(r, red[i]);
  tm.sync();
  return r;
}

// |A|_F^2 and off(A)^2 from the upper triangle
template <class Team>
__device__ void jacobi_norms(const Team &tm, const JacobiScratch &js, int dp, double &norm2,
                             double &off2) {
  double a2 = 0.0, o2 = 0.0;
  for (int e = tm.rank; e < dp * dp; e += tm.size()) {
    const int i = e / dp, j = e - i * dp;
    if (j < i) continue;
    const double a = js.A[i * js.lda + j];
    if (i == j) {
      a2 += a * a;
    } else {
      a2 += 2.0 * (a * a);
      o2 += 2.0 * (a * a);
    }
  }
  norm2 = team_sum(tm, a2, js.red);
  off2 = team_sum(tm, o2, js.red);
}

// Eigenvector-update items of one thread: item (k, c) = pair k, 16-byte column
// chunks c + j nq (j < 4) of rows p_k, q_k; consecutive threads take
// consecutive pairs (rows of consecutive players -> distinct bank groups, see
// jacobi_ldv).  The mapping is fixed for a whole solve, so the divisions are
// done once (VItems), not per round.
struct VItems {
  int k0, c0, dk, dc, total, nq, n2;
  bool on;
};

template <class Team>
__device__ __forceinline__ VItems jacobi_vitems(const Team &tm, int d, int dp, int first) {
  VItems v;
  const int T = tm.size() - first, me = tm.rank - first;
  const int half = dp / 2;
  v.n2 = (d + 1) >> 1;      // 16-byte chunks per row
  v.nq = (v.n2 + 3) >> 2;   // items per pair
  v.total = half * v.nq;
  v.on = me >= 0 && me < v.total;
  v.k0 = me >= 0 ? me % half : 0;
  v.c0 = me >= 0 ? me / half : 0;
  v.dk = T % half;
  v.dc = T / half;
  return v;
}

// Apply the rotations of parameter buffer b (one round) to the eigenvector rows.
template <class Team>
__device__ __forceinline__ void jacobi_vupdate(const Team &tm, JacobiScratch &js, int dp, int b,
                                               const VItems &vi) {
  if (!vi.on) return;
  const int half = dp / 2;
  const double *rc = js.rc + b * half, *rs = js.rs + b * half;
  const int2 *pq = js.pq + b * half;
  const int nq = vi.nq, n2 = vi.n2, ldv = js.ldv;
  int k = vi.k0, c = vi.c0;
  for (;;) {
    const double sn = rs[k], cs = rc[k];
    const int2 pk = pq[k];
    double2 *vp = reinterpret_cast<double2 *>(js.Vt + pk.x * ldv);
    double2 *vq = reinterpret_cast<double2 *>(js.Vt + pk.y * ldv);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = c + j * nq;
      if (cc < n2) {
        const double2 p0 = vp[cc], q0 = vq[cc];
        vp[cc] = make_double2(cs * p0.x - sn * q0.x, cs * p0.y - sn * q0.y);
        vq[cc] = make_double2(sn * p0.x + cs * q0.x, sn * p0.y + cs * q0.y);
      }
    }
    k += vi.dk;
    c += vi.dc;
    if (k >= half) {
      k -= half;
      ++c;
    }
    if (c * half + k >= vi.total) break;
  }
}

// Cyclic Jacobi on the symmetric A (dp x dp, padded); rotations accumulate
// into the rows of Vt.  Only the upper triangle is maintained during the
// sweeps; the full symmetric A (diagonal = eigenvalues, off-diagonal = the
// remainder) is restored on exit.  Returns the number of sweeps performed.
template <class Team>
__device__ int jacobi_sweeps(const Team &tm, JacobiScratch &js, int d, int dp, int *order = nullptr,
                             int max_order = 0) {
  double *A = js.A;
  const int lda = js.lda, half = dp / 2, noff = half * (half - 1) / 2;
  const int T = tm.size();
  // threads that only update eigenvectors during phase P (block teams)
  const int vfirst = (T > 32 && T - ((half + 31) & ~31) >= 64) ? ((half + 31) & ~31) : 0;
  const VItems vi_p = jacobi_vitems(tm, d, dp, vfirst), vi_all = jacobi_vitems(tm, d, dp, 0);
  double norm2, off2;
  jacobi_norms(tm, js, dp, norm2, off2);
  const double thr = sqrt(norm2) * 8.673617379884035e-19;  // 2^-60 |A|_F
  const double stop2 = norm2 * 1.925929944387236e-34;      // (2^-56 |A|_F)^2
  int sweep = 0, round = 0;
  bool pending = false;
  // Perturbative exits (psd_rebuild_perturbative): with g the smallest
  // |diagonal| (no eigenvalue can change sign while off <= g / 1000), the
  // projection of D + E by its order-k expansion around D has error
  // O(off^(k+1) / g^k).  The sweeps stop at the first order whose bound is
  // below 1e-15 |A|_F -- about the rounding floor of the reconstruction
  // V diag(l+) V' itself (n eps |A|).
  if (order) *order = 0;
  const double tau = 1e-15 * sqrt(norm2);
  for (; sweep < kMaxSweeps; ++sweep) {
    if (!(off2 > stop2)) break;  // also stops on NaN
    if (order && max_order > 0) {
      double g = CUDART_INF;
      for (int i = tm.rank; i < d; i += T) g = fmin(g, fabs(A[i * lda + i]));
      g = team_min(tm, g, js.red);
      if (js.dbg) {  // diagnostics: g and the cross-class (P-N) part of off(A)
        double pn = 0.0;
        for (int e = tm.rank; e < dp * dp; e += T) {
          const int i = e / dp, j = e - i * dp;
          if (j <= i || i >= d || j >= d) continue;
          if ((A[i * lda + i] > 0.0) != (A[j * lda + j] > 0.0)) {
            const double a = A[i * lda + j];
            pn += 2.0 * (a * a);
          }
        }
        pn = team_sum(tm, pn, js.red);
        if (tm.rank == 0) {
          js.dbg[63] = g / sqrt(norm2);
          if (sweep < 20) js.dbg[40 + sweep] = sqrt(pn / norm2);
        }
      }
      if (max_order > 2 && off2 <= 0.01 * g * g) {  // class split (cta_class_split)
        *order = 3;
        break;
      }
      if (off2 <= 1e-6 * g * g) {
        const double off = sqrt(off2);
        if (off2 <= tau * g) {
          *order = 1;
          break;
        }
        if (max_order > 1 && off2 * off <= tau * g * g) {
          *order = 2;
          break;
        }
      }
    }
    if (tm.rank == 0) js.flag[0] = 0;
    tm.sync();
    for (int r = 0; r < dp - 1; ++r, ++round) {
      const int b = round & 1;
      double *rc = js.rc + b * half, *rs = js.rs + b * half;
      int2 *pq = js.pq + b * half;
      // ---- phase P: parameters of round r | eigenvector update of round r-1
      for (int k = tm.rank; k < half; k += T) {
        const int p = tour_player(k, r, dp), q = tour_player(dp - 1 - k, r, dp);
        const double apq = A[sym_at(p, q, lda)];
        double c = 1.0, s = 0.0, t = 0.0;
        if (fabs(apq) > thr) {
          const double diff = A[q * lda + q] - A[p * lda + p];
          const double rr = sqrt(diff * diff + 4.0 * apq * apq);
          t = (2.0 * apq) / (fabs(diff) + rr);
          if (diff < 0.0) t = -t;
          c = rsqrt(1.0 + t * t);
          s = t * c;
          js.flag[0] = 1;
        }
        rc[k] = c;
        rs[k] = s;
        pq[k] = make_int2(p, q);
        js.tt[k] = t;
      }
      if (pending) jacobi_vupdate(tm, js, dp, b ^ 1, vi_p);
      tm.sync();
      // ---- phase A: off-diagonal 2x2 blocks (upper triangle), then the
      // diagonal blocks
      for (int it = tm.rank; it < noff; it += T) {
        const int kl = js.offtab[it];
        const int k = kl & 0xffff, l = kl >> 16;
        const double sk = rs[k], sl = rs[l], ck = rc[k], cl = rc[l];
        const int2 PK = pq[k], PL = pq[l];
        const int i_pp = sym_at(PK.x, PL.x, lda), i_pq = sym_at(PK.x, PL.y, lda);
        const int i_qp = sym_at(PK.y, PL.x, lda), i_qq = sym_at(PK.y, PL.y, lda);
        const double a = A[i_pp], bb = A[i_pq], cc = A[i_qp], ee = A[i_qq];
        const double r_pp = ck * a - sk * cc, r_pq = ck * bb - sk * ee;
        const double r_qp = sk * a + ck * cc, r_qq = sk * bb + ck * ee;
        A[i_pp] = cl * r_pp - sl * r_pq;
        A[i_pq] = sl * r_pp + cl * r_pq;
        A[i_qp] = cl * r_qp - sl * r_qq;
        A[i_qq] = sl * r_qp + cl * r_qq;
      }
      for (int k = tm.rank; k < half; k += T) {
        const double t = js.tt[k];
        if (t == 0.0) continue;
        const int2 PK = pq[k];
        const int ipq = sym_at(PK.x, PK.y, lda);
        const double apq = A[ipq];
        A[PK.x * lda + PK.x] -= t * apq;
        A[PK.y * lda + PK.y] += t * apq;
        A[ipq] = 0.0;
      }
      pending = true;
      tm.sync();
    }
    const int rotated = js.flag[0];
    double n2;
    jacobi_norms(tm, js, dp, n2, off2);  // (team barriers inside)
    if (js.dbg && tm.rank == 0 && sweep < 63) js.dbg[1 + sweep] = sqrt(off2 / norm2);
    if (!rotated) {
      ++sweep;
      break;  // every pair below the rotation threshold
    }
  }
  if (pending) jacobi_vupdate(tm, js, dp, (round - 1) & 1, vi_all);
  // restore the strict lower triangle
  for (int e = tm.rank; e < dp * dp; e += T) {
    const int i = e / dp, j = e - i * dp;
    if (j < i) A[i * lda + j] = A[j * lda + i];
  }
  tm.sync();
  return sweep;
}

// ---------------------------------------------------------------------------
// register-tiled team GEMMs on d x d shared-memory operands.
// Thread t owns the interleaved 4x4 tiles (u, v) = (q / nt, q % nt) for
// q = t, t + T, ... (MT tiles at most): rows {u + nt a}, cols {v + nt b},
// nt = ceil(d / 4); consecutive threads read consecutive rows of R, so R
// should use an odd leading dimension.  Requires nt * nt <= MT * team size.

template <int MT>
struct GemmTiles {
  int u[MT], v[MT];
  bool on[MT];
};

template <int MT, class Team>
__device__ __forceinline__ GemmTiles<MT> gemm_tiles(const Team &tm, int nt) {
  GemmTiles<MT> g;
#pragma unroll
  for (int q = 0; q < MT; ++q) {
    const int t = tm.rank + q * tm.size();
    g.on[q] = t < nt * nt;
    g.u[q] = g.on[q] ? t / nt : 0;
    g.v[q] = g.on[q] ? t - g.u[q] * nt : 0;
  }
  return g;
}

// out = L * R'   (out[i][j] = sum_k L[i][k] R[j][k]); out may alias L or R.
template <int MT = 1, class Team>
__device__ void team_gemm_nt(const Team &tm, const double *L, int ldl, const double *R, int ldr,
                             double *out, int ldo, int d) {
  const int nt = (d + 3) >> 2;
  const GemmTiles<MT> g = gemm_tiles<MT>(tm, nt);
  double acc[MT][4][4];
#pragma unroll
  for (int q = 0; q < MT; ++q) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[q][a][b] = 0.0;
    if (g.on[q]) {
      int ri[4], rj[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        ri[a] = min(g.u[q] + nt * a, d - 1) * ldl;
        rj[a] = min(g.v[q] + nt * a, d - 1) * ldr;
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
          for (int b = 0; b < 4; ++b) acc[q][a][b] = fma(l[a], r[b], acc[q][a][b]);
      }
    }
  }
  tm.sync();
#pragma unroll
  for (int q = 0; q < MT; ++q)
    if (g.on[q]) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = g.u[q] + nt * a, j = g.v[q] + nt * b;
          if (i < d && j < d) out[i * ldo + j] = acc[q][a][b];
        }
    }
  tm.sync();
}

// P = W' V over the first r rows (P[i][j] = sum_k W[k][i] V[vrow[k]][j]),
// symmetric output: tiles with u <= v compute; every unordered pair {i, j}
// is emitted exactly once (caller mirrors).
template <int MT = 1, class Team, class Emit>
__device__ void team_gemm_tn_sym(const Team &tm, const double *W, int ldw, const double *V,
                                 int ldv, const int *vrow, int r, int d, Emit emit) {
  const int nt = (d + 3) >> 2;
  const GemmTiles<MT> g = gemm_tiles<MT>(tm, nt);
#pragma unroll
  for (int q = 0; q < MT; ++q) {
    if (!g.on[q] || g.u[q] > g.v[q]) continue;
    const int u = g.u[q], v = g.v[q];
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
      const int vk = (vrow ? vrow[k] : k) * ldv;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        w[a] = W[k * ldw + ci[a]];
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
}

// compacted positive eigenvalues (warp 0 ballot, ascending position order)
template <class Team>
__device__ int compact_positive(const Team &tm, JacobiScratch &js, int d) {
  if (tm.rank < 32) {
    int base = 0;
    for (int i0 = 0; i0 < d; i0 += 32) {
      const int i = i0 + tm.rank;
      const double lam = i < d ? js.A[i * js.lda + i] : 0.0;
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
  const int ldv = js.ldv;
  const int r = compact_positive(tm, js, d);
  const int nt = (d + 3) >> 2;
  if (tm.size() <= 32 || nt * nt > tm.size()) {
    // warp teams (d <= 32) or too large for one tile per thread: direct sums
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
        acc += (js.lam[k] * js.Vt[pi * ldv + a]) * js.Vt[pi * ldv + b];
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
    W[k * js.lda + i] = js.lam[k] * js.Vt[js.pos[k] * ldv + i];
  }
  tm.sync();
  team_gemm_tn_sym(tm, W, js.lda, js.Vt, ldv, js.pos, r, d, [&](int i, int j, double v) {
    emit(i, j, v);
    if (i != j) emit(j, i, v);
  });
  tm.sync();
}

// out = L * R   (out[i][j] = sum_k L[i][k] R[k][j]); out may alias L.
template <int MT = 1, class Team>
__device__ void team_gemm_nn(const Team &tm, const double *L, int ldl, const double *R, int ldr,
                             double *out, int ldo, int d) {
  const int nt = (d + 3) >> 2;
  const GemmTiles<MT> g = gemm_tiles<MT>(tm, nt);
  double acc[MT][4][4];
#pragma unroll
  for (int q = 0; q < MT; ++q) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[q][a][b] = 0.0;
    if (g.on[q]) {
      int ri[4], cj[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        ri[a] = min(g.u[q] + nt * a, d - 1) * ldl;
        cj[a] = min(g.v[q] + nt * a, d - 1);
      }
      for (int k = 0; k < d; ++k) {
        double l[4], r[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          l[a] = L[ri[a] + k];
          r[a] = R[k * ldr + cj[a]];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[q][a][b] = fma(l[a], r[b], acc[q][a][b]);
      }
    }
  }
  tm.sync();
#pragma unroll
  for (int q = 0; q < MT; ++q)
    if (g.on[q]) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = g.u[q] + nt * a, j = g.v[q] + nt * b;
          if (i < d && j < d) out[i * ldo + j] = acc[q][a][b];
        }
    }
  tm.sync();
}

// out(i, j) = sum_k la(i, k) rb(k, j) over d x d (accessor operands); every
// read completes (team barrier) before the first emit(i, j, value).
template <int MT, class Team, class LA, class RB, class Emit>
__device__ void team_gemm_fn(const Team &tm, int d, LA la, RB rb, Emit emit) {
  const int nt = (d + 3) >> 2;
  const GemmTiles<MT> g = gemm_tiles<MT>(tm, nt);
  double acc[MT][4][4];
#pragma unroll
  for (int q = 0; q < MT; ++q) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[q][a][b] = 0.0;
    if (g.on[q]) {
      int ri[4], cj[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        ri[a] = min(g.u[q] + nt * a, d - 1);
        cj[a] = min(g.v[q] + nt * a, d - 1);
      }
      for (int k = 0; k < d; ++k) {
        double l[4], r[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          l[a] = la(ri[a], k);
          r[a] = rb(k, cj[a]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[q][a][b] = fma(l[a], r[b], acc[q][a][b]);
      }
    }
  }
  tm.sync();
#pragma unroll
  for (int q = 0; q < MT; ++q)
    if (g.on[q]) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = g.u[q] + nt * a, j = g.v[q] + nt * b;
          if (i < d && j < d) emit(i, j, acc[q][a][b]);
        }
    }
  tm.sync();
}

// fp64 tensor-core MMA (m8n8k4): D += A B, A 8 x 4 row-major, B 4 x 8.
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// CTA-team GEMM on the fp64 tensor cores: out(i, j) = sum_{k < K} la(i, k) rb(k, j)
// for i, j < d, one 8 x 8 output tile per warp at a time (fragments: a =
// A[lane/4][lane%4], b = B[lane%4][lane/4], d = D[lane/4][2 (lane%4) + {0,1}]).
// emit may not write an operand.  SYM: only tiles bi <= bj, emitted to both
// triangles (exactly symmetric).  Ends with a team barrier.
template <bool SYM, class LA, class RB, class Emit>
__device__ void mma_gemm_mn(int M, int N, int K, LA la, RB rb, Emit emit) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int mt = (M + 7) >> 3, ntc = (N + 7) >> 3, K4 = (K + 3) & ~3;
  const int ntiles = mt * ntc;
  for (int t = w; t < ntiles; t += nw) {
    const int bi = t / ntc, bj = t - bi * ntc;
    if (SYM && bi > bj) continue;
    const int ia = bi * 8 + (lane >> 2), jb = bj * 8 + (lane >> 2);
    double d0 = 0.0, d1 = 0.0;
    for (int k0 = 0; k0 < K4; k0 += 4) {
      const int k = k0 + (lane & 3);
      const double a = (ia < M && k < K) ? la(ia, k) : 0.0;
      const double b = (jb < N && k < K) ? rb(k, jb) : 0.0;
      dmma884(d0, d1, a, b);
    }
    const int i = bi * 8 + (lane >> 2), j = bj * 8 + 2 * (lane & 3);
    if (i >= M) continue;
    if (!SYM) {
      if (j < N) emit(i, j, d0);
      if (j + 1 < N) emit(i, j + 1, d1);
    } else if (bi < bj) {
      if (j < N) {
        emit(i, j, d0);
        emit(j, i, d0);
      }
      if (j + 1 < N) {
        emit(i, j + 1, d1);
        emit(j + 1, i, d1);
      }
    } else {
      if (j < N && i <= j) {
        emit(i, j, d0);
        if (i != j) emit(j, i, d0);
      }
      if (j + 1 < N && i <= j + 1) {
        emit(i, j + 1, d1);
        if (i != j + 1) emit(j + 1, i, d1);
      }
    }
  }
  __syncthreads();
}

template <bool SYM, class LA, class RB, class Emit>
__device__ void mma_gemm(int d, int K, LA la, RB rb, Emit emit) {
  mma_gemm_mn<SYM>(d, d, K, la, rb, emit);
}

// Second-order projection of a nearly diagonal B = D + E (Daleckii-Krein to
// second order, f = max(., 0), P / N = positive / non-positive diagonal):
//   M_PP = D_P + E_PP - T1,  M_NN = -T1,
//   M_PN = l_i G_ij + (-l_j T2_ij + l_i T3_ij) / (l_i - l_j)      (i in P, j in N)
// with G_ij = E_ij / (l_i - l_j) on the P-N entries (0 elsewhere), E_S the
// same-class entries of E, T1 = G |L| G, T2 = E_S G, T3 = G E_S; error
// O(|E|^3 / g^2).  Every denominator is >= 2 g.  A holds E_S + G (its
// diagonal in lam); M is assembled in the global scratch Mg (d x d), then
// P = V' M V by two team GEMMs.
template <int MT, class Team, class Emit>
__device__ void psd_rebuild_second_order(const Team &tm, JacobiScratch &js, int d, double *Mg, Emit emit) {
  double *A = js.A;
  const int lda = js.lda, ldv = js.ldv;
  double *lam = js.lam;
  for (int i = tm.rank; i < d; i += tm.size()) lam[i] = A[i * lda + i];
  tm.sync();
  for (int e = tm.rank; e < d * d; e += tm.size()) {
    const int i = e / d, j = e - i * d;
    const double li = lam[i], lj = lam[j];
    if (i == j) A[i * lda + j] = 0.0;
    else if ((li > 0.0) != (lj > 0.0)) A[i * lda + j] = A[i * lda + j] / (li - lj);
  }
  tm.sync();
  auto cls = [&](int i) { return lam[i] > 0.0; };
  auto g_of = [&](int i, int k) { return cls(i) != cls(k) ? A[i * lda + k] : 0.0; };
  auto s_of = [&](int i, int k) { return cls(i) == cls(k) ? A[i * lda + k] : 0.0; };
  // T1 on the same-class entries
  team_gemm_fn<MT>(
      tm, d, g_of, [&](int k, int j) { return fabs(lam[k]) * g_of(k, j); },
      [&](int i, int j, double t1) {
        if (cls(i) != cls(j)) return;
        double base = 0.0;
        if (i == j) base = lam[i] > 0.0 ? lam[i] : 0.0;
        else if (cls(i)) base = A[i * lda + j];
        Mg[i * d + j] = base - t1;
      });
  // T2, then T3, on the P x N entries (mirrored into N x P)
  team_gemm_fn<MT>(tm, d, s_of, g_of, [&](int i, int j, double t2) {
    if (!cls(i) || cls(j)) return;
    Mg[i * d + j] = lam[i] * A[i * lda + j] - lam[j] * t2 / (lam[i] - lam[j]);
  });
  team_gemm_fn<MT>(tm, d, g_of, s_of, [&](int i, int j, double t3) {
    if (!cls(i) || cls(j)) return;
    const double v = Mg[i * d + j] + lam[i] * t3 / (lam[i] - lam[j]);
    Mg[i * d + j] = v;
    Mg[j * d + i] = v;
  });
  for (int e = tm.rank; e < d * d; e += tm.size()) {
    const int i = e / d, j = e - i * d;
    A[i * lda + j] = Mg[i * d + j];
  }
  tm.sync();
  team_gemm_nn<MT>(tm, A, lda, js.Vt, ldv, A, lda, d);  // T = M Vt
  team_gemm_tn_sym<MT>(tm, js.Vt, ldv, A, lda, nullptr, d, d, [&](int i, int j, double v) {
    emit(i, j, v);
    if (i != j) emit(j, i, v);
  });
  tm.sync();
}

// First-order projection of a nearly diagonal B = D + E (CTA teams):
//   P(B) = P(D) + L_D(E) + O(|E|^2 / g),  L_D(E)_ij = E_ij (l_i+ - l_j+) / (l_i - l_j)
// (the Frechet derivative of the spectral function max(., 0); the divided
// difference is 1 between positive, 0 between non-positive eigenvalues), g the
// smallest |l_i|.  It is exact within same-sign pairs; jacobi_sweeps selects it
// when |E|_F^2 <= 1e-15 |A|_F g and |E|_F <= g / 1000.  P = V' M V with
// M = diag(l+) + L_D(E) by two team GEMMs.
template <int MT, class Team, class Emit>
__device__ void psd_rebuild_first_order(const Team &tm, JacobiScratch &js, int d, Emit emit) {
  double *A = js.A;
  const int lda = js.lda, ldv = js.ldv;
  for (int i = tm.rank; i < d; i += tm.size()) js.lam[i] = A[i * lda + i];
  tm.sync();
  for (int e = tm.rank; e < d * d; e += tm.size()) {
    const int i = e / d, j = e - i * d;
    const double li = js.lam[i], lj = js.lam[j];
    double m;
    if (i == j) {
      m = li > 0.0 ? li : 0.0;
    } else {
      double dd;
      if (li > 0.0 && lj > 0.0) dd = 1.0;
      else if (li <= 0.0 && lj <= 0.0) dd = 0.0;
      else dd = (fmax(li, 0.0) - fmax(lj, 0.0)) / (li - lj);
      m = A[i * lda + j] * dd;
    }
    A[i * lda + j] = m;  // each element read and written by one thread
  }
  tm.sync();
  team_gemm_nn<MT>(tm, A, lda, js.Vt, ldv, A, lda, d);  // T = M Vt
  team_gemm_tn_sym<MT>(tm, js.Vt, ldv, A, lda, nullptr, d, d, [&](int i, int j, double v) {
    emit(i, j, v);
    if (i != j) emit(j, i, v);
  });
  tm.sync();
}

// ---------------------------------------------------------------------------
// CTA teams: the dense products on the fp64 tensor cores (mma_gemm), with the
// per-CTA global scratch Mg (d x d, L2-resident) as the intermediate so no
// GEMM writes an operand.

// B = V X V' from the previous eigenvectors (rows of Vt): T = Vt X -> Mg, B = T Vt'
__device__ void cta_warm_start(JacobiScratch &js, int d, double *Mg) {
  double *A = js.A, *Vt = js.Vt;
  const int lda = js.lda, ldv = js.ldv;
  mma_gemm<false>(
      d, d, [&](int i, int k) { return Vt[i * ldv + k]; }, [&](int k, int j) { return A[k * lda + j]; },
      [&](int i, int j, double v) { Mg[i * d + j] = v; });
  mma_gemm<true>(
      d, d, [&](int i, int k) { return Mg[i * d + k]; }, [&](int k, int j) { return Vt[j * ldv + k]; },
      [&](int i, int j, double v) { A[i * lda + j] = v; });
}

// P = sum_{lambda > 0} lambda v v' (converged sweeps)
template <class Emit>
__device__ void cta_rebuild_full(const BlockTeam &tm, JacobiScratch &js, int d, Emit emit) {
  const int r = compact_positive(tm, js, d);
  double *W = js.A, *Vt = js.Vt;
  const int lda = js.lda, ldv = js.ldv;
  for (int e = tm.rank; e < r * d; e += tm.size()) {
    const int k = e / d, i = e - k * d;
    W[k * lda + i] = js.lam[k] * Vt[js.pos[k] * ldv + i];
  }
  tm.sync();
  const int *pos = js.pos;
  mma_gemm<true>(
      d, r, [&](int i, int k) { return W[k * lda + i]; }, [&](int k, int j) { return Vt[pos[k] * ldv + j]; },
      emit);
}

// P = V M V' with M = D+ + L1(E) (order 1) or + L2(E, E) (order 2), see
// psd_rebuild_first_order / psd_rebuild_second_order
template <class Emit>
__device__ void cta_rebuild_perturbative(const BlockTeam &tm, JacobiScratch &js, int d, int order, double *Mg,
                                         Emit emit) {
  double *A = js.A, *Vt = js.Vt, *lam = js.lam;
  const int lda = js.lda, ldv = js.ldv;
  for (int i = tm.rank; i < d; i += tm.size()) lam[i] = A[i * lda + i];
  tm.sync();
  if (order == 1) {
    for (int e = tm.rank; e < d * d; e += tm.size()) {
      const int i = e / d, j = e - i * d;
      const double li = lam[i], lj = lam[j];
      double m;
      if (i == j) {
        m = li > 0.0 ? li : 0.0;
      } else {
        double dd;
        if (li > 0.0 && lj > 0.0) dd = 1.0;
        else if (li <= 0.0 && lj <= 0.0) dd = 0.0;
        else dd = (fmax(li, 0.0) - fmax(lj, 0.0)) / (li - lj);
        m = A[i * lda + j] * dd;
      }
      A[i * lda + j] = m;
    }
    tm.sync();
  } else {
    // class-sorted order (positive first): pos[0, r) = P, pos[r, d) = N; the
    // P-N entries of E become G, the same-class ones stay, all into Mg
    int *perm = js.pos;
    int r = 0;
    if (tm.rank < 32) {
      int base = 0;
      for (int pass = 0; pass < 2; ++pass)
        for (int i0 = 0; i0 < d; i0 += 32) {
          const int i = i0 + tm.rank;
          const bool pk = i < d && ((lam[i] > 0.0) == (pass == 0));
          const unsigned mk = __ballot_sync(0xffffffffu, pk);
          if (pk) perm[base + __popc(mk & ((1u << tm.rank) - 1u))] = i;
          base += __popc(mk);
          if (pass == 0 && i0 + 32 >= d && tm.rank == 0) perm[d] = base;
        }
    }
    tm.sync();
    r = perm[d];
    for (int e = tm.rank; e < d * d; e += tm.size()) {
      const int i = e / d, j = e - i * d;
      const int pi = perm[i], pj = perm[j];
      double v = 0.0;
      if (i != j) {
        v = A[pi * lda + pj];
        if ((i < r) != (j < r)) v /= (lam[pi] - lam[pj]);
      }
      Mg[i * d + j] = v;
    }
    tm.sync();
    const int n = d - r;
    // M (sorted) into A:  M_PP = D_P + E_PP - G_PN |L_N| G_NP
    mma_gemm_mn<false>(
        r, r, n, [&](int i, int k) { return Mg[i * d + r + k]; },
        [&](int k, int j) { return fabs(lam[perm[r + k]]) * Mg[(r + k) * d + j]; },
        [&](int i, int j, double t1) {
          const double base = (i == j) ? lam[perm[i]] : Mg[i * d + j];
          A[i * lda + j] = base - t1;
        });
    //                  M_NN = -G_NP L_P G_PN
    mma_gemm_mn<false>(
        n, n, r, [&](int i, int k) { return Mg[(r + i) * d + k]; },
        [&](int k, int j) { return lam[perm[k]] * Mg[k * d + r + j]; },
        [&](int i, int j, double t1) { A[(r + i) * lda + r + j] = -t1; });
    //                  M_PN = l_i G + (-l_j E_PP G + l_i G E_NN) / (l_i - l_j)
    mma_gemm_mn<false>(
        r, n, r, [&](int i, int k) { return Mg[i * d + k]; }, [&](int k, int j) { return Mg[k * d + r + j]; },
        [&](int i, int j, double t2) {
          const double li = lam[perm[i]], lj = lam[perm[r + j]];
          A[i * lda + r + j] = li * Mg[i * d + r + j] - lj * t2 / (li - lj);
        });
    mma_gemm_mn<false>(
        r, n, n, [&](int i, int k) { return Mg[i * d + r + k]; },
        [&](int k, int j) { return Mg[(r + k) * d + r + j]; },
        [&](int i, int j, double t3) {
          const double li = lam[perm[i]], lj = lam[perm[r + j]];
          const double v = A[i * lda + r + j] + li * t3 / (li - lj);
          A[i * lda + r + j] = v;
          A[(r + j) * lda + i] = v;
        });
    // T = M Vt(perm) -> Mg, P = Vt(perm)' T
    mma_gemm<false>(
        d, d, [&](int i, int k) { return A[i * lda + k]; },
        [&](int k, int j) { return Vt[perm[k] * ldv + j]; }, [&](int i, int j, double v) { Mg[i * d + j] = v; });
    mma_gemm<true>(
        d, d, [&](int i, int k) { return Vt[perm[k] * ldv + i]; }, [&](int k, int j) { return Mg[k * d + j]; },
        emit);
    return;
  }
  // T = M Vt -> Mg, P = Vt' T
  mma_gemm<false>(
      d, d, [&](int i, int k) { return A[i * lda + k]; }, [&](int k, int j) { return Vt[k * ldv + j]; },
      [&](int i, int j, double v) { Mg[i * d + j] = v; });
  mma_gemm<true>(
      d, d, [&](int i, int k) { return Vt[k * ldv + i]; }, [&](int k, int j) { return Mg[k * d + j]; }, emit);
}

// ---------------------------------------------------------------------------
// Class-split exit (CTA teams, warm hot path): exact projection without a
// Jacobi sweep when B = V' X V is close to diagonal.
//
// With the diagonal classes P (l > 0, r of them) and N (n = d - r) in sorted
// order, the positive invariant subspace of B is span [I; X] (X: n x r), the
// solution near 0 of the Riccati equation
//     X L_P - L_N X = B_NP + E_NN X - X (E_PP + B_PN X)
// (L = diagonal, E = off-diagonal within a class).  Every denominator
// l_j - l_i (j in P, i in N) is >= 2g, g = min |l|, so the fixed-point
// iteration contracts at about off(B) / 2g whatever the within-class
// spacing; within-class coupling never has to be rotated away.  With
// Z_P = [I; X] (I + X'X)^-1/2 and Z_N = [-X'; I] (I + XX')^-1/2 (exact
// orthonormal bases of the two invariant subspaces; the inverse square roots
// by their binomial series, |X'X| <= (off / 2g)^2),
//     P = V'_P C V'_P',   V'_P = V Z_P,   C = Z_P' B Z_P = S_P (I + X'X) R S_P,
// R = L_P + E_PP + B_PN X  (B [I; X] = [I; X] R), and V' = V [Z_P, Z_N] is
// the next warm start.  No truncation: the only error is the fixed point's
// (stopped at <= 2.5e-16) and rounding.  Taken when off(B) <= g / 10 (then no
// eigenvalue changes sign, Weyl); otherwise, or if the iteration stalls, the
// caller runs the sweeps.

constexpr int kSplitMaxIter = 14;

// one m8n8k4 output tile t of out(i, j) = sum_k la(i, k) rb(k, j) (M x N)
template <class LA, class RB, class Emit>
__device__ __forceinline__ void mma_tile(int t, int M, int N, int K, LA la, RB rb, Emit emit, int lane) {
  const int ntc = (N + 7) >> 3;
  const int bi = t / ntc, bj = t - bi * ntc;
  const int ia = bi * 8 + (lane >> 2), jb = bj * 8 + (lane >> 2);
  double d0 = 0.0, d1 = 0.0;
  const int K4 = (K + 3) & ~3;
  for (int k0 = 0; k0 < K4; k0 += 4) {
    const int k = k0 + (lane & 3);
    const double a = (ia < M && k < K) ? la(ia, k) : 0.0;
    const double b = (jb < N && k < K) ? rb(k, jb) : 0.0;
    dmma884(d0, d1, a, b);
  }
  const int i = bi * 8 + (lane >> 2), j = bj * 8 + 2 * (lane & 3);
  if (i >= M) return;
  if (j < N) emit(i, j, d0);
  if (j + 1 < N) emit(i, j + 1, d1);
}

// two independent GEMMs in one pass (one barrier)
template <class LA1, class RB1, class E1, class LA2, class RB2, class E2>
__device__ void mma_gemm_dual(int M1, int N1, int K1, LA1 la1, RB1 rb1, E1 e1, int M2, int N2, int K2, LA2 la2,
                              RB2 rb2, E2 e2) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int t1 = ((M1 + 7) >> 3) * ((N1 + 7) >> 3), t2 = ((M2 + 7) >> 3) * ((N2 + 7) >> 3);
  for (int t = w; t < t1 + t2; t += nw) {
    if (t < t1) mma_tile(t, M1, N1, K1, la1, rb1, e1, lane);
    else mma_tile(t - t1, M2, N2, K2, la2, rb2, e2, lane);
  }
  __syncthreads();
}

// Mg: 5 d x d regions.  vst: the clique's eigenvector store (row c = basis
// vector c).  Returns false (nothing emitted, vst and A untouched) when the
// split does not apply; js.Vt is used as scratch either way.
template <class Emit>
__device__ bool cta_class_split(const BlockTeam &tm, JacobiScratch &js, int d, double *Mg, double *vst, Emit emit) {
  double *A = js.A, *lam = js.lam;
  const int lda = js.lda;
  double g = CUDART_INF, o2 = 0.0;
  for (int e = tm.rank; e < d * d; e += tm.size()) {
    const int i = e / d, j = e - i * d;
    const double a = A[i * lda + j];
    if (i == j) {
      lam[i] = a;
      g = fmin(g, fabs(a));
    } else {
      o2 += a * a;
    }
  }
  g = team_min(tm, g, js.red);
  o2 = team_sum(tm, o2, js.red);
  if (js.dbg && tm.rank == 0) js.dbg[62] = sqrt(o2) / g;
  if (!(g > 0.0) || !(o2 <= 0.01 * g * g)) return false;  // also NaN
  // class-sorted order: perm[0, r) = P, perm[r, d) = N
  int *perm = js.pos;
  if (tm.rank < 32) {
    int base = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (int i0 = 0; i0 < d; i0 += 32) {
        const int i = i0 + tm.rank;
        const bool pk = i < d && ((lam[i] > 0.0) == (pass == 0));
        const unsigned mk = __ballot_sync(0xffffffffu, pk);
        if (pk) perm[base + __popc(mk & ((1u << tm.rank) - 1u))] = i;
        base += __popc(mk);
        if (pass == 0 && i0 + 32 >= d && tm.rank == 0) perm[d] = base;
      }
  }
  tm.sync();
  const int r = perm[d], n = d - r;
  const int64_t dd = (int64_t)d * d;
  double *Y = Mg, *YP = Mg + dd, *YN = YP + r * r, *SA = Mg + 2 * dd, *SB = Mg + 3 * dd, *R4 = Mg + 4 * dd;
  double *X0 = js.Vt, *X1 = js.Vt + n * r;
  auto bt = [&](int i, int j) { return A[perm[i] * lda + perm[j]]; };  // sorted B
  // ---- Riccati fixed point from X1 = B_NP / Delta
  double x2 = 0.0;
  for (int e = tm.rank; e < n * r; e += tm.size()) {
    const int i = e / r, j = e - i * r;
    const double x = bt(r + i, j) / (lam[perm[j]] - lam[perm[r + i]]);
    X0[e] = x;
    x2 += x * x;
  }
  double prev = sqrt(team_sum(tm, x2, js.red));  // (barriers inside)
  bool ok = prev == 0.0;
  int it = 0;
  for (; !ok && it < kSplitMaxIter; ++it) {
    // Y = E_PP + B_PN X
    mma_gemm_mn<false>(
        r, r, n, [&](int i, int k) { return bt(i, r + k); }, [&](int k, int j) { return X0[k * r + j]; },
        [&](int i, int j, double v) { Y[i * r + j] = v + (i != j ? bt(i, j) : 0.0); });
    // X' = (B_NP + [E_NN | X] [X; -Y]) / Delta
    double acc = 0.0;
    mma_gemm_mn<false>(
        n, r, d,
        [&](int i, int k) { return k < n ? (k != i ? bt(r + i, r + k) : 0.0) : X0[i * r + (k - n)]; },
        [&](int k, int j) { return k < n ? X0[k * r + j] : -Y[(k - n) * r + j]; },
        [&](int i, int j, double v) {
          const int pi = perm[r + i], pj = perm[j];
          const double x = (A[pi * lda + pj] + v) / (lam[pj] - lam[pi]);
          const double dx = x - X0[i * r + j];
          acc += dx * dx;
          X1[i * r + j] = x;
        });
    const double delta = sqrt(team_sum(tm, acc, js.red));
    double *t = X0;
    X0 = X1;
    X1 = t;
    const double rho = delta / prev;
    if (delta == 0.0 || (rho < 0.5 && delta * rho <= 2.5e-16 * (1.0 - rho))) ok = true;
    else if (!(rho < 0.5)) break;  // stalled (or NaN): let the sweeps handle it
    prev = delta;
  }
  if (js.dbg && tm.rank == 0) js.dbg[60] = ok ? it : -1.0 - it;
  if (!ok) return false;
  // R - L_P = E_PP + B_PN X with the final X
  mma_gemm_mn<false>(
      r, r, n, [&](int i, int k) { return bt(i, r + k); }, [&](int k, int j) { return X0[k * r + j]; },
      [&](int i, int j, double v) { Y[i * r + j] = v + (i != j ? bt(i, j) : 0.0); });
  // ---- Y_P = X'X, Y_N = XX' (|Y_P|_F = |Y_N|_F sizes the series)
  double acc = 0.0;
  mma_gemm_dual(
      r, r, n, [&](int i, int k) { return X0[k * r + i]; }, [&](int k, int j) { return X0[k * r + j]; },
      [&](int i, int j, double v) {
        YP[i * r + j] = v;
        acc += v * v;
      },
      n, n, r, [&](int i, int k) { return X0[i * r + k]; }, [&](int k, int j) { return X0[j * r + k]; },
      [&](int i, int j, double v) { YN[i * n + j] = v; });
  const double y = sqrt(team_sum(tm, acc, js.red));
  // (1 + y)^-1/2 = sum c_k y^k, c_k = c_{k-1} (-(2k - 1) / 2k): terms while y^k > 1e-17
  int K = 0;
  if (y > 0.0) {
    double p = y;
    while (K < 24 && p > 1e-17) {
      ++K;
      p *= y;
    }
  }
  double cK = 1.0;
  for (int k = 1; k <= K; ++k) cK *= -(2.0 * k - 1.0) / (2.0 * k);
  // Horner: S = c_K I; S <- c_k I + Y S
  double *SP = SA, *SN = SA + r * r, *TP = SB, *TN = SB + r * r;
  for (int e = tm.rank; e < r * r + n * n; e += tm.size()) {
    const bool inP = e < r * r;
    const int q = inP ? e : e - r * r, m = inP ? r : n;
    const int i = q / m, j = q - i * m;
    SA[e] = (i == j) ? cK : 0.0;
  }
  tm.sync();
  double c = cK;
  for (int k = K - 1; k >= 0; --k) {
    c *= -(2.0 * (k + 1)) / (2.0 * (k + 1) - 1.0);  // c_k from c_{k+1}
    mma_gemm_dual(
        r, r, r, [&](int i, int q) { return YP[i * r + q]; }, [&](int q, int j) { return SP[q * r + j]; },
        [&](int i, int j, double v) { TP[i * r + j] = v + (i == j ? c : 0.0); },
        n, n, n, [&](int i, int q) { return YN[i * n + q]; }, [&](int q, int j) { return SN[q * n + j]; },
        [&](int i, int j, double v) { TN[i * n + j] = v + (i == j ? c : 0.0); });
    double *t = SP;
    SP = TP;
    TP = t;
    t = SN;
    SN = TN;
    TN = t;
  }
  // ---- [U | W] = V [[I, -X'], [X, I]] (sorted columns of V), into A
  auto vh = [&](int i, int c) { return vst[perm[c] * d + i]; };
  mma_gemm_dual(
      d, r, n, [&](int i, int k) { return vh(i, r + k); }, [&](int k, int j) { return X0[k * r + j]; },
      [&](int i, int j, double v) { A[i * lda + j] = vh(i, j) + v; },
      d, n, r, [&](int i, int k) { return vh(i, k); }, [&](int k, int j) { return X0[j * r + k]; },
      [&](int i, int j, double v) { A[i * lda + r + j] = vh(i, r + j) - v; });
  // V' = [U S_P | W S_N] -> vst (rows 0..r-1: positive subspace)
  mma_gemm_dual(
      d, r, r, [&](int i, int k) { return A[i * lda + k]; }, [&](int k, int j) { return SP[k * r + j]; },
      [&](int i, int j, double v) { vst[j * d + i] = v; },
      d, n, n, [&](int i, int k) { return A[i * lda + r + k]; }, [&](int k, int j) { return SN[k * n + j]; },
      [&](int i, int j, double v) { vst[(r + j) * d + i] = v; });
  // C = S_P (I + Y_P) R S_P, R = L_P + Y
  mma_gemm_mn<false>(
      r, r, r, [&](int i, int k) { return YP[i * r + k] + (i == k ? 1.0 : 0.0); },
      [&](int k, int j) { return Y[k * r + j] + (k == j ? lam[perm[j]] : 0.0); },
      [&](int i, int j, double v) { R4[i * r + j] = v; });
  mma_gemm_mn<false>(
      r, r, r, [&](int i, int k) { return SP[i * r + k]; }, [&](int k, int j) { return R4[k * r + j]; },
      [&](int i, int j, double v) { YP[i * r + j] = v; });
  mma_gemm_mn<true>(
      r, r, r, [&](int i, int k) { return YP[i * r + k]; }, [&](int k, int j) { return SP[k * r + j]; },
      [&](int i, int j, double v) { R4[i * r + j] = v; });
  // P = (V'_P C) V'_P'
  mma_gemm_mn<false>(
      d, r, r, [&](int i, int k) { return vst[k * d + i]; }, [&](int k, int j) { return R4[k * r + j]; },
      [&](int i, int j, double v) { A[i * lda + j] = v; });
  mma_gemm<true>(
      d, r, [&](int i, int k) { return A[i * lda + k]; }, [&](int k, int j) { return vst[k * d + j]; }, emit);
  return true;
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
  double *pscratch; // CTA teams: d x d global scratch per CTA (second-order rebuild)
  int64_t pstride;
  int slot;         // this team's scratch slot
  int split_refresh; // k_cone_split: fixed-point iterations beyond which V is refreshed
  int split_vupdate; // k_cone_split: rotate V onto the new invariant subspaces
  int *cfail;        // cold path (hsde_cold.cuh): [count] 1 = handed to the Jacobi path
  int fail_only;     // k_cone_block: only the slots flagged in cfail (HOT: raw X in W.xarg)
  int cold;          // k_cone_split: hand-overs go to the cold path (X kept in W.xarg)
  int cold_pass;     // k_cone_cold after k_cone_split: 0 the predicted cliques (W.ccur), 1 its hand-overs
  int pf_ahead;      // k_cone_split: resident CTA slots (0 = off); slot b prefetches the inputs of slot b + pf_ahead into L2
  double pol_f2c;    // fast path -> cold next iteration when off(B)^2 > pol_f2c g^2 (default 0.1225: off > 0.35 g)
  double pol_c2f;    // cold path -> fast next iteration when |X - X_prev|_F^2 <= pol_c2f g^2 (default 0.36: |dX| <= 0.6 g)
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
  const int lda = js.lda, ldv = js.ldv;
  double *A = js.A;
  constexpr bool kCta = std::is_same<Team, BlockTeam>::value;
  // k_cone_split ran first for CTA cliques on the hot path (hsde_split.cuh)
  int cst = SPLIT_UNTOUCHED;
  if (MODE == CONE_HOT && kCta && W.cstate) {
    cst = W.cstate[k];
    // finished by the fast path (also after a refresh, SPLIT_DONE + 16) or here
    if (cst == SPLIT_DONE || cst >= SPLIT_DONE + 16) return;
  }
  const bool xcold = MODE == CONE_HOT && ca.fail_only;  // cold-path failure: raw X in W.xarg
  const bool handoff = !xcold && cst >= SPLIT_HANDOFF;  // A <- B = Vt X Vt' from W.xarg
  const int age = (MODE == CONE_HOT && ca.warm) ? (W.vvalid[k] & ~kVRefresh) : 0;
  constexpr int MT = TeamTiles<Team>::value;
  const int ntile = (d + 3) >> 2;
  const bool warm = handoff || (!xcold && age > 0 && age < kWarmMaxAge && ntile * ntile <= MT * tm.size());
  if (MODE == CONE_HOT && W.dbg && k == W.dbg_clique) {
    js.dbg = W.dbg;
    if (tm.rank == 0) {
      for (int i = 0; i < 64; ++i) W.dbg[i] = -1.0;
      W.dbg[0] = warm ? 1.0 : 0.0;
    }
  }
  jacobi_prepare(tm, js, dp, !warm);
  // load (raw) and the previous eigenvectors (warm)
  for (int e = tm.rank; e < d * d; e += tm.size()) {
    const int a = e / d, bcol = e - a * d;
    double v;
    if (MODE == CONE_HOT) v = (handoff || xcold) ? W.xarg[off + e] : hot_slot_load(P, S, W, off + e, shift);
    else v = ca.in[off + e] * ca.in_scale;
    A[a * lda + bcol] = v;
    if (warm) js.Vt[a * ldv + bcol] = W.vstore[off + e];
  }
  if (d & 1) {
    for (int e = tm.rank; e < dp; e += tm.size()) {
      A[d * lda + e] = 0.0;
      A[e * lda + d] = 0.0;
    }
  }
  if (warm) {
    // zero padding columns / dummy row of Vt (identity on the dummy)
    for (int e = tm.rank; e < dp * ldv; e += tm.size()) {
      const int i = e / ldv, j = e - i * ldv;
      if (i >= d || j >= d) js.Vt[e] = (i == j) ? 1.0 : 0.0;
    }
  }
  tm.sync();
  // sym = 0.5 (B + B')  (symmat.py:157)
  for (int e = tm.rank; e < d * d; e += tm.size()) {
    const int a = e / d, bcol = e - a * d;
    if (a < bcol) {
      const double s = 0.5 * (A[a * lda + bcol] + A[bcol * lda + a]);
      A[a * lda + bcol] = s;
      A[bcol * lda + a] = s;
    }
  }
  tm.sync();
  double *Mg = ca.pscratch ? ca.pscratch + (int64_t)ca.slot * ca.pstride : nullptr;
  if (handoff) {
    // B already in A
  } else if (kCta && warm && Mg) {
    cta_warm_start(js, d, Mg);
  } else if (warm) {
    // B = V X V' (rows of Vt are the previous eigenvectors): T1 = Vt X, then
    // B' = Vt T1' (= B for symmetric X) with the odd-ld operand on the right
    team_gemm_nt<MT>(tm, js.Vt, ldv, A, lda, A, lda, d);
    team_gemm_nt<MT>(tm, js.Vt, ldv, A, lda, A, lda, d);
    for (int e = tm.rank; e < d * d; e += tm.size()) {
      const int a = e / d, bcol = e - a * d;
      if (a < bcol) {
        const double s = 0.5 * (A[a * lda + bcol] + A[bcol * lda + a]);
        A[a * lda + bcol] = s;
        A[bcol * lda + a] = s;
      }
    }
    tm.sync();
  }
  // first-order exit for CTA teams whose GEMM tiles fit (not for MINEIG)
  int order = 0;
  const bool fo_ok = MODE != CONE_MINEIG && (Mg || ntile * ntile <= MT * tm.size());
  // class split (CTA teams, hot path with the eigenvector store): exact exit
  // as soon as off(B) <= g / 10, after 0 sweeps (warm) or a few (cold)
  bool split_ok = kCta && MODE == CONE_HOT && ca.warm && Mg != nullptr;
  int sw = 0;
  for (;;) {
    sw += jacobi_sweeps(tm, js, d, dp, fo_ok ? &order : nullptr, fo_ok ? (Mg ? (split_ok ? 3 : 2) : 1) : 0);
    if constexpr (kCta) {
      if (order == 3) {
        // the split reads V from the store and uses js.Vt as scratch
        for (int e = tm.rank; e < d * d; e += tm.size()) {
          const int a = e / d, bcol = e - a * d;
          W.vstore[off + e] = js.Vt[a * ldv + bcol];
        }
        tm.sync();
        auto emit_split = [&](int a, int bcol, double v) {
          const int64_t j = so + off + (int64_t)a * d + bcol;
          S.u[j] = v;
          S.w[j] += v;
        };
        if (cta_class_split(tm, js, d, Mg, W.vstore + off, emit_split)) {
          if (tm.rank == 0) {
            W.vvalid[k] = warm ? age + 1 : 1;
            if (W.sweeps) W.sweeps[k] = sw;
          }
          return;
        }
        // stalled: restore Vt and continue sweeping without the split
        for (int e = tm.rank; e < dp * ldv; e += tm.size()) {
          const int i = e / ldv, j = e - i * ldv;
          js.Vt[e] = (i < d && j < d) ? W.vstore[off + (int64_t)i * d + j] : (i == j ? 1.0 : 0.0);
        }
        tm.sync();
        split_ok = false;
        order = 0;
        continue;
      }
    }
    break;
  }
  if (MODE == CONE_HOT && tm.rank == 0 && W.sweeps) W.sweeps[k] = sw;
  // non-finite eigenvalue -> EigenFailure (symmat.py:162-163)
  double nb = 0.0;
  for (int i = tm.rank; i < d; i += tm.size()) nb += isfinite(A[i * lda + i]) ? 0.0 : 1.0;
  const bool bad = team_sum(tm, nb, js.red) > 0.0;
  if (bad && tm.rank == 0) atomicOr(W.err, 1);
  if (MODE == CONE_MINEIG) {
    double mn = CUDART_INF;
    for (int i = 0; i < d; ++i) mn = fmin(mn, A[i * lda + i]);
    if (tm.rank == 0) ca.out[k] = mn;
    tm.sync();
    return;
  }
  if (MODE == CONE_HOT && ca.warm) {
    for (int e = tm.rank; e < d * d; e += tm.size()) {
      const int a = e / d, bcol = e - a * d;
      W.vstore[off + e] = js.Vt[a * ldv + bcol];
    }
    if (tm.rank == 0) W.vvalid[k] = bad ? 0 : (warm ? age + 1 : 1);
  }
  auto emit_hot = [&](int a, int bcol, double v) {
    const int64_t j = so + off + (int64_t)a * d + bcol;
    S.u[j] = v;
    S.w[j] += v;
  };
  auto emit_plain = [&](int a, int bcol, double v) { ca.out[off + (int64_t)a * d + bcol] = v; };
  if constexpr (kCta) {
    if (Mg) {
      if (order > 0) {
        if (MODE == CONE_HOT) cta_rebuild_perturbative(tm, js, d, order, Mg, emit_hot);
        else cta_rebuild_perturbative(tm, js, d, order, Mg, emit_plain);
      } else {
        if (MODE == CONE_HOT) cta_rebuild_full(tm, js, d, emit_hot);
        else cta_rebuild_full(tm, js, d, emit_plain);
      }
      return;
    }
  }
  if (order == 2) {
    if (MODE == CONE_HOT) psd_rebuild_second_order<MT>(tm, js, d, Mg, emit_hot);
    else psd_rebuild_second_order<MT>(tm, js, d, Mg, emit_plain);
  } else if (order == 1) {
    if (MODE == CONE_HOT) psd_rebuild_first_order<MT>(tm, js, d, emit_hot);
    else psd_rebuild_first_order<MT>(tm, js, d, emit_plain);
  } else {
    if (MODE == CONE_HOT) psd_rebuild(tm, js, d, emit_hot);
    else psd_rebuild(tm, js, d, emit_plain);
  }
}

constexpr int kConeBlock = 512;  // threads per CTA team (d > 32)

// one warp per clique (d <= 32); dynamic smem = warps * scratch(dpmax)
template <int MODE>
__global__ void __launch_bounds__(kBlock) k_cone_warp(DevProblem P, DevState S, DevWork W, ConeArgs ca) {
  extern __shared__ __align__(16) double smem[];
  const int wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + wid;
  if (gw >= ca.count) return;
  if (ca.fail_only && !ca.cfail[gw]) return;  // after the warp cold path: its failures only
  double *scratch = smem + (int64_t)wid * jacobi_scratch_doubles(ca.dpmax);
  WarpTeam tm{(int)(threadIdx.x & 31)};
  ConeArgs c2 = ca;
  c2.pscratch = nullptr;  // warp teams: first order only
  cone_one<MODE>(tm, P, S, W, c2, ca.ids[gw], scratch);
}

// one CTA per clique (d > 32)
template <int MODE>
__global__ void __launch_bounds__(kConeBlock, 2) k_cone_block(DevProblem P, DevState S, DevWork W, ConeArgs ca) {
  extern __shared__ __align__(16) double smem[];
  if ((int)blockIdx.x >= ca.count) return;
  if (ca.fail_only && !ca.cfail[blockIdx.x]) return;  // after the cold path: its failures only
  BlockTeam tm{(int)threadIdx.x, (int)blockDim.x};
  ConeArgs c2 = ca;
  c2.slot = blockIdx.x;
  const int k = ca.ids[blockIdx.x];
  const int cst = (MODE == CONE_HOT && W.cstate) ? W.cstate[k] : -1;
  cone_one<MODE>(tm, P, S, W, c2, k, smem);
  // after k_cone_split: mark the cliques finished here (32 + the state they came in with)
  if (MODE == CONE_HOT && W.cstate && threadIdx.x == 0 &&
      (cst == SPLIT_UNTOUCHED || (cst >= SPLIT_HANDOFF && cst <= SPLIT_HANDOFF + 2)))
    W.cstate[k] = SPLIT_DONE + 32 + cst;
}
