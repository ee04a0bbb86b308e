// hsde_cold.cuh -- cold path of the clique PSD projection for CTA-sized
// cliques (reference: chordalsdp/symmat.py:153-165 `project_psd_batch`, LAPACK
// dsyevd + einsum there): a full eigendecomposition X = V diag(lam) V' of one
// clique block per CTA, then P = V max(lam, 0) V'.
//
// One CTA of four warps per clique, three CTAs per SM (~71 KB of shared
// memory each for d = 80): the 400 cliques of config 4 run in one wave.
//
//   1. Householder tridiagonalisation in the order of LAPACK dsytd2 (lower):
//      H_s = I - tau_s v_s v_s' from column s, A <- H_s A H_s.  A lives in the
//      CTA's registers (column k in warp k % 4, row i in lane i % 32); a
//      warp's produced columns are shifted out, so the live block is always
//      its first slots and dead blocks are skipped, not masked.  Per step the
//      owner of column s (the *producer*) forms the reflector while the other
//      warps are still finishing the previous update (named barrier); the
//      partial sums of p = tau A v meet in shared memory (two CTA barriers).
//      The reflectors go to the CTA's global scratch (L2).
//   2. Eigenvalues of the tridiagonal T by bisection on each unreduced block
//      (Sturm counts by the three-term determinant recurrence: three fp64
//      operations per step, exact power-of-two rescaling; g threads per
//      eigenvalue when d is small).
//   3. Eigenvectors of T by twisted factorisations (stationary / progressive
//      qd on T - lam I, twist at min |gamma|), one thread per eigenvalue,
//      written straight into the sorted column of Z.
//   4. Back transformation V = H_0 H_1 ... H_{d-3} Z in compact-WY blocks of
//      8 reflectors (LAPACK dlarft forward): Z <- Z - W (T (W' Z)), three
//      GEMMs per block on the fp64 tensor cores (DMMA).
//   5. Newton-Schulz V <- V (3I - V'V) / 2 on DMMA (repeated while max |V'V -
//      I| > 2^-42, at most 3 times): the twisted vectors of close eigenvalues
//      are orthogonal only to ~eps |T| / gap; the kept basis feeds the warm
//      path for hundreds of iterations.
//   6. P = V_P diag(lam_P) V_P' (or X + V_N |lam_N| V_N' when the negative
//      class is the smaller one) on DMMA, upper 16 x 16 blocks mirrored.
// V is left in the per-clique store as the basis of the warm path.
//
// (included inside namespace hsde by hsde_kernels.cuh, after hsde_split.cuh)

constexpr int kColdNW = 4;
constexpr int kColdThreads = kColdNW * 32;
constexpr int kColdMaxD = 96;
constexpr int kColdNB = 8;  // reflectors per compact-WY block
constexpr int kColdLoadBatch = 4;  // hot-path slots per thread in flight (128 threads per CTA)
constexpr int kColdSturmPts = 1;  // bracket points per thread and bisection round (independent Sturm chains)

enum ColdStatus { COLD_OK = 0, COLD_FAIL = 1 };

// phase timestamps of the CTA with blockIdx.x == 0 (diagnostics: dbg[32 + i], clock64)
#define COLD_STAMP(dbg, i)                                                                 \
  do {                                                                                     \
    if ((dbg) && blockIdx.x == 0 && threadIdx.x == 0) (dbg)[32 + (i)] = (double)clock64(); \
  } while (0)

__host__ __device__ inline int cold_lv(int d) { return split_ld(d); }  // DMMA operands: 4 (mod 16)
__host__ __device__ inline int cold_rl(int d) { return (d + 31) & ~31; }
__host__ __device__ inline int64_t cold_hoff(int s, int d) {  // packed reflector s (entries s+1 .. d-1)
  return (int64_t)s * (d - 1) - (int64_t)s * (s - 1) / 2;
}
__host__ __device__ inline int64_t cold_hv_doubles(int d) { return (int64_t)d * (d - 1) / 2 + 2; }

struct ColdSmem {
  double *Z;  // d x lv: X, then Z, then V (scaled for P)
  // union: tridiagonalisation buffers / back-transformation tiles
  double *vbuf, *red, *pbuf, *dotw, *tbuf;  // [2][rl], [2][NW][rl], [rl], [2][NW], [2]
  double *Wt, *Yb, *Gb, *Tb;                // d x NB, NB x lv, NB x NB, NB x NB
  double *dg, *es, *e2, *taus, *lam, *lamu;  // [d] each (lam: sorted, unscaled)
  double *misc;                              // [8]
  int *rank, *bs, *be, *flag;
  int lv, rl;
};

__host__ __device__ inline int64_t cold_union_doubles(int d) {
  const int rl = cold_rl(d), lv = cold_lv(d);
  const int64_t tri = 2 * rl + 2 * kColdNW * rl + 2 * rl + 2 * kColdNW + 2;
  const int64_t bt = (int64_t)d * kColdNB + kColdNB * lv + 2 * kColdNB * kColdNB;
  return tri > bt ? tri : bt;
}

__host__ __device__ inline int64_t cold_smem_doubles(int d) {
  return (int64_t)d * cold_lv(d) + cold_union_doubles(d) + 6 * (int64_t)d + 8 + (3 * d + 2) / 2 + 2;
}

__device__ inline ColdSmem cold_carve(double *base, int d) {
  ColdSmem c;
  c.lv = cold_lv(d);
  c.rl = cold_rl(d);
  c.Z = base;
  double *u = c.Z + (int64_t)d * c.lv;
  c.vbuf = u;
  c.red = c.vbuf + 2 * c.rl;
  c.pbuf = c.red + 2 * kColdNW * c.rl;  // (+ colbuf [rl])
  c.dotw = c.pbuf + 2 * c.rl;
  c.tbuf = c.dotw + 2 * kColdNW;
  c.Wt = u;
  c.Yb = c.Wt + d * kColdNB;
  c.Gb = c.Yb + kColdNB * c.lv;
  c.Tb = c.Gb + kColdNB * kColdNB;
  c.dg = u + cold_union_doubles(d);
  c.es = c.dg + d;
  c.e2 = c.es + d;
  c.taus = c.e2 + d;
  c.lam = c.taus + d;
  c.lamu = c.lam + d;
  c.misc = c.lamu + d;
  c.rank = reinterpret_cast<int *>(c.misc + 8);
  c.bs = c.rank + d;
  c.be = c.bs + d;
  c.flag = c.be + d;
  return c;
}

__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// 1. tridiagonalisation.  Slot c of warp w holds column w + NW c,
// a[c][r] = A(32 r + lane, w + NW c).  Outputs dg (diagonal), es (subdiagonal
// T(s+1, s)), taus, the packed reflectors hv (global; v_s(s+1) = 1 stored).
// Dead blocks (columns <= s: slots below c0; rows <= s: chunks below r0) are
// skipped; rows <= s inside a live chunk are frozen (zero multipliers).  The
// owner of column s + 1 leaves it in colbuf while updating it, so the next
// producer reads it from shared memory instead of selecting a register slot.
// f(a[c]) for a run-time slot c in [LO, HI): a tree of warp-uniform branches
template <int LO, int HI, int MC, int MR, class F>
__device__ __forceinline__ void slot_dispatch(double (&a)[MC][MR], int c, F f) {
  if constexpr (HI - LO == 1) {
    f(a[LO]);
  } else {
    constexpr int MID = (LO + HI) / 2;
    if (c < MID) slot_dispatch<LO, MID>(a, c, f);
    else slot_dispatch<MID, HI>(a, c, f);
  }
}

template <int MC, int MR>
__device__ void cold_tridiag(double (&a)[MC][MR], int d, const ColdSmem &cs, double *hv, double *dbg) {
  constexpr int NW = kColdNW;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rl = cs.rl;
  double *colbuf = cs.pbuf + rl;  // [rl]
  if (w == 0)
#pragma unroll
    for (int r = 0; r < MR; ++r)
      if (32 * r + lane < rl) colbuf[32 * r + lane] = a[0][r];
  __syncwarp();
  int buf = 0;
  for (int s = 0; s + 2 < d; ++s) {
    double *vb = cs.vbuf + buf * rl;
    double *rb = cs.red + buf * NW * rl;
    double *db = cs.dotw + buf * NW;
    const bool stamp = dbg && s == 20 && blockIdx.x == 0 && threadIdx.x == 32;
    if (stamp) dbg[16] = (double)clock64();
    if (w == (s & (NW - 1))) {
      // producer (LAPACK dlarfg: beta = -sign(x0) |x|)
      double x[MR], sig = 0.0, x0 = 0.0, dss = 0.0;
#pragma unroll
      for (int r = 0; r < MR; ++r) {
        const int i = 32 * r + lane;
        x[r] = i < rl ? colbuf[i] : 0.0;
        if (i > s + 1 && i < d) sig = fma(x[r], x[r], sig);
        if (i == s + 1) x0 = x[r];
        if (i == s) dss = x[r];
      }
      sig = warp_allsum(sig);
      x0 = __shfl_sync(0xffffffffu, x0, (s + 1) & 31);
      dss = __shfl_sync(0xffffffffu, dss, s & 31);
      double tau = 0.0, beta = x0, scal = 0.0;
      if (sig > 0.0) {
        const double n2 = fma(x0, x0, sig), rn = rsqrt(n2), nx = n2 * rn;  // |x|, 1 / |x|
        beta = -copysign(nx, x0);
        tau = fma(fabs(x0), rn, 1.0);                   // (beta - x0) / beta
        scal = copysign(__drcp_rn(fabs(x0) + nx), x0);  // 1 / (x0 - beta)
      }
      const int64_t ho = cold_hoff(s, d);
#pragma unroll
      for (int r = 0; r < MR; ++r) {
        const int i = 32 * r + lane;
        const double v = i == s + 1 ? 1.0 : ((i > s + 1 && i < d) ? x[r] * scal : 0.0);
        if (i < rl) vb[i] = v;
        if (i > s && i < d) hv[ho + (i - s - 1)] = v;
      }
      if (lane == 0) {
        cs.tbuf[buf] = tau;
        cs.dg[s] = dss;
        cs.es[s] = beta;
        cs.taus[s] = tau;
      }
      named_arrive(1, NW * 32);
    } else {
      named_sync(1, NW * 32);
    }
    if (stamp) dbg[17] = (double)clock64();
    const double tau = cs.tbuf[buf];
    const int c0 = s + 1 > w ? (s + 1 - w + NW - 1) / NW : 0;  // first slot with column > s
    // (dead columns inside a live group of four slots have v_k = 0 exactly)
    double vr[MR], pr[MR], pq[MR];
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int i = 32 * r + lane;
      vr[r] = i < rl ? vb[i] : 0.0;  // 0 for rows <= s
      pr[r] = 0.0;
      pq[r] = 0.0;
    }
#pragma unroll
    for (int g = 0; g < MC; g += 4) {
      if (g + 3 >= c0 && w + NW * g < d) {
        double v4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v4[u] = g + u < MC ? vb[w + NW * (g + u)] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int r = 0; r < MR; ++r)
            if (g + u < MC) {  // (dead row chunks too: their products are never read)
              if (u & 1) pq[r] = fma(a[g + u][r], v4[u], pq[r]);
              else pr[r] = fma(a[g + u][r], v4[u], pr[r]);
            }
      }
    }
#pragma unroll
    for (int r = 0; r < MR; ++r) pr[r] += pq[r];
    double dw = 0.0;
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int i = 32 * r + lane;
      dw = fma(pr[r], vr[r], dw);
      if (i < rl) rb[w * rl + i] = pr[r];
    }
    dw = warp_sum(dw);
    if (lane == 0) db[w] = dw;
    if (stamp) dbg[18] = (double)clock64();
    __syncthreads();
    if (stamp) dbg[19] = (double)clock64();
    double dot = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) dot += db[q];
    const double K = -0.5 * tau * tau * dot;  // w = p + K v (dsytd2)
    {  // p = tau A v and w = p + K v, one thread per row (0 on the dead rows): the
       // update reads w_k with one load per column instead of p_k, v_k and an fma
      const int t = threadIdx.x;
      if (t < rl) {
        double wv = 0.0;
        if (t > s && t < d) {
          double p = 0.0;
#pragma unroll
          for (int q = 0; q < NW; ++q) p += rb[q * rl + t];
          wv = fma(K, vb[t], tau * p);
        }
        cs.pbuf[t] = wv;
      }
    }
    __syncthreads();
    double wr[MR];
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int i = 32 * r + lane;
      wr[r] = i < rl ? cs.pbuf[i] : 0.0;
    }
#pragma unroll
    for (int g = 0; g < MC; g += 4) {
      if (g + 3 >= c0 && w + NW * g < d) {
        double v4[4], w4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = w + NW * (g + u);
          v4[u] = g + u < MC ? vb[k] : 0.0;
          w4[u] = (g + u < MC && k < d) ? cs.pbuf[k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int r = 0; r < MR; ++r)
            if (g + u < MC) a[g + u][r] = fma(-vr[r], w4[u], fma(-wr[r], v4[u], a[g + u][r]));
      }
    }
    // the owner of column s + 1 (slot (s + 1) / NW) hands it to the next producer;
    // the slot is found by a uniform branch tree (the register file cannot be
    // indexed: a predicated chain over all MC slots cost ~4 MC instructions on the
    // warp that is the next step's critical path)
    if (w == ((s + 1) & (NW - 1))) {
      slot_dispatch<0, MC>(a, (s + 1) / NW, [&](const double (&col)[MR]) {
#pragma unroll
        for (int r = 0; r < MR; ++r)
          if (32 * r + lane < rl) colbuf[32 * r + lane] = col[r];
      });
    }
    __syncwarp();
    if (stamp) dbg[20] = (double)clock64();
    buf ^= 1;
  }
  // the last 2 x 2 (or the whole of d <= 2)
#pragma unroll
  for (int c = 0; c < MC; ++c) {
    const int k = w + NW * c;
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int i = 32 * r + lane;
      if (d >= 2 && k == d - 2 && i == d - 2) cs.dg[d - 2] = a[c][r];
      if (d >= 2 && k == d - 2 && i == d - 1) cs.es[d - 2] = a[c][r];
      if (k == d - 1 && i == d - 1) cs.dg[d - 1] = a[c][r];
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// 2. Sturm count: eigenvalues of the unreduced block [bs, be] of T below x.
// Three-term recurrence p_k = (a_k - x) p_{k-1} - e_{k-1}^2 p_{k-2}; a sign
// change between p_{k-1} and p_k is an eigenvalue of T_k below x.
__device__ __forceinline__ int sgn_bit(double v) { return (int)((unsigned)__double2hiint(v) >> 31); }

__device__ __forceinline__ int sturm_count(const double *da, const double *e2, int bs, int be, double x) {
  // an exact zero p_k counts as positive; with e_k != 0 inside a block the
  // next p then has the sign of -p_{k-1}, so the pair contributes one change
  // either way (Sturm), and a zero at the end counts lambda = x as not below x
  double pp = 1.0, pc = da[bs] - x;
  int c = sgn_bit(pc);
  int k = bs + 1;
  // eight steps per trip (loads off the FMA chain), exact rescale once per
  // trip: |T| < 1, so |p| grows by less than 2^16 over a trip
  for (; k + 7 <= be; k += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double pn = fma(da[k + u] - x, pc, -e2[k + u - 1] * pp);
      c += sgn_bit(pn) ^ sgn_bit(pc);
      pp = pc;
      pc = pn;
    }
    const int ex = (__double2hiint(pc) >> 20) & 0x7ff;  // biased exponent (integer pipe)
    if (ex > 1023 + 300 || (ex < 1023 - 300 && ex > 0)) {
      const double f = ex > 1023 ? 0x1p-300 : 0x1p300;
      pc *= f;
      pp *= f;
    }
  }
  for (; k <= be; ++k) {
    const double pn = fma(da[k] - x, pc, -e2[k - 1] * pp);
    c += sgn_bit(pn) ^ sgn_bit(pc);
    pp = pc;
    pc = pn;
  }
  return c;
}

// NP Sturm counts of the same block at once (independent recurrences
// interleaved).  pk[k] = (a_k, e_{k-1}^2) packed: one 16-byte shared-memory load
// per step; the signs of p_k go through a funnel-shift register and the changes
// are counted once per eight steps (the step is bound by issued instructions:
// 2 loads + 3 fp64 + 2 integer before, 1 + 3 + 1 now).
template <int NP>
__device__ __forceinline__ void sturm_count_n(const double2 *pk, int bs, int be, const double (&x)[NP],
                                              int (&c)[NP]) {
  double pp[NP], pc[NP];
  unsigned sh[NP];
  const double a0 = pk[bs].x;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    pp[p] = 1.0;
    pc[p] = a0 - x[p];
    sh[p] = (unsigned)sgn_bit(pc[p]);
    c[p] = (int)sh[p];
  }
  int k = bs + 1;
  for (; k + 7 <= be; k += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double2 v = pk[k + u];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const double pn = fma(v.x - x[p], pc[p], -v.y * pp[p]);
        sh[p] = __funnelshift_l((unsigned)__double2hiint(pn), sh[p], 1);  // sign bit shifted in
        pp[p] = pc[p];
        pc[p] = pn;
      }
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      c[p] += __popc((sh[p] ^ (sh[p] >> 1)) & 0xffu);  // the eight sign changes of this trip
      const int ex = (__double2hiint(pc[p]) >> 20) & 0x7ff;  // biased exponent (integer pipe)
      if (ex > 1023 + 300 || (ex < 1023 - 300 && ex > 0)) {
        const double f = ex > 1023 ? 0x1p-300 : 0x1p300;
        pc[p] *= f;
        pp[p] *= f;
      }
    }
  }
  for (; k <= be; ++k) {
    const double2 v = pk[k];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double pn = fma(v.x - x[p], pc[p], -v.y * pp[p]);
      c[p] += sgn_bit(pn) ^ sgn_bit(pc[p]);
      pp[p] = pc[p];
      pc[p] = pn;
    }
  }
}

// 3. twisted-factorisation eigenvector of the block [bs, be] of T for lam,
// written (unnormalised L / U first, then z) into column zc of Z (stride lz).
// Returns false when the vector is not finite.
__device__ bool twisted_vector(const double *da, const double *es, int bs, int be, double lam, double *zc, int lz,
                               int d) {
  const double pivmin = 0x1p-400;
  for (int i = 0; i < bs; ++i) zc[(int64_t)i * lz] = 0.0;
  for (int i = be + 1; i < d; ++i) zc[(int64_t)i * lz] = 0.0;
  if (bs == be) {
    zc[(int64_t)bs * lz] = 1.0;
    return true;
  }
  // stationary qd: T - lam I = L+ D+ L+'  (L_k = e_k / D+_k stored at row k)
  double dp = da[bs] - lam;
  for (int k = bs; k < be; ++k) {
    if (fabs(dp) < pivmin) dp = dp < 0.0 ? -pivmin : pivmin;
    const double L = es[k] * __drcp_rn(dp);
    zc[(int64_t)k * lz] = L;
    dp = (da[k + 1] - lam) - L * es[k];
  }
  // progressive qd from below: T - lam I = U- D- U-'; gamma_k = D+_k + D-_k - (a_k - lam)
  double dm = da[be] - lam;
  double gbest = fabs(dp);
  int r = be;
  for (int k = be - 1; k >= bs; --k) {
    if (fabs(dm) < pivmin) dm = dm < 0.0 ? -pivmin : pivmin;
    const double U = es[k] * __drcp_rn(dm);
    const double ak = da[k] - lam;
    dm = ak - U * es[k];
    const double dpk = k == bs ? ak : ak - zc[(int64_t)(k - 1) * lz] * es[k - 1];
    const double g = fabs(dpk + dm - ak);
    if (g < gbest) {
      gbest = g;
      r = k;
    }
  }
  // U_k for k in [r, be) at row k + 1 (rows > r no longer need L)
  dm = da[be] - lam;
  for (int k = be - 1; k >= r; --k) {
    if (fabs(dm) < pivmin) dm = dm < 0.0 ? -pivmin : pivmin;
    const double U = es[k] * __drcp_rn(dm);
    zc[(int64_t)(k + 1) * lz] = U;
    dm = (da[k] - lam) - U * es[k];
  }
  // z_r = 1; z_k = -L_k z_{k+1} (k < r); z_{k+1} = -U_k z_k (k >= r)
  zc[(int64_t)r * lz] = 1.0;
  double amax = 1.0, z = 1.0;
  for (int k = r - 1; k >= bs; --k) {
    z = -zc[(int64_t)k * lz] * z;
    zc[(int64_t)k * lz] = z;
    amax = fmax(amax, fabs(z));
  }
  z = 1.0;
  for (int k = r; k < be; ++k) {
    z = -zc[(int64_t)(k + 1) * lz] * z;
    zc[(int64_t)(k + 1) * lz] = z;
    amax = fmax(amax, fabs(z));
  }
  if (!(amax < CUDART_INF)) return false;
  const double sa = 1.0 / amax;
  double nrm = 0.0;
  for (int k = bs; k <= be; ++k) {
    const double t = zc[(int64_t)k * lz] * sa;
    nrm = fma(t, t, nrm);
  }
  const double f = sa / sqrt(nrm);
  for (int k = bs; k <= be; ++k) zc[(int64_t)k * lz] *= f;
  return true;
}

// ---------------------------------------------------------------------------
// 4. V = Q Z, Q = H_0 H_1 ... H_{d-3}, in compact-WY blocks of NB reflectors
// from the last block to the first: Q_b = H_s0 ... H_s0+nb-1 = I - W T W'
// (dlarft, forward, columnwise), Z <- Z - W (T (W' Z)).  Z in shared memory
// (ld lv); hv the packed reflectors (global).
__device__ void cold_backtransform(int d, const ColdSmem &cs, const double *hv) {
  constexpr int NB = kColdNB;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, w = tid >> 5;
  const int lv = cs.lv, nref = d - 2;
  if (nref <= 0) return;
  // W tile of block b: W(i, j) = v_{s0 + j}(i) from the packed reflectors
  // (global); the next block's tile is fetched into registers while this
  // block's GEMMs run
  constexpr int PF = (kColdMaxD * NB + kColdThreads - 1) / kColdThreads;
  auto wval = [&](int b, int e) {
    const int s0 = b * NB, nb = min(NB, nref - s0);
    const int i = e / NB, j = e - i * NB, s = s0 + j;
    return (j < nb && i > s) ? hv[cold_hoff(s, d) + (i - s - 1)] : 0.0;
  };
  double wp[PF];
  const int blast = (nref - 1) / NB;
#pragma unroll
  for (int q = 0; q < PF; ++q) {
    const int e = tid + q * T;
    wp[q] = e < d * NB ? wval(blast, e) : 0.0;
  }
  for (int b = blast; b >= 0; --b) {
    const int s0 = b * NB, nb = min(NB, nref - s0);
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int e = tid + q * T;
      if (e < d * NB) cs.Wt[e] = wp[q];
    }
    if (b > 0)
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int e = tid + q * T;
        wp[q] = e < d * NB ? wval(b - 1, e) : 0.0;
      }
    __syncthreads();
    // G = W'W (NB x NB)
    team_mm1<false, false>(NB, NB, Opd{cs.Wt, 1, NB}, Opd{cs.Wt, NB, 1}, d,
                           [&](int a, int c, double v) { cs.Gb[a * NB + c] = v; });
    if (w == 0) {
      // T (upper): T(i, i) = tau_i, T(l, i) = -tau_i sum_{l <= m < i} T(l, m) G(m, i); lane l holds row l
      double tr[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const double ti = i < nb ? cs.taus[s0 + i] : 0.0;
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < i; ++m)
          if (m >= lane) acc = fma(tr[m], cs.Gb[m * NB + i], acc);
        tr[i] = lane == i ? ti : (lane < i ? -ti * acc : 0.0);
      }
      if (lane < NB)
#pragma unroll
        for (int i = 0; i < NB; ++i) cs.Tb[lane * NB + i] = tr[i];
    }
    __syncthreads();
    // Y = W' Z (NB x d), then Y <- T Y in place, then Z <- Z - W Y
    team_mm1<false, false>(NB, d, Opd{cs.Wt, 1, NB}, Opd{cs.Z, lv, 1}, d,
                           [&](int a, int c, double v) { cs.Yb[a * lv + c] = v; });
    team_mm1<false, true>(NB, d, Opd{cs.Tb, NB, 1}, Opd{cs.Yb, lv, 1}, NB,
                          [&](int a, int c, double v) { cs.Yb[a * lv + c] = v; });
    team_mm1<false, false>(d, d, Opd{cs.Wt, NB, 1}, Opd{cs.Yb, lv, 1}, NB,
                           [&](int a, int c, double v) { cs.Z[a * lv + c] -= v; });
  }
}

// ---------------------------------------------------------------------------
// The eigendecomposition.  On entry Z holds the symmetric X (ld lv, rows /
// columns < d).  On exit (COLD_OK): cs.lam = eigenvalues ascending
// (unscaled), and -- unless values_only -- Z = V (columns = eigenvectors,
// same order).  hv: global scratch for the reflectors.
template <int MC, int MR>
__device__ int cold_eig(int d, const ColdSmem &cs, bool values_only, double *hv, double *dbg) {
  constexpr int NW = kColdNW;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, w = tid >> 5;
  {
    double a[MC][MR];
#pragma unroll
    for (int c = 0; c < MC; ++c)
#pragma unroll
      for (int r = 0; r < MR; ++r) {
        const int i = 32 * r + lane, k = w + NW * c;
        a[c][r] = (i < d && k < d) ? cs.Z[(int64_t)k * cs.lv + i] : 0.0;  // X symmetric: A(i, k) = X(k, i)
      }
    __syncthreads();
    COLD_STAMP(dbg, 1);
    cold_tridiag<MC, MR>(a, d, cs, hv, dbg);
    COLD_STAMP(dbg, 2);
  }
  // ---- scale T to |T| ~ 1 (exact powers of two), split tiny off-diagonals
  double gl = CUDART_INF, gh = -CUDART_INF;
  for (int i = tid; i < d; i += T) {
    const double el = i > 0 ? fabs(cs.es[i - 1]) : 0.0, er = i + 1 < d ? fabs(cs.es[i]) : 0.0;
    gl = fmin(gl, cs.dg[i] - el - er);
    gh = fmax(gh, cs.dg[i] + el + er);
  }
  gl = cta_min(gl, cs.misc);
  gh = -cta_min(-gh, cs.misc);
  const double tn = fmax(fabs(gl), fabs(gh));
  if (!(tn < CUDART_INF)) {
    if (tid == 0) *cs.flag = 2;  // non-finite input: EigenFailure
    __syncthreads();
    return COLD_FAIL;
  }
  double sc = 1.0;
  if (tn > 0.0) {
    int ex;
    frexp(tn, &ex);
    sc = ldexp(1.0, -ex);
  }
  for (int i = tid; i < d; i += T) {
    cs.dg[i] *= sc;
    if (i + 1 < d) {
      const double e = cs.es[i] * sc;
      cs.es[i] = fabs(e) <= 0x1p-52 ? 0.0 : e;  // |T| ~ 1: a 2^-52 perturbation
      cs.e2[i] = cs.es[i] * cs.es[i];
    }
  }
  if (tid == 0) *cs.flag = 0;
  __syncthreads();
  // (a_k, e_{k-1}^2) packed for the Sturm recurrence, in the (dead) tridiagonalisation buffers
  double2 *pk = reinterpret_cast<double2 *>(cs.vbuf);
  for (int i = tid; i < d; i += T) pk[i] = make_double2(cs.dg[i], i > 0 ? cs.e2[i - 1] : 0.0);
  // ---- unreduced blocks; bisection, g threads per eigenvalue (multisection)
  for (int j = tid; j < d; j += T) {
    int b0 = j, b1 = j;
    while (b0 > 0 && cs.es[b0 - 1] != 0.0) --b0;
    while (b1 < d - 1 && cs.es[b1] != 0.0) ++b1;
    cs.bs[j] = b0;
    cs.be[j] = b1;
  }
  __syncthreads();
  {
    int g = 1;
    while (2 * g * d <= T && g < 16) g *= 2;
    if (tid < g * d) {
      // (g NP + 1)-section: thread q of the eigenvalue's group of g takes the NP
      // interior points q NP + 1 .. q NP + NP of the current bracket
      constexpr int NP = kColdSturmPts;
      const double lo0 = gl * sc - 0x1p-40, hi0 = gh * sc + 0x1p-40;
      const float bits = log2f((float)(g * NP + 1));
      const int rounds = (int)ceilf(54.0f / bits);
      const double ig = 1.0 / (g * NP + 1);
      const int j = tid / g, q = tid - j * g;
      const int b0 = cs.bs[j], b1 = cs.be[j], jj = j - b0;
      double lo = lo0, hi = hi0;
      const unsigned gm = g == 32 ? 0xffffffffu : (((1u << g) - 1u) << (lane & ~(g - 1)));
      for (int rd = 0; rd < rounds; ++rd) {
        double x[NP];
        int c[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) x[p] = fma(hi - lo, (q * NP + p + 1) * ig, lo);
        sturm_count_n<NP>(pk, b0, b1, x, c);
        double lc = -CUDART_INF, hc = CUDART_INF;
#pragma unroll
        for (int p = 0; p < NP; ++p) {  // x ascending: the last point with count <= jj, the first above
          if (c[p] <= jj) lc = x[p];
          if (c[p] > jj && hc == CUDART_INF) hc = x[p];
        }
        for (int o = g >> 1; o > 0; o >>= 1) {
          lc = fmax(lc, __shfl_xor_sync(gm, lc, o));
          hc = fmin(hc, __shfl_xor_sync(gm, hc, o));
        }
        lo = fmax(lo, lc);
        hi = fmin(hi, hc);
      }
      if (q == 0) cs.lamu[j] = 0.5 * (lo + hi);
    }
  }
  __syncthreads();
  COLD_STAMP(dbg, 3);
  // ---- sorted order; a pair closer than 2^-40 |T| inside one unreduced block
  // is not separable by twisted factorisations: the Jacobi path takes the clique
  for (int j = tid; j < d; j += T) {
    const double lj = cs.lamu[j];
    int rk = 0;
    for (int i = 0; i < d; ++i) {
      const double li = cs.lamu[i];
      rk += (li < lj) || (li == lj && i < j);
    }
    cs.rank[j] = rk;
    cs.lam[rk] = lj / sc;
    if (j > cs.bs[j] && !(lj - cs.lamu[j - 1] > 0x1p-40)) atomicOr(cs.flag, 1);
    if (!(fabs(lj) < CUDART_INF)) atomicOr(cs.flag, 2);
  }
  __syncthreads();
  if (*cs.flag) return COLD_FAIL;
  if (values_only) return COLD_OK;
  // ---- eigenvectors of T into the sorted columns of Z
  for (int j = tid; j < d; j += T)
    if (!twisted_vector(cs.dg, cs.es, cs.bs[j], cs.be[j], cs.lamu[j], cs.Z + cs.rank[j], cs.lv, d))
      atomicOr(cs.flag, 1);
  __syncthreads();
  COLD_STAMP(dbg, 4);
  if (*cs.flag) return COLD_FAIL;
  cold_backtransform(d, cs, hv);
  COLD_STAMP(dbg, 5);
  return COLD_OK;
}

// 5. + 6.  V (= Z, shared) -> the basis store vst (row j = eigenvector j,
// global) after Newton-Schulz, and P emitted as emit(i, j, value) over the
// full d x d (exactly symmetric).  xat(i, j) reads X (needed when the
// negative class is the smaller one).  g2: d x d global scratch.
template <class XAt, class Emit>
__device__ void cold_finish(int d, const ColdSmem &cs, double *vst, double *g2, XAt xat, Emit emit,
                            double *dbg) {
  const int tid = threadIdx.x;
  const int lv = cs.lv;
  double *Vs = cs.Z;
  for (int it = 0; it < 3; ++it) {
    double dev = 0.0;
    team_mm1<true, false>(d, d, Opd{Vs, 1, lv}, Opd{Vs, lv, 1}, d, [&](int a, int b, double v) {
      g2[(int64_t)a * d + b] = v;
      dev = fmax(dev, fabs(v - (a == b ? 1.0 : 0.0)));
    });
    dev = -cta_min(-dev, cs.misc);
    if (dev <= 0x1p-46) {  // orthogonal to rounding already: V -> the store as is
      for (int e = tid; e < d * d; e += blockDim.x) {
        const int k = e / d, i = e - k * d;
        vst[e] = Vs[(int64_t)i * lv + k];
      }
      break;
    }
    team_mm1<false, false, false, 5>(d, d, Opd{Vs, lv, 1}, Opd{g2, d, 1}, d, [&](int a, int b, double v) {  // G from L2
      vst[(int64_t)b * d + a] = fma(-0.5, v, 1.5 * Vs[(int64_t)a * lv + b]);
    });
    {  // V back from the store, eight loads in flight per thread
      const float invd = 1.0f / d;
      for (int e0 = tid; e0 < d * d; e0 += 8 * blockDim.x) {
        double v8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v8[q] = vst[min(e0 + q * (int)blockDim.x, d * d - 1)];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = e0 + q * blockDim.x;
          if (e < d * d) {
            const int k = qdiv(e, invd), i = e - k * d;
            Vs[(int64_t)i * lv + k] = v8[q];
          }
        }
      }
    }
    __syncthreads();
    // one step takes a departure of 2^-26 below rounding; a second one covers
    // tight clusters (departure ~1e-5 -> 1e-20)
    if (dev <= 0x1p-26 || it == 1) break;
  }
  __syncthreads();
  COLD_STAMP(dbg, 6);
  // positive / negative class of the sorted eigenvalues; the smaller one as
  // W = V_C sqrt|lam_C| (in place, V is in the store): P = W W' or X + W W'
  int r = 0;
  for (int i = 0; i < d; ++i) r += cs.lam[i] > 0.0;
  const bool pos = r <= d - r;
  const int c0 = pos ? d - r : 0, K = pos ? r : d - r;
  for (int e = tid; e < d * K; e += blockDim.x) {
    const int k = e / d, i = e - k * d;
    Vs[(int64_t)i * lv + c0 + k] *= sqrt(fabs(cs.lam[c0 + k]));
  }
  __syncthreads();
  if (K == 0) {
    for (int e = tid; e < d * d; e += blockDim.x) {
      const int a = e / d, b = e - a * d;
      emit(a, b, pos ? 0.0 : xat(a, b));
    }
    __syncthreads();
    return;
  }
  team_mm1<true, false>(d, d, Opd{Vs + c0, lv, 1}, Opd{Vs + c0, 1, lv}, K, [&](int a, int b, double v) {
    emit(a, b, pos ? v : xat(a, b) + v);
  });
  COLD_STAMP(dbg, 7);
}

// ---------------------------------------------------------------------------
// One clique through the cold path (blockDim = kColdThreads).
//   CONE_HOT:   X from the hot-path slot update (solver.py:222-244, :316,
//               :388-394) or, when xin, from W.xarg (the fast path already
//               did the slot update); raw X is left in W.xarg; P -> u_s,
//               w_s += P; V -> the basis store (age 1).
//   CONE_PLAIN: X = in_scale * in (stacked s layout); P -> out.
//   CONE_MINEIG: smallest eigenvalue -> out[k].
// Returns COLD_FAIL (nothing emitted; X in W.xarg for the hot path) when the
// spectrum has a pair closer than 2^-40 |T| inside one unreduced block: the
// caller hands the clique to the Jacobi path.  pscratch slot: reflectors,
// Gram matrix, (plain) V.
template <int MODE, int MC, int MR>
__device__ int cold_one(const DevProblem &P, const DevState &S, const DevWork &W, const ConeArgs &ca, int k,
                        double *smem, bool xin) {
  const int d = P.cl_size[k];
  const int tid = threadIdx.x, T = blockDim.x;
  const int64_t off = P.cl_off[k], so = P.n_c;
  const ColdSmem cs = cold_carve(smem, d);
  const float invd = 1.0f / d;
  double *xg = W.xarg + off;
  double *scr = ca.pscratch + (int64_t)ca.slot * ca.pstride;
  double *hv = scr, *g2 = scr + cold_hv_doubles(d), *vpl = g2 + (int64_t)d * d;
  COLD_STAMP(W.dbg, 0);
  double dx2 = 0.0;  // |X - X_prev|_F^2 (hot path): bounds off(V' X V) for the basis kept now
  // ---- X (raw) into Z, then symmetrised (symmat.py:157)
  if (MODE == CONE_HOT) {
    const double shift = W.scal[S_SHIFT];
    if (xin) {
      for (int e = tid; e < d * d; e += T) {
        const int a = qdiv(e, invd), b = e - a * d;
        cs.Z[a * cs.lv + b] = xg[e];
      }
    } else {
      constexpr int NB = kColdLoadBatch;  // every load of the batch in flight before the stores (they may alias)
      for (int e0 = tid; e0 < d * d; e0 += NB * T) {
        double xv[NB], xo[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) {
          const int e = e0 + q * T;
          xv[q] = e < d * d ? hot_slot_load(P, S, W, off + e, shift) : 0.0;
          xo[q] = e < d * d ? xg[e] : 0.0;  // X of the previous iteration (either path)
        }
#pragma unroll
        for (int q = 0; q < NB; ++q) {
          const int e = e0 + q * T;
          if (e < d * d) {
            const int a = qdiv(e, invd), b = e - a * d;
            cs.Z[a * cs.lv + b] = xv[q];
            xg[e] = xv[q];
            dx2 = fma(xv[q] - xo[q], xv[q] - xo[q], dx2);
          }
        }
      }
    }
  } else {
    for (int e = tid; e < d * d; e += T) {
      const int a = qdiv(e, invd), b = e - a * d;
      cs.Z[a * cs.lv + b] = ca.in[off + e] * ca.in_scale;
    }
  }
  __syncthreads();
  for (int e = tid; e < d * d; e += T) {
    const int a = qdiv(e, invd), b = e - a * d;
    if (a < b) {
      const double s = 0.5 * (cs.Z[a * cs.lv + b] + cs.Z[b * cs.lv + a]);
      cs.Z[a * cs.lv + b] = s;
      cs.Z[b * cs.lv + a] = s;
    }
  }
  __syncthreads();
  const int st = cold_eig<MC, MR>(d, cs, MODE == CONE_MINEIG, hv, W.dbg);
  if (st != COLD_OK) {
    const int fl = *cs.flag;
    __syncthreads();
    if ((fl & 2) && tid == 0) atomicOr(W.err, 1);  // non-finite: EigenFailure (symmat.py:162-163)
    return (fl & 2) ? COLD_OK : COLD_FAIL;         // (a non-finite clique is not retried)
  }
  if (MODE == CONE_MINEIG) {
    if (tid == 0) ca.out[k] = cs.lam[0];
    __syncthreads();
    return COLD_OK;
  }
  if (MODE == CONE_HOT && W.cnext && !xin) {
    // next iteration on the fast path when it would apply with margin:
    // off(B) <= |X_next - X|_F, predicted by |X - X_prev|_F, against min |lam|
    // (the fast path's g; hsde_split.cuh applies at off(B) <= 0.45 g)
    dx2 = cta_sum(dx2, cs.misc);
    double g = CUDART_INF;
    for (int i = 0; i < d; ++i) g = fmin(g, fabs(cs.lam[i]));
    const bool prev = (W.vvalid[k] & ~kVRefresh) > 0;
    // (measured on config 4: off(B) / |X - X_prev|_F ~ 0.3 - 0.5, so |dX| <= 0.6 g
    // predicts off(B) <~ 0.3 g, inside the fast path's 0.45 g)
    if (tid == 0) W.cnext[k] = (prev && dx2 <= ca.pol_c2f * g * g) ? 0 : 1;  // default |dX| <= 0.6 g
  }
  if (MODE == CONE_HOT) {
    double *su = S.u + so + off, *sw = S.w + so + off;
    auto xat = [&](int a, int b) { return 0.5 * (xg[a * d + b] + xg[b * d + a]); };
    cold_finish(
        d, cs, W.vstore + off, g2, xat, [&](int a, int b, double v) { su[a * d + b] = v; }, W.dbg);
    __syncthreads();
    for (int e0 = tid; e0 < d * d; e0 += 8 * T) {  // w_s = (w_s - us_h) + P (solver.py:391-394), batched loads
      double a8[8], b8[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = min(e0 + q * T, d * d - 1);
        a8[q] = sw[e];
        b8[q] = su[e];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (e0 + q * T < d * d) sw[e0 + q * T] = a8[q] + b8[q];
    }
    if (tid == 0) {
      W.vvalid[k] = 1;
      if (W.sweeps) W.sweeps[k] = 0;
    }
  } else {
    double *out = ca.out + off;
    const double *in = ca.in + off;
    const double isc = ca.in_scale;
    auto xat = [&](int a, int b) { return 0.5 * (in[a * d + b] * isc + in[b * d + a] * isc); };
    cold_finish(
        d, cs, vpl, g2, xat, [&](int a, int b, double v) { out[a * d + b] = v; }, W.dbg);
  }
  __syncthreads();
  return COLD_OK;
}

// One CTA (four warps) per clique of the plan.  HOT after k_cone_split
// (W.cstate set): only the cliques it did not finish -- untouched ones
// (no basis: slot update here) and hand-overs (X in W.xarg).  Failures are
// flagged in ca.cfail[slot] for a follow-up Jacobi launch (k_cone_block with
// ca.fail_only); larger cliques than the variant holds are flagged too.
template <int MODE, int MC, int MR, int MINB>
__global__ void __launch_bounds__(kColdThreads, MINB) k_cone_cold(DevProblem P, DevState S, DevWork W, ConeArgs ca) {
  extern __shared__ __align__(16) double smem[];
  if ((int)blockIdx.x >= ca.count) return;
  const int k = ca.ids[blockIdx.x];
  const int d = P.cl_size[k];
  int cst = SPLIT_UNTOUCHED;
  bool xin = false;
  if (MODE == CONE_HOT && W.ccur) {
    if (ca.cold_pass == 0 && !W.ccur[k]) {  // on the warm path this iteration (k_cone_split)
      if (threadIdx.x == 0 && ca.cfail) ca.cfail[blockIdx.x] = 0;
      return;
    }
    if (ca.cold_pass == 1) {  // after k_cone_split: its hand-overs (X in W.xarg)
      cst = W.cstate[k];
      if (W.ccur[k] || cst < SPLIT_HANDOFF || cst > SPLIT_HANDOFF + 3) return;
      xin = true;
    }
  }
  ConeArgs c2 = ca;
  c2.slot = blockIdx.x;
  const bool fits = d <= 32 * MR && d <= kColdNW * MC;
  int st = COLD_FAIL;
  if (fits) {
    st = cold_one<MODE, MC, MR>(P, S, W, c2, k, smem, xin);
  } else if (MODE == CONE_HOT && !xin) {
    // the Jacobi fallback reads raw X from W.xarg: do the slot update here
    const double shift = W.scal[S_SHIFT];
    const int64_t off = P.cl_off[k];
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) W.xarg[off + e] = hot_slot_load(P, S, W, off + e, shift);
  }
  if (threadIdx.x == 0) {
    if (ca.cfail) ca.cfail[blockIdx.x] = st == COLD_FAIL ? 1 : 0;
    if (MODE == CONE_HOT && W.cstate) W.cstate[k] = SPLIT_DONE + 32 + cst;  // (stats: finished here)
    if (MODE == CONE_HOT && W.ckey) W.ckey[k] = 1;
    if (MODE == CONE_HOT && xin && W.cnext) W.cnext[k] = 1;  // a hand-over: cold next time too
  }
}

// One CTA per CTA-sized clique on the hot path: the fast path when the
// clique has a valid eigenbasis (hsde_split.cuh).  COLD: cliques without a
// basis and hand-overs are left to k_cone_cold (X kept in W.xarg); otherwise
// the Jacobi path (cone_one) finishes them in the same CTA.
template <bool COLD, int THREADS = kSplitThreads>
__global__ void __launch_bounds__(THREADS, 2) k_cone_split(DevProblem P, DevState S, DevWork W, ConeArgs ca) {
  extern __shared__ __align__(16) double smem[];
  if ((int)blockIdx.x >= ca.count) return;
  const int k = ca.ids[blockIdx.x];
  const int d = P.cl_size[k];
  const int vv = W.vvalid[k];
  ConeArgs c2 = ca;
  c2.slot = blockIdx.x;
  c2.cold = COLD;
  if (W.ccur && W.ccur[k]) return;  // this iteration on the cold path (k_cone_cold, concurrent)
  int st = SPLIT_UNTOUCHED;
  // (B's upper 16 x 16 blocks must fit the warps' register blocks: d <= 96 with
  // twelve warps, d <= 80 with ten)
  const int nbd = (d + 15) >> 4;
  const bool fits = nbd * (nbd + 1) / 2 <= kSplitMaxB * (THREADS / 32);
  if (ca.warm && vv > 0 && !(vv & kVRefresh) && d <= kSplitMaxD && d >= 8 && fits)
    st = split_one(P, S, W, c2, k, smem);
  if (threadIdx.x == 0) W.cstate[k] = st;
  if (st == SPLIT_DONE || st == SPLIT_DONE + 16) return;
  if (threadIdx.x == 0 && W.cnext && st != SPLIT_UNTOUCHED) W.cnext[k] = 1;  // handed over: cold next
  if (COLD && st != SPLIT_UNTOUCHED) return;  // k_cone_cold (cold_pass 1) finishes it from W.xarg

  __syncthreads();  // cstate and the hand-off B are visible to the whole CTA
  BlockTeam tm{(int)threadIdx.x, (int)blockDim.x};
  cone_one<CONE_HOT>(tm, P, S, W, c2, k, smem);
  if (threadIdx.x == 0) {
    W.cstate[k] = SPLIT_DONE + 32 + st;  // (stats: finished by the Jacobi path)
    W.ckey[k] = 1;                        // schedule first next time
  }
}

// ===========================================================================
// Warp-sized cliques (d <= 32): the same cold eigensolver run by one warp per
// clique, the matrix in the warp's shared-memory slice (lane i owns row i;
// no CTA barriers, __syncwarp only).  Replaces the warp Jacobi sweeps on the
// hot path of the many-small-clique configurations.

__host__ __device__ inline int wcold_ld(int dp) { return dp | 1; }
__host__ __device__ inline int64_t wcold_scratch_doubles(int dp) {
  const int ld = wcold_ld(dp);
  const int64_t n = (int64_t)dp * ld + ((int64_t)dp * (dp - 1) / 2 + 2) + 2 * 32 + 6 * 32 + 8 + (3 * 32 + 2) / 2 + 2;
  return (n + 1) & ~int64_t(1);
}

struct WColdSmem {
  double *Z, *Hv, *vb, *wb, *dg, *es, *e2, *taus, *lam, *lamu, *misc;
  int *rank, *bs, *be, *flag;
  int ld;
};

__device__ inline WColdSmem wcold_carve(double *base, int dp) {
  WColdSmem c;
  c.ld = wcold_ld(dp);
  c.Z = base;
  c.Hv = c.Z + (int64_t)dp * c.ld;
  c.vb = c.Hv + ((int64_t)dp * (dp - 1) / 2 + 2);
  c.wb = c.vb + 32;
  c.dg = c.wb + 32;
  c.es = c.dg + 32;
  c.e2 = c.es + 32;
  c.taus = c.e2 + 32;
  c.lam = c.taus + 32;
  c.lamu = c.lam + 32;
  c.misc = c.lamu + 32;
  c.rank = reinterpret_cast<int *>(c.misc + 8);
  c.bs = c.rank + 32;
  c.be = c.bs + 32;
  c.flag = c.be + 32;
  return c;
}

__device__ __forceinline__ double warp_allmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_allmin(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// eigendecomposition of the symmetric X in Z (rows / columns < d <= 32):
// COLD_OK with lam ascending (unscaled) and, unless values_only, Z = V
__device__ int wcold_eig(int d, const WColdSmem &c, bool values_only) {
  const int l = threadIdx.x & 31, ld = c.ld;
  // ---- Householder tridiagonalisation (dsytd2 order), lane i owns row i
  for (int s = 0; s + 2 < d; ++s) {
    const double x = l < d ? c.Z[l * ld + s] : 0.0;
    const double sig = warp_allsum((l > s + 1 && l < d) ? x * x : 0.0);
    const double x0 = __shfl_sync(0xffffffffu, x, (s + 1) & 31), dss = __shfl_sync(0xffffffffu, x, s & 31);
    double tau = 0.0, beta = x0, scal = 0.0;
    if (sig > 0.0) {
      const double n2 = fma(x0, x0, sig), rn = rsqrt(n2), nx = n2 * rn;
      beta = -copysign(nx, x0);
      tau = fma(fabs(x0), rn, 1.0);
      scal = copysign(__drcp_rn(fabs(x0) + nx), x0);
    }
    const double v = l == s + 1 ? 1.0 : ((l > s + 1 && l < d) ? x * scal : 0.0);
    c.vb[l] = v;
    if (l > s && l < d) c.Hv[cold_hoff(s, d) + (l - s - 1)] = v;
    if (l == 0) {
      c.dg[s] = dss;
      c.es[s] = beta;
      c.taus[s] = tau;
    }
    __syncwarp();
    double p = 0.0;
    if (l > s && l < d)
      for (int k = s + 1; k < d; ++k) p = fma(c.Z[l * ld + k], c.vb[k], p);
    p *= tau;
    const double K = -0.5 * tau * warp_allsum(p * v);
    const double wv = fma(K, v, p);
    c.wb[l] = wv;
    __syncwarp();
    if (l > s && l < d)
      for (int k = s + 1; k < d; ++k) c.Z[l * ld + k] = fma(-v, c.wb[k], fma(-wv, c.vb[k], c.Z[l * ld + k]));
    __syncwarp();
  }
  if (l == 0) {
    if (d >= 2) {
      c.dg[d - 2] = c.Z[(d - 2) * ld + d - 2];
      c.es[d - 2] = c.Z[(d - 1) * ld + d - 2];
    }
    c.dg[d - 1] = c.Z[(d - 1) * ld + d - 1];
  }
  __syncwarp();
  // ---- scale T, split, blocks
  double gl = CUDART_INF, gh = -CUDART_INF;
  if (l < d) {
    const double el = l > 0 ? fabs(c.es[l - 1]) : 0.0, er = l + 1 < d ? fabs(c.es[l]) : 0.0;
    gl = c.dg[l] - el - er;
    gh = c.dg[l] + el + er;
  }
  gl = warp_allmin(gl);
  gh = warp_allmax(gh);
  const double tn = fmax(fabs(gl), fabs(gh));
  if (!(tn < CUDART_INF)) return COLD_FAIL + 1;  // non-finite
  double sc = 1.0;
  if (tn > 0.0) {
    int ex;
    frexp(tn, &ex);
    sc = ldexp(1.0, -ex);
  }
  __syncwarp();
  if (l < d) {
    c.dg[l] *= sc;
    if (l + 1 < d) {
      const double e = c.es[l] * sc;
      c.es[l] = fabs(e) <= 0x1p-52 ? 0.0 : e;
      c.e2[l] = c.es[l] * c.es[l];
    }
  }
  __syncwarp();
  if (l < d) {
    int b0 = l, b1 = l;
    while (b0 > 0 && c.es[b0 - 1] != 0.0) --b0;
    while (b1 < d - 1 && c.es[b1] != 0.0) ++b1;
    c.bs[l] = b0;
    c.be[l] = b1;
  }
  __syncwarp();
  // ---- bisection (multisection: g lanes per eigenvalue)
  {
    int g = 1;
    while (2 * g * d <= 32) g *= 2;
    const double lo0 = gl * sc - 0x1p-40, hi0 = gh * sc + 0x1p-40;
    const int rounds = (int)ceilf(54.0f / log2f((float)(g + 1)));
    const double ig = 1.0 / (g + 1);
    const int j = min(l / g, d - 1), q = l - (l / g) * g;
    const int b0 = c.bs[j], b1 = c.be[j], jj = j - b0;
    double lo = lo0, hi = hi0;
    for (int rd = 0; rd < rounds; ++rd) {
      const double xx = fma(hi - lo, (q + 1) * ig, lo);
      const int cnt = sturm_count(c.dg, c.e2, b0, b1, xx);
      double lc = cnt <= jj ? xx : -CUDART_INF, hc = cnt > jj ? xx : CUDART_INF;
      for (int o = g >> 1; o > 0; o >>= 1) {
        lc = fmax(lc, __shfl_xor_sync(0xffffffffu, lc, o));
        hc = fmin(hc, __shfl_xor_sync(0xffffffffu, hc, o));
      }
      lo = fmax(lo, lc);
      hi = fmin(hi, hc);
    }
    if (q == 0 && l < g * d) c.lamu[j] = 0.5 * (lo + hi);
  }
  __syncwarp();
  int bad = 0;
  if (l < d) {
    const double lj = c.lamu[l];
    int rk = 0;
    for (int i = 0; i < d; ++i) {
      const double li = c.lamu[i];
      rk += (li < lj) || (li == lj && i < l);
    }
    c.rank[l] = rk;
    c.lam[rk] = lj / sc;
    if (l > c.bs[l] && !(lj - c.lamu[l - 1] > 0x1p-40)) bad = 1;
    if (!(fabs(lj) < CUDART_INF)) bad = 2;
  }
  bad = __reduce_max_sync(0xffffffffu, bad);
  __syncwarp();
  if (bad) return COLD_FAIL + (bad == 2);
  if (values_only) return COLD_OK;
  // ---- eigenvectors of T into the sorted columns of Z (the reduced matrix is dead)
  if (l < d && !twisted_vector(c.dg, c.es, c.bs[l], c.be[l], c.lamu[l], c.Z + c.rank[l], ld, d)) bad = 1;
  bad = __reduce_max_sync(0xffffffffu, bad);
  __syncwarp();
  if (bad) return COLD_FAIL;
  // ---- back transformation, lane j owns column j
  if (l < d)
    for (int s = d - 3; s >= 0; --s) {
      const double tau = c.taus[s];
      if (tau == 0.0) continue;
      const double *hv = c.Hv + cold_hoff(s, d) - (s + 1);
      double t = 0.0;
      for (int i = s + 1; i < d; ++i) t = fma(hv[i], c.Z[i * ld + l], t);
      t *= tau;
      for (int i = s + 1; i < d; ++i) c.Z[i * ld + l] = fma(-t, hv[i], c.Z[i * ld + l]);
    }
  __syncwarp();
  return COLD_OK;
}

// one warp per clique; failures flagged in ca.cfail[warp slot] for the warp
// Jacobi launch that follows (k_cone_warp with ca.fail_only)
template <int MODE>
__device__ int wcold_one(const DevProblem &P, const DevState &S, const DevWork &W, const ConeArgs &ca, int k,
                         double *scratch) {
  const int d = P.cl_size[k];
  const int l = threadIdx.x & 31;
  const int64_t off = P.cl_off[k], so = P.n_c;
  if (d == 1) {  // np.maximum(b, 0.0)
    if (l == 0) {
      const double a = MODE == CONE_HOT ? hot_slot_load(P, S, W, off, W.scal[S_SHIFT]) : ca.in[off] * ca.in_scale;
      const double pr = (a != a) ? a : (a > 0.0 ? a : 0.0);
      if (MODE == CONE_HOT) {
        S.u[so + off] = pr;
        S.w[so + off] += pr;
      } else if (MODE == CONE_PLAIN) {
        ca.out[off] = pr;
      } else {
        ca.out[k] = a;
      }
    }
    return COLD_OK;
  }
  const WColdSmem c = wcold_carve(scratch, ca.dpmax);
  const int ld = c.ld;
  double *xg = W.xarg + off;
  if (MODE == CONE_HOT) {
    const double shift = W.scal[S_SHIFT];
    for (int e = l; e < d * d; e += 32) {
      const int a = e / d, b = e - a * d;
      const double x = hot_slot_load(P, S, W, off + e, shift);
      c.Z[a * ld + b] = x;
      xg[e] = x;
    }
  } else {
    for (int e = l; e < d * d; e += 32) {
      const int a = e / d, b = e - a * d;
      c.Z[a * ld + b] = ca.in[off + e] * ca.in_scale;
    }
  }
  __syncwarp();
  for (int e = l; e < d * d; e += 32) {  // sym = 0.5 (B + B')  (symmat.py:157)
    const int a = e / d, b = e - a * d;
    if (a < b) {
      const double s = 0.5 * (c.Z[a * ld + b] + c.Z[b * ld + a]);
      c.Z[a * ld + b] = s;
      c.Z[b * ld + a] = s;
    }
  }
  __syncwarp();
  const int st = wcold_eig(d, c, MODE == CONE_MINEIG);
  if (st == COLD_FAIL + 1) {  // non-finite eigenvalue: EigenFailure (symmat.py:162-163)
    if (l == 0) atomicOr(W.err, 1);
    return COLD_OK;
  }
  if (st != COLD_OK) return COLD_FAIL;
  if (MODE == CONE_MINEIG) {
    if (l == 0) ca.out[k] = c.lam[0];
    return COLD_OK;
  }
  // ---- one Newton-Schulz step when V'V departs from I (lane j: column j)
  {
    double gcol[32];
    double dev = 0.0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      double g = 0.0;
      if (q < d && l < d)
        for (int i = 0; i < d; ++i) g = fma(c.Z[i * ld + l], c.Z[i * ld + q], g);
      gcol[q] = g;
      if (q < d && l < d) dev = fmax(dev, fabs(g - (q == l ? 1.0 : 0.0)));
    }
    dev = warp_allmax(dev);
    if (dev > 0x1p-46)
      for (int i = 0; i < d; ++i) {  // row by row: every lane reads row i, then writes its entry
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (q < d) acc = fma(c.Z[i * ld + q], gcol[q], acc);
        const double vn = l < d ? fma(-0.5, acc, 1.5 * c.Z[i * ld + l]) : 0.0;
        __syncwarp();
        if (l < d) c.Z[i * ld + l] = vn;
        __syncwarp();
      }
  }
  // ---- P = W W' (W = V_C sqrt |lam_C|, the smaller class C) or X + W W'
  int r = 0;
  for (int i = 0; i < d; ++i) r += c.lam[i] > 0.0;
  const bool pos = r <= d - r;
  const int c0 = pos ? d - r : 0, K = pos ? r : d - r;
  if (l >= c0 && l < c0 + K) {
    const double f = sqrt(fabs(c.lam[l]));
    for (int i = 0; i < d; ++i) c.Z[i * ld + l] *= f;
  }
  __syncwarp();
  double wrow[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) wrow[q] = (l < d && q < K) ? c.Z[l * ld + c0 + q] : 0.0;
  double *su = S.u + so + off, *sw = S.w + so + off;
  for (int i = 0; i < d; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (q < K) acc = fma(c.Z[i * ld + c0 + q], wrow[q], acc);
    if (l < d) {
      double pv = acc;
      if (!pos) {
        const double xa = MODE == CONE_HOT ? 0.5 * (xg[i * d + l] + xg[l * d + i])
                                           : 0.5 * (ca.in[off + i * d + l] + ca.in[off + l * d + i]) * ca.in_scale;
        pv += xa;
      }
      if (MODE == CONE_HOT) {
        su[i * d + l] = pv;
        sw[i * d + l] += pv;  // w_s = (w_s - us_h) + P (solver.py:391-394)
      } else {
        ca.out[off + i * d + l] = pv;
      }
    }
  }
  if (MODE == CONE_HOT && l == 0 && W.sweeps) W.sweeps[k] = 0;
  return COLD_OK;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_cone_wcold(DevProblem P, DevState S, DevWork W, ConeArgs ca) {
  extern __shared__ __align__(16) double smem[];
  const int wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + wid;
  if (gw >= ca.count) return;
  double *scratch = smem + (int64_t)wid * wcold_scratch_doubles(ca.dpmax);
  const int k = ca.ids[gw];
  const int st = P.cl_size[k] <= 32 ? wcold_one<MODE>(P, S, W, ca, k, scratch) : COLD_FAIL;
  if ((threadIdx.x & 31) == 0 && ca.cfail) ca.cfail[gw] = st == COLD_FAIL ? 1 : 0;
}
