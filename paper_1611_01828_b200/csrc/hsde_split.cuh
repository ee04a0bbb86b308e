// hsde_split.cuh -- fast path of the clique PSD projection for CTA-sized
// cliques (32 < d <= kSplitMaxD) on the warm hot path (reference:
// chordalsdp/symmat.py:153-165 `project_psd_batch` called from
// solver.py:335-342; the result is the same P = Q max(Lambda, 0) Q').
//
// The previous iteration's eigenbasis V (rows of the per-clique store, Vt)
// nearly diagonalises the new argument X.  With B = Vt X Vt' split by the
// sign of its diagonal into the classes P (r entries) and N (n = d - r), in
// class-sorted order, the positive invariant subspace of B is span Q,
// Q = [I; Y_X] with Y_X (n x r) the solution near 0 of the Riccati equation
//     Y_X L_P - L_N Y_X = B_NP + E_NN Y_X - Y_X (E_PP + B_PN Y_X)
// (L = diagonal, E = off-diagonal within a class; every denominator is
// >= 2 g, g = min |diag B|, so the fixed point contracts at about
// off(B) / 2g).  Then B Q = Q R with R = L_P + E_PP + B_PN Y_X, and the
// orthogonal projector onto span Q is Q G Q' with G = (I + Y_X' Y_X)^-1, so
//     P(B) = B Q G Q' = Q (R G) Q'      and      P(X) = Ut' K Ut,
// Ut = Vt_P + Y_X' Vt_N (r x d), K = R G (r x r).  No truncation: the only
// errors are the fixed point's (residual <= kSplitTol |B|_F) and rounding.  V
// itself is left unchanged, so it never loses orthogonality here.
//
// The path applies when off(B) <= g / 10 (then no eigenvalue changes sign,
// Weyl) and r <= n; otherwise -- or when the fixed point stalls -- the kernel
// writes B to the per-clique hand-off buffer and k_cone_block finishes the
// clique from there (Jacobi sweeps warm-started from B and V, which also
// refresh V).  Cliques without a valid V go to k_cone_block untouched.
//
// All products run on the fp64 tensor cores (mma.sync m8n8k4, DMMA) from
// shared memory with 16 x 16 output blocks per warp (four independent
// accumulator chains, one shared-memory load per DMMA); leading dimensions
// are 4 (mod 16) doubles, which makes every fragment load of either
// orientation bank-conflict free (two wavefronts per 32 lanes).  V is read
// from the store (L2) where it is an operand.
//
// (included inside namespace hsde by hsde_kernels.cuh, after hsde_eig.cuh)

constexpr int kSplitThreads = 384;
// plans whose largest clique has order <= kSplitSmallD run ten warps per CTA: the
// register cap rises from 80 to 96 per thread (two CTAs per SM either way) and B's 15
// upper blocks still fit 10 x 2 register blocks (config 4: +2% in steady state)
constexpr int kSplitThreadsSmall = 320;
constexpr int kSplitSmallD = 80;
constexpr int kSplitStrip = 32;  // warm-start strip width (columns of T = Vt X)
constexpr int kSplitMaxB = 2;    // 16 x 16 blocks a warp keeps in registers
constexpr int kSplitMaxD = 96;   // upper blocks of B: <= kSplitMaxB per warp
// B's upper 16 x 16 blocks live in registers during the warm start: all of
// them must be owned by some warp (nb = 6 -> 21 blocks <= 2 x 12)
static_assert(((kSplitMaxD + 15) / 16) * ((kSplitMaxD + 15) / 16 + 1) / 2 <= kSplitMaxB * (kSplitThreads / 32),
              "kSplitMaxD: B's upper blocks exceed the warps' register blocks");
static_assert(((kSplitSmallD + 15) / 16) * ((kSplitSmallD + 15) / 16 + 1) / 2 <= kSplitMaxB * (kSplitThreadsSmall / 32),
              "kSplitSmallD: B's upper blocks exceed the warps' register blocks");
constexpr int kSplitRefreshIters = 1000;  // fixed-point passes that ask for a Jacobi refresh of V
constexpr int kLoadBatch = 4;          // hot-path slots per thread in flight
constexpr double kSplitOff2 = 0.2;  // fast path while off(B)^2 <= kSplitOff2 g^2 (off < 0.45 g: Weyl keeps the inertia)
constexpr int kSplitMaxPasses = 24;     // fixed-point passes before handing over
// fixed-point stop: estimated remaining Riccati residual <= kSplitTol |B|_F
// (below the rounding of the d-term products themselves, ~ d eps |B|)
constexpr double kSplitTol = 1e-15;
constexpr double kSplitStall = 0.8;  // pass-to-pass ratio taken as a stall
// schedule key: off(B)^2 above kSplitKey2 of the bound marks a refresh candidate
constexpr double kSplitKey2 = 0.25;

__host__ __device__ inline int split_ld(int c) { return ((c + 11) & ~15) + 4; }

// R2 = [Y (r x ly) | S_N (n x ln), same region] [Ut (r x L)], or the strip buffer
__host__ __device__ inline int64_t split_r2_doubles(int d) {
  int64_t best = 2 * (int64_t)d * split_ld(kSplitStrip);  // strip buffers XS, TS
  for (int r = 1; r <= d / 2; ++r) {
    const int n = d - r;
    const int64_t y = (int64_t)r * split_ld(r), sn = (int64_t)n * split_ld(n);
    const int64_t need = (y > sn ? y : sn) + (int64_t)r * split_ld(d);
    if (need > best) best = need;
  }
  return best;
}

__host__ __device__ inline int64_t split_smem_doubles(int d) {
  // R1 | R2 | lam[d] | red[32] | ints: perm[d], pinv[d], cnt[4]
  return (int64_t)d * split_ld(d) + split_r2_doubles(d) + d + 32 + (2 * d + 4 + 1) / 2 + 1;
}

// operand view: element (row, col) at p[row * rs + col * cs]
struct Opd {
  const double *p;
  int rs, cs;
};

// One 16 x 16 output block (2 x 2 m8n8k4 tiles) of sum_{k < K} A(i, k) B(k, j)
// accumulated into c (lane (q, kk) = (lane / 4, lane % 4) holds
// c[a][b][e] = D(i0 + 8a + q, j0 + 8b + 2kk + e)).  Rows >= M and columns >= N
// read a clamped valid row / column (their results are discarded by the
// caller); k >= K is zero-filled.  BROW: B's row k is brow[k] (row gather).
// UNR: k-steps per trip (an operand in global memory wants the loads of several
// k-steps in flight: L2 latency, not shared-memory latency, paces the chain).
template <bool BROW = false, int UNR = 2>
__device__ __forceinline__ void blk16(double (&c)[2][2][2], const Opd &A, const Opd &B, int i0, int j0, int M,
                                      int N, int K, const int *brow = nullptr) {
  const int lane = threadIdx.x & 31, q = lane >> 2, kk = lane & 3;
  const int ia0 = min(i0 + q, M - 1), ia1 = min(i0 + 8 + q, M - 1);
  const int jb0 = min(j0 + q, N - 1), jb1 = min(j0 + 8 + q, N - 1);
  const double *a0 = A.p + ia0 * A.rs + kk * A.cs, *a1 = A.p + ia1 * A.rs + kk * A.cs;
  const double *b0 = B.p + jb0 * B.cs, *b1 = B.p + jb1 * B.cs;
  if (!BROW) {
    b0 += kk * B.rs;
    b1 += kk * B.rs;
  }
  const int sa = 4 * A.cs, sb = 4 * B.rs;
  const int K4 = K & ~3;
  // second tile row / column outside the output: skip its products (warp-uniform)
  const bool ha = i0 + 8 < M, hb = j0 + 8 < N;
  int k0 = 0;
  if (UNR > 2) {
    // batches of UNR k-steps: every operand load of the batch issued before its products
    for (; k0 + 4 * UNR <= K4; k0 += 4 * UNR) {
      double x0[UNR], x1[UNR], y0[UNR], y1[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        x0[u] = a0[u * sa];
        x1[u] = a1[u * sa];
        if (BROW) {
          const int ro = brow[k0 + 4 * u + kk] * B.rs;
          y0[u] = b0[ro];
          y1[u] = b1[ro];
        } else {
          y0[u] = b0[u * sb];
          y1[u] = b1[u * sb];
        }
      }
      a0 += UNR * sa;
      a1 += UNR * sa;
      if (!BROW) {
        b0 += UNR * sb;
        b1 += UNR * sb;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        dmma884(c[0][0][0], c[0][0][1], x0[u], y0[u]);
        if (hb) dmma884(c[0][1][0], c[0][1][1], x0[u], y1[u]);
        if (ha) dmma884(c[1][0][0], c[1][0][1], x1[u], y0[u]);
        if (ha && hb) dmma884(c[1][1][0], c[1][1][1], x1[u], y1[u]);
      }
    }
  }
#pragma unroll 2
  for (; k0 < K4; k0 += 4) {
    double x0 = *a0, x1 = *a1, y0, y1;
    if (BROW) {
      const int ro = brow[k0 + kk] * B.rs;
      y0 = b0[ro];
      y1 = b1[ro];
    } else {
      y0 = *b0;
      y1 = *b1;
      b0 += sb;
      b1 += sb;
    }
    a0 += sa;
    a1 += sa;
    dmma884(c[0][0][0], c[0][0][1], x0, y0);
    if (hb) dmma884(c[0][1][0], c[0][1][1], x0, y1);
    if (ha) dmma884(c[1][0][0], c[1][0][1], x1, y0);
    if (ha && hb) dmma884(c[1][1][0], c[1][1][1], x1, y1);
  }
  if (k0 < K) {
    double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
    if (k0 + kk < K) {
      x0 = *a0;
      x1 = *a1;
      if (BROW) {
        const int ro = brow[k0 + kk] * B.rs;
        y0 = b0[ro];
        y1 = b1[ro];
      } else {
        y0 = *b0;
        y1 = *b1;
      }
    }
    dmma884(c[0][0][0], c[0][0][1], x0, y0);
    dmma884(c[0][1][0], c[0][1][1], x0, y1);
    dmma884(c[1][0][0], c[1][0][1], x1, y0);
    dmma884(c[1][1][0], c[1][1][1], x1, y1);
  }
}

__device__ __forceinline__ void blk16_zero(double (&c)[2][2][2]) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) c[a][b][0] = c[a][b][1] = 0.0;
}

// visit the valid elements of a block: f(i, j, v)
template <class F>
__device__ __forceinline__ void blk16_each(const double (&c)[2][2][2], int i0, int j0, int M, int N, F f) {
  const int lane = threadIdx.x & 31, q = lane >> 2, kk = lane & 3;
  if (i0 + 16 <= M && j0 + 16 <= N) {  // interior block (warp-uniform): no per-element bounds tests
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) f(i0 + 8 * a + q, j0 + 8 * b + 2 * kk + e, c[a][b][e]);
    return;
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = i0 + 8 * a + q, j = j0 + 8 * b + 2 * kk + e;
        if (i < M && j < N) f(i, j, c[a][b][e]);
      }
}

// block t of the upper triangle (bi <= bj) of an nb x nb block grid
__device__ __forceinline__ void upper_block(int t, int nb, int &bi, int &bj) {
  bi = 0;
  while (t >= nb - bi) {
    t -= nb - bi;
    ++bi;
  }
  bj = bi + t;
}

// out = A1 B1 (K1) + A2 B2 (K2) over M x N in 16 x 16 blocks, round-robin
// over the warps.  SYM (M == N): upper blocks only, emitted to both
// triangles from the upper values (exactly symmetric).  INPLACE: every warp
// finishes reading before the first emit (the output may overwrite an
// operand; at most kSplitMaxB blocks per warp).  Ends with a barrier.
template <bool SYM, bool INPLACE, bool BROW = false, int UNR = 2, class Emit>
__device__ void team_mm(int M, int N, const Opd &A1, const Opd &B1, int K1, const Opd &A2, const Opd &B2, int K2,
                        Emit emit, const int *brow = nullptr) {
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int mb = (M + 15) >> 4, nb = (N + 15) >> 4;
  const int nblk = SYM ? mb * (mb + 1) / 2 : mb * nb;
  auto place = [&](int t, int &i0, int &j0) {
    int bi, bj;
    if (SYM) upper_block(t, mb, bi, bj);
    else {
      bi = t / nb;
      bj = t - bi * nb;
    }
    i0 = bi * 16;
    j0 = bj * 16;
  };
  auto out = [&](const double (&c)[2][2][2], int i0, int j0) {
    if (SYM) {
      blk16_each(c, i0, j0, M, N, [&](int i, int j, double v) {
        if (i0 != j0 || i < j) {
          emit(i, j, v);
          emit(j, i, v);
        } else if (i == j) {
          emit(i, j, v);
        }
      });
    } else {
      blk16_each(c, i0, j0, M, N, emit);
    }
  };
  if (INPLACE) {
    double c[kSplitMaxB][2][2][2];
#pragma unroll
    for (int s = 0; s < kSplitMaxB; ++s) {
      blk16_zero(c[s]);
      const int t = w + s * nw;
      if (t < nblk) {
        int i0, j0;
        place(t, i0, j0);
        if (K1 > 0) blk16<BROW, UNR>(c[s], A1, B1, i0, j0, M, N, K1, brow);
        if (K2 > 0) blk16(c[s], A2, B2, i0, j0, M, N, K2);
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kSplitMaxB; ++s) {
      const int t = w + s * nw;
      if (t < nblk) {
        int i0, j0;
        place(t, i0, j0);
        out(c[s], i0, j0);
      }
    }
  } else {
    for (int t = w; t < nblk; t += nw) {
      double c[2][2][2];
      blk16_zero(c);
      int i0, j0;
      place(t, i0, j0);
      if (K1 > 0) blk16<BROW, UNR>(c, A1, B1, i0, j0, M, N, K1, brow);
      if (K2 > 0) blk16(c, A2, B2, i0, j0, M, N, K2);
      out(c, i0, j0);
    }
  }
  __syncthreads();
}

template <bool SYM, bool INPLACE, bool BROW = false, int UNR = 2, class Emit>
__device__ __forceinline__ void team_mm1(int M, int N, const Opd &A, const Opd &B, int K, Emit emit,
                                         const int *brow = nullptr) {
  team_mm<SYM, INPLACE, BROW, UNR>(M, N, A, B, K, A, B, 0, emit, brow);
}

__device__ __forceinline__ double cta_sum(double v, double *red) {
  BlockTeam tm{(int)threadIdx.x, (int)blockDim.x};
  return team_sum(tm, v, red);
}
__device__ __forceinline__ double cta_min(double v, double *red) {
  BlockTeam tm{(int)threadIdx.x, (int)blockDim.x};
  return team_min(tm, v, red);
}

// phase timestamps of the first CTA (diagnostics: W.dbg[48 + i], clock64)
#define SPLIT_STAMP(i)                                                                      \
  do {                                                                                      \
    if (W.dbg && blockIdx.x == 0 && threadIdx.x == 0) W.dbg[48 + (i)] = (double)clock64(); \
  } while (0)

// floor(e / m) for 0 <= e < 2^21 and 1 <= m <= 4096 from inv = 1.0f / m: the
// exact quotient of e + 1/2 sits >= 1/(2m) from an integer, far above the
// float rounding (no integer division in the element loops)
__device__ __forceinline__ int qdiv(int e, float inv) { return (int)(((float)e + 0.5f) * inv); }

// 1 / x to ~1 ulp without the division's slow-path branch (a float seed and
// three Newton steps, no branch: the element loops interleave several of
// these).  The Riccati denominators
// only need a consistent, accurate value: an ulp in 1 / Delta moves the fixed
// point like an ulp in diag B.
__device__ __forceinline__ double fast_rcp(double x) {
  // (x outside the float range gives inf / NaN: the fixed point then reads as
  // stalled and the clique goes to the cold path)
  double y = (double)__frcp_rn(__double2float_rn(x));
  y = fma(y, fma(-x, y, 1.0), y);
  y = fma(y, fma(-x, y, 1.0), y);
  y = fma(y, fma(-x, y, 1.0), y);
  return y;
}

// every in-place pass keeps its output blocks in registers (kSplitMaxB per warp)
__device__ __forceinline__ bool split_fits(int r, int n, int nw) {
  const int br = (r + 15) >> 4, bn = (n + 15) >> 4, bd = (r + n + 15) >> 4, cap = kSplitMaxB * nw;
  return bn * br <= cap && bn * bn + br * br <= cap && bn * bd <= cap;
}

// sum over the CTA of one value per thread, after the caller's barrier has
// made the per-warp partials (red[w], written by lane 0) visible
__device__ __forceinline__ double red_total(const double *red, int nw) {
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

// The fast path for clique k (argument load included).  Returns SPLIT_DONE,
// or a hand-off code with B = Vt X Vt' (original order) written to W.xarg.
__device__ int split_one(const DevProblem &P, const DevState &S, const DevWork &W, const ConeArgs &ca, int k,
                         double *smem) {
  const int d = P.cl_size[k];
  const int tid = threadIdx.x, T = blockDim.x;
  const int64_t off = P.cl_off[k], so = P.n_c;
  const double shift = W.scal[S_SHIFT];
  const double *vst = W.vstore + off;  // row c = basis vector c
  const int L = split_ld(d);
  double *R1 = smem, *R2 = R1 + d * L;
  double *lam = R2 + split_r2_doubles(d), *red = lam + d;
  int *perm = reinterpret_cast<int *>(red + 32), *pinv = perm + d, *cnt = pinv + d;
  const int w = tid >> 5, nw = T >> 5, lane = tid & 31;
  const float invd = 1.0f / d;
  double *su = S.u + so + off, *sw = S.w + so + off;
  bool refreshed = false;  // (stats) Jacobi sweeps refreshed the basis in this call
  SPLIT_STAMP(0);

  {
  // ---- argument X (hot-path slot update, solver.py:222-244, :316, :388-394),
    //      kLoadBatch slots per thread at a time: every load of the batch is
    //      issued before the first store (the stores may alias later loads)
    {
      constexpr int NB = kLoadBatch;
      const int64_t vo = P.n_c + P.n_d + P.m;
      const double *mzs = P.mz + P.n_c + off, *mzv = P.mz + vo + off;
      double *vu = S.u + vo + off, *vw = S.w + vo + off;
      for (int e0 = tid; e0 < d * d; e0 += NB * T) {
        double us[NB], ws[NB], uv[NB], wv[NB], hu[NB], ms[NB], mv[NB];
        int cv[NB];
  #pragma unroll
        for (int q = 0; q < NB; ++q) {
          const int e = min(e0 + q * T, d * d - 1);
          us[q] = su[e];
          ws[q] = sw[e];
          uv[q] = vu[e];
          wv[q] = vw[e];
          ms[q] = mzs[e];
          mv[q] = mzv[e];
          cv[q] = P.slot_cov[off + e];
        }
  #pragma unroll
        for (int q = 0; q < NB; ++q) hu[q] = W.ua[cv[q]];
  #pragma unroll
        for (int q = 0; q < NB; ++q) {
          const int e = e0 + q * T;
          if (e >= d * d) break;
          const double as = us[q] + ws[q], av = uv[q] + wv[q];            // a = u + w
          const double gb = as - av;                                      // solver.py:222
          const double ub = (gb + hu[q]) * 0.5;                           // :237-239
          const double uvn = (ub - hu[q]) + av;                           // :242-244
          const double us_h = relax(ub - shift * ms[q], us[q], P.alpha);  // :316, :388-390
          const double uv_h = relax(uvn - shift * mv[q], uv[q], P.alpha);
          const double vn = uv_h - wv[q];                                 // free block: identity
          vu[e] = vn;
          vw[e] = (wv[q] - uv_h) + vn;                                    // :393-394
          sw[e] = ws[q] - us_h;                                           // completed after projection
          const int a = qdiv(e, invd), b = e - a * d;
          R1[a * L + b] = us_h - ws[q];                                   // :391
        }
      }
    }
    __syncthreads();
    for (int e = tid; e < d * d; e += T) {  // sym = 0.5 (B + B')  (symmat.py:157)
      const int a = qdiv(e, invd), b = e - a * d;
      if (a < b) {
        const double s = 0.5 * (R1[a * L + b] + R1[b * L + a]);
        R1[a * L + b] = s;
        R1[b * L + a] = s;
      }
    }
    __syncthreads();
    SPLIT_STAMP(1);
  }
  // ---- second wave: the clique that takes a slot of this wave next
  //      (blockIdx + resident slots) gets its inputs prefetched into L2 now --
  //      HBM is idle while the first wave computes (its loads all came at once)
  if (ca.pf_ahead > 0 && (int)blockIdx.x + ca.pf_ahead < ca.count) {
    const int kp = ca.ids[blockIdx.x + ca.pf_ahead];
    if (!(W.ccur && W.ccur[kp])) {
      const int64_t po = P.cl_off[kp], vo = P.n_c + P.n_d + P.m;
      const int dq = P.cl_size[kp];
      const int nl = (dq * dq * 8 + 127) >> 7;  // 128-byte lines per d x d array
      auto pf = [&](const double *base) {
        for (int ln = tid; ln < nl; ln += T)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char *>(base) + ((int64_t)ln << 7)));
      };
      pf(S.u + so + po);
      pf(S.w + so + po);
      pf(S.u + vo + po);
      pf(S.w + vo + po);
      pf(P.mz + P.n_c + po);
      pf(P.mz + vo + po);
      pf(W.vstore + po);
      for (int e = tid; e < (nl + 1) / 2; e += T)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char *>(P.slot_cov + po) + ((int64_t)e << 7)));
    }
  }
  // ---- B = Vt X Vt' by column strips of T = Vt X, all from shared memory:
  //      X -> the hand-off buffer (global, L2-resident), Vt -> R1, then per
  //      strip J: X[:, J] -> XS, T_J = Vt X[:, J] -> TS, B += T_J Vt[:, J]'
  //      (upper 16 x 16 blocks of B held in registers); the next strip of X
  //      is fetched while the tensor cores work on the current one
  const int nb = (d + 15) >> 4, nbu = nb * (nb + 1) / 2;
  const int LS = split_ld(kSplitStrip);
  double *XS = R2, *TS = R2 + d * LS;
  double *xg = W.xarg + off;
  double cb[kSplitMaxB][2][2][2];
  int bi0[kSplitMaxB], bj0[kSplitMaxB];
#pragma unroll
  for (int s = 0; s < kSplitMaxB; ++s) {
    blk16_zero(cb[s]);
    const int t = w + s * nw;
    int bi = 0, bj = 0;
    if (t < nbu) upper_block(t, nb, bi, bj);
    bi0[s] = bi * 16;
    bj0[s] = bj * 16;
  }
  {
  for (int e = tid; e < d * d; e += T) {
    const int a = qdiv(e, invd), b = e - a * d;
    xg[e] = R1[a * L + b];
  }
  __syncthreads();
  for (int e = tid; e < d * d; e += T) {
    const int a = qdiv(e, invd), b = e - a * d;
    R1[a * L + b] = vst[e];
  }
  {
    const int s0 = min(kSplitStrip, d);
    for (int e = tid; e < d * s0; e += T) {
      const int a = qdiv(e, 1.0f / s0), b = e - a * s0;
      XS[a * LS + b] = xg[a * d + b];
    }
  }
  __syncthreads();
  constexpr int kPf = (kSplitMaxD * kSplitStrip + kSplitThreadsSmall - 1) / kSplitThreadsSmall;  // covers both CTA sizes
  for (int j0 = 0; j0 < d; j0 += kSplitStrip) {
    const int sw_ = min(kSplitStrip, d - j0), nbs = (sw_ + 15) >> 4;
    for (int t = w; t < nb * nbs; t += nw) {
      const int bi = qdiv(t, 1.0f / nbs), bj = t - bi * nbs;
      double c[2][2][2];
      blk16_zero(c);
      blk16(c, Opd{R1, L, 1}, Opd{XS, LS, 1}, bi * 16, bj * 16, d, sw_, d);
      blk16_each(c, bi * 16, bj * 16, d, sw_, [&](int i, int j, double v) { TS[i * LS + j] = v; });
    }
    __syncthreads();
    // next strip of X: loads issued before this strip's products, stored after
    const int j1 = j0 + kSplitStrip, s1 = j1 < d ? min(kSplitStrip, d - j1) : 0;
    const float inv1 = 1.0f / max(s1, 1);
    double pf[kPf];
#pragma unroll
    for (int q = 0; q < kPf; ++q) {
      const int e = tid + q * T;
      pf[q] = 0.0;
      if (e < d * s1) {
        const int a = qdiv(e, inv1), b = e - a * s1;
        pf[q] = xg[a * d + j1 + b];
      }
    }
#pragma unroll
    for (int s = 0; s < kSplitMaxB; ++s)
      if (w + s * nw < nbu) blk16(cb[s], Opd{TS, LS, 1}, Opd{R1 + j0, 1, L}, bi0[s], bj0[s], d, d, sw_);
#pragma unroll
    for (int q = 0; q < kPf; ++q) {
      const int e = tid + q * T;
      if (e < d * s1) {
        const int a = qdiv(e, inv1), b = e - a * s1;
        XS[a * LS + b] = pf[q];
      }
    }
    __syncthreads();
  }
  }
  SPLIT_STAMP(2);

  // ---- diagonal, g = min |diag|, off(B)^2 (upper values, mirrored)
  double o2, g, nb2;  // off(B)^2, min |diag|, |B|_F^2
  auto measure = [&]() {
    o2 = 0.0;
#pragma unroll
    for (int s = 0; s < kSplitMaxB; ++s)
      if (w + s * nw < nbu)
        blk16_each(cb[s], bi0[s], bj0[s], d, d, [&](int i, int j, double v) {
          if (i == j) lam[i] = v;
          else if (i < j) o2 += 2.0 * v * v;
        });
    __syncthreads();
    g = CUDART_INF;
    double l2 = 0.0;
    for (int i = tid; i < d; i += T) {
      g = fmin(g, fabs(lam[i]));
      l2 += lam[i] * lam[i];
    }
    g = cta_min(g, red);
    o2 = cta_sum(o2, red);
    nb2 = o2 + cta_sum(l2, red);
  };
  measure();
  if (!(o2 <= kSplitOff2 * g * g) && g > 0.0 && o2 < CUDART_INF && ca.cold && o2 > 0.36 * g * g) {
    // the kept basis is far from diagonalising X (off(B) > 0.6 g): the cold path
    // (hsde_cold.cuh) re-diagonalises X (still in xg); closer to the bound a
    // warm Jacobi refresh in this CTA is cheaper (below)
    return SPLIT_HANDOFF + 3;
  }
  if (!(o2 <= kSplitOff2 * g * g) && g > 0.0 && o2 < CUDART_INF) {
    // far above the bound (off(B) > 0.6 g): the cold path next iteration
    if (tid == 0 && W.cnext) W.cnext[k] = o2 > 0.36 * g * g ? 1 : 0;
    // (Jacobi variant) Jacobi sweeps on B, warm from V (hsde_eig.cuh), in this
    // CTA until the class-split point; then the split goes on with the
    // rotated B and V.  (B is in registers, X and V in global memory: the
    // Jacobi scratch may overwrite the whole shared-memory area.)
    const int dp = d + (d & 1);
    BlockTeam tm{tid, T};
    JacobiScratch js = jacobi_carve(smem, dp);
#pragma unroll
    for (int s = 0; s < kSplitMaxB; ++s)
      if (w + s * nw < nbu)
        blk16_each(cb[s], bi0[s], bj0[s], d, d, [&](int i, int j, double v) {
          if (i <= j) {
            js.A[i * js.lda + j] = v;
            js.A[j * js.lda + i] = v;
          }
        });
    for (int e = tid; e < dp * js.ldv; e += T) {
      const int i = e / js.ldv, j = e - i * js.ldv;
      js.Vt[e] = (i < d && j < d) ? vst[i * d + j] : (i == j ? 1.0 : 0.0);
    }
    if (d & 1)
      for (int e = tid; e < dp; e += T) {
        js.A[d * js.lda + e] = 0.0;
        js.A[e * js.lda + d] = 0.0;
      }
    jacobi_prepare(tm, js, dp, false);
    __syncthreads();
    int order = 0;
    jacobi_sweeps(tm, js, d, dp, &order, 3);
    double *vw = W.vstore + off;
    for (int e = tid; e < d * d; e += T) {
      const int a = qdiv(e, invd), b = e - a * d;
      vw[e] = js.Vt[a * js.ldv + b];
    }
    {
      const int q = lane >> 2, kk = lane & 3;
#pragma unroll
      for (int s = 0; s < kSplitMaxB; ++s)
        if (w + s * nw < nbu)
#pragma unroll
          for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
            for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
              for (int e2 = 0; e2 < 2; ++e2) {
                const int i = min(bi0[s] + 8 * a2 + q, d - 1), j = min(bj0[s] + 8 * b2 + 2 * kk + e2, d - 1);
                cb[s][a2][b2][e2] = js.A[i * js.lda + j];
              }
    }
    __syncthreads();  // the scratch overlaps lam / red / perm
    if (tid == 0 && W.sweeps) W.sweeps[k] = 0;
    measure();
    refreshed = true;
  }
  // class-sorted order: perm[0, r) = P (diag > 0), perm[r, d) = N
  auto classify = [&]() {
    if (tid < 32) {
      int base = 0;
      for (int pass = 0; pass < 2; ++pass)
        for (int i0 = 0; i0 < d; i0 += 32) {
          const int i = i0 + tid;
          const bool pk = i < d && ((lam[i] > 0.0) == (pass == 0));
          const unsigned mk = __ballot_sync(0xffffffffu, pk);
          if (pk) {
            const int pos = base + __popc(mk & ((1u << tid) - 1u));
            perm[pos] = i;
            pinv[i] = pos;
          }
          base += __popc(mk);
          if (pass == 0 && i0 + 32 >= d && tid == 0) cnt[0] = base;
        }
    }
    __syncthreads();
  };
  classify();
  // more positive than non-positive eigenvalues: project -B instead, X+ = X + (-X)+
  // (the paths below need r <= n)
  const bool neg = 2 * cnt[0] > d;
  if (neg) {
#pragma unroll
    for (int s = 0; s < kSplitMaxB; ++s)
#pragma unroll
      for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) {
          cb[s][a2][b2][0] = -cb[s][a2][b2][0];
          cb[s][a2][b2][1] = -cb[s][a2][b2][1];
        }
    if (tid < d) lam[tid] = -lam[tid];
    __syncthreads();
    classify();
  }
  const double bsign = neg ? -1.0 : 1.0;  // hand-overs carry B itself
  const int r = cnt[0], n = d - r;
  const float invr = 1.0f / max(r, 1), invn = 1.0f / max(n, 1);
  // off(B) < g keeps the inertia (Weyl: |E|_2 <= |E|_F < min |diag|); the
  // fixed point contracts at about off / 2g, so a looser bound only costs passes
  const bool applies = g > 0.0 && o2 <= kSplitOff2 * g * g && r <= n &&  // also false on NaN
                       split_fits(r, n, nw);
  if (!applies && ca.cold) return SPLIT_HANDOFF + 1;  // X stays in xg for the cold path
  if (!applies) {
    // hand B (original order) to the Jacobi path
    double *xb = W.xarg + off;
#pragma unroll
    for (int s = 0; s < kSplitMaxB; ++s)
      if (w + s * nw < nbu)
        blk16_each(cb[s], bi0[s], bj0[s], d, d, [&](int i, int j, double v) {
          if (i <= j) {
            xb[i * d + j] = bsign * v;
            xb[j * d + i] = bsign * v;
          }
        });
    return r > n ? SPLIT_HANDOFF + 1 : SPLIT_HANDOFF;  // reason: r > n / off(B) > g / 10
  }
  // sorted B with a zero diagonal into R1 (X is dead), sorted diagonal into lam
  const double lsv = tid < d ? lam[perm[tid]] : 0.0;
#pragma unroll
  for (int s = 0; s < kSplitMaxB; ++s)
    if (w + s * nw < nbu)
      blk16_each(cb[s], bi0[s], bj0[s], d, d, [&](int i, int j, double v) {
        const int pi = pinv[i], pj = pinv[j];
        if (i < j) {
          R1[pi * L + pj] = v;
          R1[pj * L + pi] = v;
        } else if (i == j) {
          R1[pi * L + pi] = 0.0;
        }
      });
  __syncthreads();
  if (tid < d) lam[tid] = lsv;
  __syncthreads();
  SPLIT_STAMP(3);

  if (r == 0) {  // no eigenvalue > 0: P = 0, or X if B was negated (w_s holds ws - us_h already)
    if (tid == 0) W.ckey[k] = 0;
    for (int e = tid; e < d * d; e += T) {
      const double p = neg ? xg[e] : 0.0;
      su[e] = p;
      if (neg) sw[e] += p;
    }
    return SPLIT_DONE;
  }

  // ---- Riccati fixed point, Y_X in the N-P block of R1 (B_NP = B_PN').
  // One product pass per iteration: the quadratic term uses the previous
  // iterate (lagged), X_{k+1} = (B_NP + E_NN X_k + X_k Yn_{k-1}) / Delta with
  // Yn_k = -(E_PP + B_PN X_k) formed in the same pass (same fixed point; the
  // lag adds ~ |X| off / 2g to the contraction factor).
  const Opd EPP{R1, L, 1}, BPN{R1 + r, L, 1}, ENN{R1 + r * L + r, L, 1}, XX{R1 + r * L, L, 1};
  const int ly = split_ld(r);
  const int ln = split_ld(n);
  const int snoff = max(r * ly, n * ln);
  double *Ybuf[2] = {R2, R2 + r * ly};  // (the second overlaps S_N / Ut, formed later)
  double *Ut = R2 + snoff;
  double x2 = 0.0;
  for (int e = tid; e < n * r; e += T) {
    const int i = qdiv(e, invr), j = e - i * r;
    const double bnp = R1[(r + i) * L + j];
    R1[(r + i) * L + j] = bnp * fast_rcp(lam[j] - lam[r + i]);
    x2 += bnp * bnp;  // the first increment in residual units (Delta * dX)
  }
  __syncthreads();
  // Yn_0 = -(E_PP + B_PN X_0)
  team_mm1<false, false>(r, r, BPN, XX, n, [&](int i, int j, double v) { Ybuf[0][i * ly + j] = -(v + R1[i * L + j]); });
  const double inb2 = nb2 > 0.0 ? 1.0 / nb2 : 0.0;
  float prev = sqrtf((float)(cta_sum(x2, red) * inb2)), prev2 = prev;  // increments relative to |B|_F
  const float tolR = (float)kSplitTol;
  bool ok = prev == 0.0f;
  int it = 0, yb = 0;
  const int mb = (n + 15) >> 4, nbr = (r + 15) >> 4, nx = mb * nbr, ny = nbr * nbr;
  const float invbr = 1.0f / nbr, invbn = 1.0f / mb, invbd = 1.0f / ((d + 15) >> 4);
  for (; !ok && it < kSplitMaxPasses; ++it) {
    // pass: X blocks staged in registers (in place), Yn_{k} blocks emitted to the other buffer
    double c[kSplitMaxB][2][2][2];
    const double *Yc = Ybuf[yb];
    double *Yo = Ybuf[yb ^ 1];
#pragma unroll
    for (int s = 0; s < kSplitMaxB; ++s) {
      blk16_zero(c[s]);
      const int t = w + s * nw;
      if (t < nx) {
        const int bi = qdiv(t, invbr), bj = t - bi * nbr;
        blk16(c[s], ENN, XX, bi * 16, bj * 16, n, r, n);
        blk16(c[s], XX, Opd{Yc, ly, 1}, bi * 16, bj * 16, n, r, r);
      }
    }
    // the quadratic term moves ~|X| off / 2g per pass (well below the linear
    // contraction): refresh Yn on odd passes only (lag <= 2; Ybuf[0] = Yn(X_0))
    const bool newy = (it & 1) != 0;
    for (int t = ((w - nx) % nw + nw) % nw; newy && t < ny; t += nw) {  // round robin after the X blocks
      const int bi = qdiv(t, invbr), bj = t - bi * nbr;
      double cy[2][2][2];
      blk16_zero(cy);
      blk16(cy, BPN, XX, bi * 16, bj * 16, r, r, n);
      blk16_each(cy, bi * 16, bj * 16, r, r, [&](int i, int j, double v) { Yo[i * ly + j] = -(v + R1[i * L + j]); });
    }
    __syncthreads();
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < kSplitMaxB; ++s) {
      const int t = w + s * nw;
      if (t < nx) {
        // the block's eight elements per lane as straight-line code on clamped
        // indices (independent chains interleave; only the stores are predicated)
        const int bi = qdiv(t, invbr), bj = t - bi * nbr;
        const int q = lane >> 2, kk = lane & 3;
#pragma unroll
        for (int h4 = 0; h4 < 2; ++h4) {  // (four at a time: eight cost spills under the 80-register cap)
          double xn[4], dxs[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int a = h4, b = u >> 1, e = u & 1;
            const int i = min(bi * 16 + 8 * a + q, n - 1), j = min(bj * 16 + 8 * b + 2 * kk + e, r - 1);
            const double dl = lam[j] - lam[r + i];
            const double x = (R1[j * L + r + i] + c[s][a][b][e]) * fast_rcp(dl);
            dxs[u] = (x - R1[(r + i) * L + j]) * dl;  // increment in residual units
            xn[u] = x;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int a = h4, b = u >> 1, e = u & 1;
            const int i = bi * 16 + 8 * a + q, j = bj * 16 + 8 * b + 2 * kk + e;
            if (i < n && j < r) {
              acc = fma(dxs[u], dxs[u], acc);
              R1[(r + i) * L + j] = xn[u];
            }
          }
        }
      }
    }
    acc = warp_sum(acc);
    double *rb = red + 16 * (it & 1);  // alternating halves: no barrier before the next pass writes
    if (lane == 0) rb[w] = acc;
    __syncthreads();
    // the decision runs in float on residuals relative to |B|_F (every thread
    // the same deterministic arithmetic; an fp64 sqrt and two divisions per pass
    // sat on the critical path of every warp)
    double tot = lane < nw ? rb[lane] : 0.0;  // butterfly: the same bits in every lane and warp
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    const float delta = sqrtf((float)(tot * inb2));
    if (newy) yb ^= 1;
    // contraction per pass: over two passes (the lagged quadratic term makes
    // consecutive increments non-monotone), over one for the first pass
    const float rho = it == 0 ? delta / prev : sqrtf(delta / prev2);
    // Increments are measured in residual units (Delta o dY, the Riccati residual
    // the pass removed), against |B|_F: X then solves the Riccati equation of a
    // matrix within ~kSplitTol |B|_F of B, and P(.) is 1-Lipschitz, so P is
    // accurate to that level even where Y itself is ill-conditioned (tiny g)
    // and stops improving at ~eps |B| / g.  Converged: the estimated remaining
    // residual delta rho / (1 - rho) is below the tolerance, or the increment
    // itself is at the rounding level; stalled: no contraction (or NaN) -- the
    // pass budget bounds slow contraction.
    if (delta <= 0.1f * tolR || (rho < (float)kSplitStall && delta * rho <= tolR * (1.0f - rho))) ok = true;
    else if (!(rho < (float)kSplitStall)) {
      if (W.dbg && tid == 0) {  // diagnostics: (refreshed, pass, rho, delta, g, off, r) of up to 4 stalls
        const unsigned long long c = atomicAdd(reinterpret_cast<unsigned long long *>(W.dbg + 23), 1ull);
        if (c < 4) {
          double *o = W.dbg + 24 + 7 * c;
          o[0] = refreshed; o[1] = it; o[2] = rho; o[3] = delta; o[4] = g; o[5] = sqrt(o2); o[6] = r;
        }
      }
      break;
    }
    prev2 = prev;
    prev = delta;
  }
  __syncthreads();  // every warp has read the last pass's partials
  if (!ok && ca.cold) return SPLIT_HANDOFF + 2;  // stalled: X stays in xg for the cold path
  if (!ok) {
    // hand B back (original order): N-P block from B_PN', diagonal from lam
    double *xb = W.xarg + off;
    for (int e = tid; e < d * d; e += T) {
      const int i = qdiv(e, invd), j = e - i * d;
      const int pi = pinv[i], pj = pinv[j];
      double v;
      if (pi == pj) v = lam[pi];
      else if (pi >= r && pj < r) v = R1[pj * L + pi];
      else v = R1[pi * L + pj];
      xb[e] = bsign * v;
    }
    return SPLIT_HANDOFF + 2;  // reason: stalled
  }
  SPLIT_STAMP(4);
  if (W.dbg && blockIdx.x == 0 && tid == 0) W.dbg[47] = it;
  // ---- one pass over the final X:  Y = E_PP + B_PN X (R = L_P + Y) -> Yb,
  //      Y_P = X' X -> YPt (Ut's region, temporary), Y_N = X X' -> E_NN block
  const bool vup = ca.split_vupdate != 0;
  const int nbn = mb;
  double *Yb = Ybuf[0], *YPt = Ut, *EX = R2;  // EX: n x ln (S_N, after Y is dead)
  double y2 = 0.0;
  {
    const int nyu = nbr * (nbr + 1) / 2, nyn = vup ? nbn * (nbn + 1) / 2 : 0;
    for (int t = w; t < ny + nyu + nyn; t += nw) {
      double cy[2][2][2];
      blk16_zero(cy);
      if (t < ny) {
        const int bi = qdiv(t, invbr), bj = t - bi * nbr;
        blk16(cy, BPN, XX, bi * 16, bj * 16, r, r, n);
        blk16_each(cy, bi * 16, bj * 16, r, r, [&](int i, int j, double v) { Yb[i * ly + j] = v + R1[i * L + j]; });
      } else if (t < ny + nyu) {
        int bi, bj;
        upper_block(t - ny, nbr, bi, bj);
        blk16(cy, Opd{R1 + r * L, 1, L}, XX, bi * 16, bj * 16, r, r, n);
        blk16_each(cy, bi * 16, bj * 16, r, r, [&](int i, int j, double v) {
          if (bi != bj || i < j) {
            YPt[i * ly + j] = v;
            YPt[j * ly + i] = v;
            y2 += 2.0 * v * v;
          } else if (i == j) {
            YPt[i * ly + i] = v;
            y2 += v * v;
          }
        });
      } else {
        int bi, bj;
        upper_block(t - ny - nyu, nbn, bi, bj);
        blk16(cy, XX, Opd{R1 + r * L, 1, L}, bi * 16, bj * 16, n, n, r);
        double *YN = R1 + r * L + r;
        blk16_each(cy, bi * 16, bj * 16, n, n, [&](int i, int j, double v) {
          if (bi != bj || i < j) {
            YN[i * L + j] = v;
            YN[j * L + i] = v;
          } else if (i == j) {
            YN[i * L + i] = v;
          }
        });
      }
    }
  }
  y2 = warp_sum(y2);
  if (lane == 0) red[w] = y2;
  __syncthreads();
  const double y = sqrt(red_total(red, nw));
  int nt = 0;  // series terms: y^(nt+1) <= 1e-17
  for (double p = y; nt < 40 && p > 1e-17; p *= y) ++nt;
  double *Kb = R1 + r;  // K = R G in the (dead) B_PN block
  // K <- R - K Y_P from K = R (error y^(nt+1))
  for (int e = tid; e < r * r; e += T) {
    const int i = qdiv(e, invr), j = e - i * r;
    Kb[i * L + j] = Yb[i * ly + j] + (i == j ? lam[i] : 0.0);
  }
  __syncthreads();
  for (int t = 0; t < nt; ++t)
    team_mm1<false, true>(r, r, Opd{Kb, L, 1}, Opd{YPt, ly, 1}, r, [&](int i, int j, double v) {
      Kb[i * L + j] = (Yb[i * ly + j] + (i == j ? lam[i] : 0.0)) - v;
    });
  if (vup) {
    // S_P = (I + Y_P)^-1/2 -> E_PP block, S_N = (I + Y_N)^-1/2 -> EX (Y is
    // dead): binomial series sum_k c_k Y^k, c_k = c_{k-1} (-(2k - 1) / 2k),
    // by Horner in place
    double *SP = R1, *SN = EX;
    const double *YN = R1 + r * L + r;
    double cK = 1.0;
    for (int q = 1; q <= nt; ++q) cK *= -(2.0 * q - 1.0) / (2.0 * q);
    for (int e = tid; e < r * r + n * n; e += T) {
      if (e < r * r) {
        const int i = qdiv(e, invr), j = e - i * r;
        SP[i * L + j] = i == j ? cK : 0.0;
      } else {
        const int q = e - r * r, i = qdiv(q, invn), j = q - i * n;
        SN[i * ln + j] = i == j ? cK : 0.0;
      }
    }
    __syncthreads();
    double c = cK;
    const int nsp = nbr * nbr;
    for (int q = nt - 1; q >= 0; --q) {
      c *= -(2.0 * (q + 1)) / (2.0 * (q + 1) - 1.0);  // c_q from c_{q+1}
      double cc[kSplitMaxB][2][2][2];
#pragma unroll
      for (int s2 = 0; s2 < kSplitMaxB; ++s2) {
        blk16_zero(cc[s2]);
        const int t = w + s2 * nw;
        if (t < nsp) {
          const int bi = qdiv(t, invbr), bj = t - bi * nbr;
          blk16(cc[s2], Opd{YPt, ly, 1}, Opd{SP, L, 1}, bi * 16, bj * 16, r, r, r);
        } else if (t < nsp + nbn * nbn) {
          const int bi = qdiv(t - nsp, invbn), bj = (t - nsp) - bi * nbn;
          blk16(cc[s2], Opd{YN, L, 1}, Opd{SN, ln, 1}, bi * 16, bj * 16, n, n, n);
        }
      }
      __syncthreads();
#pragma unroll
      for (int s2 = 0; s2 < kSplitMaxB; ++s2) {
        const int t = w + s2 * nw;
        if (t < nsp) {
          const int bi = qdiv(t, invbr), bj = t - bi * nbr;
          blk16_each(cc[s2], bi * 16, bj * 16, r, r,
                     [&](int i, int j, double v) { SP[i * L + j] = v + (i == j ? c : 0.0); });
        } else if (t < nsp + nbn * nbn) {
          const int bi = qdiv(t - nsp, invbn), bj = (t - nsp) - bi * nbn;
          blk16_each(cc[s2], bi * 16, bj * 16, n, n,
                     [&](int i, int j, double v) { SN[i * ln + j] = v + (i == j ? c : 0.0); });
        }
      }
      __syncthreads();
    }
  }
  SPLIT_STAMP(5);
  double *Tt = R1 + r * L;  // rows r.. of R1
  const int nbd = (d + 15) >> 4, nut = nbr * nbd, nwt = vup ? nbn * nbd : 0;
  {
    // one pass: Ut = Vt_P + Y_X' Vt_N (r x d) -> R2, and (vup) Wt = Vt_N - Y_X Vt_P
    // (n x d) in place over rows r.. of R1 (staged; Y_X, Y_N are dead after);
    // rows of V gathered through perm
    double cw[kSplitMaxB][2][2][2];
#pragma unroll
    for (int s2 = 0; s2 < kSplitMaxB; ++s2) {
      blk16_zero(cw[s2]);
      const int t = w + s2 * nw;
      if (t < nwt) {
        const int bi = qdiv(t, invbd), bj = t - bi * nbd;
        blk16<true>(cw[s2], XX, Opd{vst, d, 1}, bi * 16, bj * 16, n, d, r, perm);
      }
    }
    for (int t = ((w - nwt) % nw + nw) % nw; t < nut; t += nw) {
      const int bi = qdiv(t, invbd), bj = t - bi * nbd;
      double cu[2][2][2];
      blk16_zero(cu);
      blk16<true>(cu, Opd{R1 + r * L, 1, L}, Opd{vst, d, 1}, bi * 16, bj * 16, r, d, n, perm + r);
      blk16_each(cu, bi * 16, bj * 16, r, d, [&](int i, int j, double v) { Ut[i * L + j] = v + vst[perm[i] * d + j]; });
    }
    __syncthreads();
#pragma unroll
    for (int s2 = 0; s2 < kSplitMaxB; ++s2) {
      const int t = w + s2 * nw;
      if (t < nwt) {
        const int bi = qdiv(t, invbd), bj = t - bi * nbd;
        blk16_each(cw[s2], bi * 16, bj * 16, n, d,
                   [&](int i, int j, double v) { Tt[i * L + j] = vst[perm[r + i] * d + j] - v; });
      }
    }
    __syncthreads();
  }
  if (vup) {
    // V' = [S_P Ut; S_N Wt] -> the store (rows 0..r-1: positive subspace), one pass
    double *vw = W.vstore + off;
    const int nvn = nbn * nbd;
    for (int t = w; t < nut + nvn; t += nw) {
      double cv[2][2][2];
      blk16_zero(cv);
      if (t < nut) {
        const int bi = qdiv(t, invbd), bj = t - bi * nbd;
        blk16(cv, Opd{R1, L, 1}, Opd{Ut, L, 1}, bi * 16, bj * 16, r, d, r);
        blk16_each(cv, bi * 16, bj * 16, r, d, [&](int i, int j, double v) { vw[i * d + j] = v; });
      } else {
        const int bi = qdiv(t - nut, invbd), bj = (t - nut) - bi * nbd;
        blk16(cv, Opd{EX, ln, 1}, Opd{Tt, L, 1}, bi * 16, bj * 16, n, d, n);
        blk16_each(cv, bi * 16, bj * 16, n, d, [&](int i, int j, double v) { vw[(r + i) * d + j] = v; });
      }
    }
    __syncthreads();
  }
  SPLIT_STAMP(6);
  // Tt = K Ut (r x d) -> rows r.. of R1 (Wt is dead)
  team_mm1<false, false>(r, d, Opd{Kb, L, 1}, Opd{Ut, L, 1}, r, [&](int i, int j, double v) { Tt[i * L + j] = v; });
  SPLIT_STAMP(7);
  // P = Ut' Tt  (d x d, symmetric) -> u_s; then w_s = (ws - us_h) + P
  // (solver.py:391-394) in a coalesced pass
  team_mm1<true, false>(d, d, Opd{Ut, 1, L}, Opd{Tt, L, 1}, r, [&](int i, int j, double v) { su[i * d + j] = v; });
  for (int e0 = tid; e0 < d * d; e0 += 4 * T) {  // (batched: the stores may alias later loads)
    double a4[4], b4[4], x4[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = min(e0 + q * T, d * d - 1);
      a4[q] = sw[e];
      b4[q] = su[e];
      x4[q] = neg ? xg[e] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (e0 + q * T < d * d) {
        const double p = neg ? x4[q] + b4[q] : b4[q];  // X+ = X + (-X)+ after a negation
        if (neg) su[e0 + q * T] = p;
        sw[e0 + q * T] = a4[q] + p;
      }
  }
  SPLIT_STAMP(8);
  if (tid == 0 && W.sweeps) W.sweeps[k] = -it;  // (stats: fixed-point iterations)
  // next iteration: the cold path when this basis was already near the bound
  // (off(B) > 0.35 g: the drift of a kept basis grows), else the fast path
  if (tid == 0 && W.cnext && !refreshed) W.cnext[k] = o2 > ca.pol_f2c * g * g ? 1 : 0;
  // schedule key for the next iteration: passes, plus a refresh risk when off(B)
  // is already near the applicability bound
  if (tid == 0) W.ckey[k] = o2 > kSplitKey2 * kSplitOff2 * g * g ? 1 : 0;
  if (refreshed) return SPLIT_DONE + 16;  // (stats: after a Jacobi refresh)
  if (tid == 0 && it > ca.split_refresh) W.vvalid[k] |= kVRefresh;
  return SPLIT_DONE;
}

// (k_cone_split, the kernel around split_one, is in hsde_cold.cuh: its hand-overs run the cold path)
