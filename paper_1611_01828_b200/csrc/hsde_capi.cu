// hsde_capi.cu -- C ABI (include/hsde.h) over the sm_100a kernels.
//
// Host responsibilities: validate and derive the device layout once
// (CSC of A, row segments over owned columns, cover lists, P^{-1},
// normalisation), assemble and factor the m x m Schur matrix
// S = I + A P^{-1} A' on the device (solver.py:248-283: dense column chunks +
// cuBLAS DGEMM, cuSOLVER Cholesky, explicit S^{-1}), solve M zeta with the
// device inner solve, capture the iteration as a CUDA graph, and run the
// residual / certificate reductions.
//
// A handle holds one or more *shards* (shard.py / SURVEY 8(e)).  Shards meet
// at three all-reduce points per iteration (separator pull-scatter partials,
// partial A t, partial c.ua):
//   single GPU     -- one shard, no reduction;
//   NCCL           -- one shard per rank, ncclAllReduce on the handle's stream
//                     (captured in the iteration graph);
//   emulated       -- all shards of one problem on one device, reductions by a
//                     device kernel summing the shard buffers in rank order
//                     (tests the sharded kernels on one GPU without ranks that
//                     wait on each other).

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hsde.h"
#include "hsde_kernels.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

using namespace hsde;

namespace {

std::string g_create_error;

// HSDE_TIMING=1: setup phase times on stderr (device synchronised per phase)
struct SetupTimer {
  bool on = std::getenv("HSDE_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void operator()(const char *what) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hsde setup] %-18s %8.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

enum ProfSlot {
  PS_PREP = 0, PS_RHS, PS_SPMV, PS_SCHUR, PS_UA, PS_SCALARS, PS_CONE_WARP, PS_CONE_BLOCK,
  PS_XUPD, PS_COMM, PS_COUNT
};
const char *kProfNames[HSDE_PROFILE_SLOTS] = {
    "k_prep_ry", "k_rhs", "k_spmv_seg", "k_schur", "k_ua", "k_scalars", "k_cone_warp",
    "k_cone_cta", "k_xupd", "allreduce", "", "", "", "", "", ""};

struct ConePlan {
  int *ids = nullptr;
  int count = 0;
  int dpmax = 0;
  size_t smem = 0;
  int per_block = 0;       // warps per CTA (warp plan)
  bool split_small = false;  // k_cone_split with kSplitThreadsSmall threads (largest clique <= kSplitSmallD)
  double *pscratch = nullptr;  // CTA plan: d x d global scratch per CTA (second-order rebuild)
  int64_t pstride = 0;
  size_t split_smem = 0;       // CTA plan: k_cone_split (0: not launched)
  int cold_cv = 0;             // CTA plan: tridiagonal cold path variant (0: Jacobi)
  size_t cold_smem = 0;
  int *cfail = nullptr;        // [count] cold-path failures (follow-up Jacobi launch)
  int wper_block = 0;          // warp plan, cold path: warps per CTA and shared memory
  size_t wsmem = 0;
};

enum Mode { MODE_SINGLE = 0, MODE_EMULATED = 1, MODE_NCCL = 2 };
enum Buf { BUF_SEP = 0, BUF_Q, BUF_RED, BUF_CHK, BUF_SCHUR, BUF_MINEIG, BUF_COUNT };

__global__ void k_set_i32(int *p, int n, int v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

// sum (or min) the G shard buffers element-wise, result written back to all
__global__ void k_reduce_ptrs(double *const *ptrs, int G, int64_t n, int64_t off, int op_min) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    double s = ptrs[0][off + k];
    for (int g = 1; g < G; ++g) s = op_min ? fmin(s, ptrs[g][off + k]) : s + ptrs[g][off + k];
    for (int g = 0; g < G; ++g) ptrs[g][off + k] = s;
  }
}

}  // namespace

struct ShardDev {
  DevProblem P{};
  DevState S{};
  DevWork W{};
  ConePlan warp_plans[3], block_plan;  // warp teams by size class dp <= 8, 16, 32
  double *d_zeta = nullptr;       // [T-1] (c, 0, -b, 0) normalised
  double *d_prev_u = nullptr, *d_prev_w = nullptr;
  double *d_tmp = nullptr, *d_tmp2 = nullptr, *d_tmp3 = nullptr;  // [T] scratch
  double *d_hv = nullptr;         // [n_c] pull-scatter scratch
  double *d_qseg2 = nullptr;
  double *d_c_orig = nullptr, *d_b_orig = nullptr;
  double *d_consts = nullptr;     // [0] sigma_b [1] sigma_c
  double *d_chk = nullptr;        // [64] check sums
  double *d_mineig = nullptr;     // [p]
  double *d_schur = nullptr;      // [m*m] partial / factored Schur (owned)
  int grid_heavy = 0, grid_nc = 1, grid_nd = 1, grid_m = 1, grid_T = 1, grid_seg = 1, grid_schur = 1;
  int grid_ua = 1;  // k_ua / k_ua_half grid = number of c.ua block partials
  int grid_rhs = 1, grid_xupd = 1;  // light CTAs of k_rhs; k_xupd grid (no partials)
  size_t schur_smem = 0;
  std::vector<int> sizes;         // clique sizes (host copy)
  std::vector<char> in_block;     // clique runs on a CTA team (block plan)
  int64_t maxcol = 0;
  double nc2_owned = 0;           // sum of c^2 over owned coordinates (original units)
};

struct hsde_handle {
  int dev = 0;
  int n_sm = 148;  // multiprocessors of the device
  cudaStream_t st = nullptr;
  // parallel branches for the independent cone launches (size classes, shards)
  static constexpr int kAux = 4;
  cudaStream_t aux[kAux] = {};
  cudaEvent_t ev_fork = nullptr, ev_xjoin = nullptr, ev_join[kAux] = {};
  hsde_settings set{};
  hsde_info_t info{};
  std::vector<void *> bufs;
  std::string err;
  std::vector<ShardDev> sh;
  int mode = MODE_SINGLE;
  ncclComm_t nccl = nullptr;
  int world = 1, rank = 0;
  double **d_ptrs[BUF_COUNT] = {};  // emulation pointer tables
  double *h_chk = nullptr;          // pinned [64]
  double norm_b = 0, norm_c = 0;    // of the iterated (normalised) data
  int n_sep = 0;
  bool schur_diag = false;
  cudaGraphExec_t g1 = nullptr, gci = nullptr;
  int gci_len = 0;
  bool factor = true;
  bool warm = true;
  bool split = true;  // k_cone_split fast path for CTA cliques (HSDE_FLAG_NO_SPLIT off)
  bool jacobi = false;  // HSDE_FLAG_JACOBI: no tridiagonal cold path
  bool multi() const { return mode != MODE_SINGLE; }
};

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      h->err = std::string(#call) + ": " + cudaGetErrorString(e_);                    \
      return HSDE_ERR_CUDA;                                                           \
    }                                                                                 \
  } while (0)

#define CKL()                                                                         \
  do {                                                                                \
    cudaError_t e_ = cudaGetLastError();                                              \
    if (e_ != cudaSuccess) {                                                          \
      h->err = std::string("launch: ") + cudaGetErrorString(e_) + " @" + std::to_string(__LINE__); \
      return HSDE_ERR_CUDA;                                                           \
    }                                                                                 \
  } while (0)

#define RC(x)            \
  do {                   \
    int rc_ = (x);       \
    if (rc_) return rc_; \
  } while (0)

namespace {

// Device memory comes from the device's stream-ordered pool, which keeps
// freed blocks (release threshold raised once): a second solve in the same
// process reuses the first one's memory instead of mapping new pages.
void retain_pool(int dev) {
  static bool done[64] = {};
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

// Pinned host slots for the check results.  cudaMallocHost / cudaFreeHost per
// handle cost 10-450 ms sporadically (measured: one solve in ~6 paid it in
// hsde_destroy or hsde_create); handles take 64-double slots from process-wide
// pinned slabs instead (portable, grown 32 slots at a time, never freed).
std::mutex g_pin_mu;
std::vector<double *> g_pin_free;

double *pinned_slot_acquire() {
  std::lock_guard<std::mutex> lock(g_pin_mu);
  if (g_pin_free.empty()) {
    double *slab = nullptr;
    if (cudaHostAlloc((void **)&slab, 32 * 64 * sizeof(double), cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    for (int i = 0; i < 32; ++i) g_pin_free.push_back(slab + 64 * i);
  }
  double *p = g_pin_free.back();
  g_pin_free.pop_back();
  return p;
}

void pinned_slot_release(double *p) {
  if (!p) return;
  std::lock_guard<std::mutex> lock(g_pin_mu);
  g_pin_free.push_back(p);
}

// pool allocation usable from any stream on return
cudaError_t pool_malloc(hsde_handle *h, void **p, size_t bytes) {
  cudaError_t e = cudaMallocAsync(p, std::max<size_t>(bytes, 1), h->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->st);
  return e;
}

void pool_free(hsde_handle *h, void *p) {
  if (p) cudaFreeAsync(p, h->st);
}

template <class T>
int dalloc(hsde_handle *h, T **p, size_t n) {
  void *q = nullptr;
  cudaError_t e = pool_malloc(h, &q, std::max<size_t>(n, 1) * sizeof(T));
  if (e != cudaSuccess) {
    h->err = std::string("cudaMallocAsync: ") + cudaGetErrorString(e);
    return HSDE_ERR_CUDA;
  }
  h->bufs.push_back(q);
  *p = static_cast<T *>(q);
  return 0;
}

// Large host->device copies from pageable memory (the caller's arrays: A
// alone is 0.46 GB for config 4) go through two pinned staging buffers: the
// host copy of a chunk is split over threads while the DMA engine moves the
// previous chunk (pageable cudaMemcpy runs at ~11 GB/s on this host).
constexpr size_t kStagedMin = 16u << 20;
constexpr size_t kStageChunk = 32u << 20;

// (staging state per device: the copy stream and events belong to the device
// that was current when they were created)
struct StageState {
  char *pin[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  cudaStream_t cs = nullptr;
};

int h2d_staged(hsde_handle *h, void *dst, const void *src, size_t bytes) {
  static std::mutex mu;
  static StageState states[64];
  std::lock_guard<std::mutex> lock(mu);
  StageState &S = states[(h->dev >= 0 && h->dev < 64) ? h->dev : 0];
  char **pin = S.pin;
  cudaEvent_t *done = S.done;
  if (!pin[0]) {
    for (int b = 0; b < 2; ++b)
      if (cudaHostAlloc((void **)&pin[b], kStageChunk, cudaHostAllocDefault) != cudaSuccess ||
          cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming) != cudaSuccess) {
        pin[0] = pin[1] = nullptr;
        cudaGetLastError();
        cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);  // no pinned memory
        if (e != cudaSuccess) {
          h->err = std::string("cudaMemcpy H2D: ") + cudaGetErrorString(e);
          return HSDE_ERR_CUDA;
        }
        return 0;
      }
    CK(cudaStreamCreateWithFlags(&S.cs, cudaStreamNonBlocking));
  }
  cudaStream_t cs = S.cs;
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const char *s8 = static_cast<const char *>(src);
  char *d8 = static_cast<char *>(dst);
  bool used[2] = {false, false};
  for (size_t off = 0, c = 0; off < bytes; off += kStageChunk, ++c) {
    const int b = (int)(c & 1);
    const size_t len = std::min(kStageChunk, bytes - off);
    if (used[b]) CK(cudaEventSynchronize(done[b]));  // its previous DMA has finished
    const size_t per = (len + hw - 1) / hw;
    std::vector<std::thread> th;
    for (unsigned t = 1; t < hw && t * per < len; ++t)
      th.emplace_back([=] { std::memcpy(pin[b] + t * per, s8 + off + t * per, std::min(per, len - t * per)); });
    std::memcpy(pin[b], s8 + off, std::min(per, len));
    for (auto &x : th) x.join();
    CK(cudaMemcpyAsync(d8 + off, pin[b], len, cudaMemcpyHostToDevice, cs));
    CK(cudaEventRecord(done[b], cs));
    used[b] = true;
  }
  CK(cudaStreamSynchronize(cs));
  return 0;
}

template <class T>
int dcopy(hsde_handle *h, T *dst, const T *src, size_t n) {
  if (n * sizeof(T) >= kStagedMin) return h2d_staged(h, dst, src, n * sizeof(T));
  if (n) {
    cudaError_t e = cudaMemcpy(dst, src, n * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      h->err = std::string("cudaMemcpy H2D: ") + cudaGetErrorString(e);
      return HSDE_ERR_CUDA;
    }
  }
  return 0;
}

template <class T>
int dupload(hsde_handle *h, T **p, const T *src, size_t n) {
  RC(dalloc(h, p, n));
  return dcopy(h, *p, src, n);
}

int grid_for(int64_t n, int cap = 148 * 8) {
  int64_t g = (n + kBlock - 1) / kBlock;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// Kernel launch with (pdl) programmatic stream serialisation: the kernel may be
// scheduled while the previous kernel of the stream drains; it calls pdl_wait()
// before touching anything (hsde_kernels.cuh).  Captured into the iteration graphs
// as programmatic dependency edges.
template <class... KArgs, class... Args>
cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, KArgs(std::forward<Args>(args))...);
}

double *buf_ptr(ShardDev &s, int which) {
  switch (which) {
    case BUF_SEP: return s.W.sepbuf;
    case BUF_Q: return s.W.qbuf;
    case BUF_RED: return s.W.red;
    case BUF_CHK: return s.d_chk;
    case BUF_SCHUR: return s.d_schur;
    default: return s.d_mineig;
  }
}

// All-reduce `n` doubles of buffer `which` (+offset) across shards / ranks.
int reduce(hsde_handle *h, int which, int64_t n, int64_t off = 0, bool op_min = false) {
  if (!h->multi() || n <= 0) return 0;
  if (h->mode == MODE_NCCL) {
    double *b = buf_ptr(h->sh[0], which) + off;
    ncclResult_t r = ncclAllReduce(b, b, (size_t)n, ncclDouble, op_min ? ncclMin : ncclSum, h->nccl, h->st);
    if (r != ncclSuccess) {
      h->err = std::string("ncclAllReduce: ") + ncclGetErrorString(r);
      return HSDE_ERR_CUDA;
    }
    return 0;
  }
  const int G = (int)h->sh.size();
  k_reduce_ptrs<<<grid_for(n), kBlock, 0, h->st>>>(h->d_ptrs[which], G, n, off, op_min ? 1 : 0);
  CKL();
  return 0;
}

// densify owned columns [c0, c1) of A (CSC) into Dm (m x w, col-major) and Ds = Dm diag(p_inv)
__global__ void k_densify(DevProblem P, int c0, int c1, double *Dm, double *Ds) {
  const int64_t w = c1 - c0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < w;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int l = c0 + (int)k;
    if (!owns(P, l)) continue;
    for (int64_t e = P.at_cp[l]; e < P.at_cp[l + 1]; ++e) {
      const int i = P.at_row[e];
      Dm[i + k * P.m] = P.at_val[e];
      Ds[i + k * P.m] = P.at_val[e] * P.p_inv[l];  // A.multiply(p_inv) (solver.py:251)
    }
  }
}

__global__ void k_add_identity(double *S, int m) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    S[i + (int64_t)i * m] += 1.0;  // solver.py:253
}

__global__ void k_identity(double *X, int m) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (int64_t)m * m;
       k += (int64_t)gridDim.x * blockDim.x)
    X[k] = (k % m == k / m) ? 1.0 : 0.0;
}

__global__ void k_symmetrize(const double *X, int m, double *out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (int64_t)m * m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / m, j = k % m;
    out[k] = 0.5 * (X[i * m + j] + X[j * m + i]);
  }
}

__global__ void k_finite_check(const double *x, int64_t n, int *flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[k])) atomicOr(flag, 1);
}

// S_ii partial = sum over owned columns of (A_il p_l) A_il (diagonal case)
__global__ void k_diag_schur(DevProblem P, double *diag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = P.a_rp[i]; k < P.a_rp[i + 1]; ++k)
      s += (P.a_val[k] * P.p_inv[P.a_col[k]]) * P.a_val[k];
    diag[i] = s;
  }
}

__global__ void k_diag_finish(double *diag, int m, int *flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const double s = diag[i] + 1.0;
    if (!(s > 0.0) || !isfinite(s)) atomicOr(flag, 1);
    diag[i] = 1.0 / s;
  }
}

// cone launches (one shard)
// part (CTA plan with the fast path and the cold path): 0 everything,
// serially; 1 the fast path; 2 the cold path on the predicted cliques
// (W.ccur, set by k_scalars; 1 and 2 run concurrently on disjoint cliques);
// 3 the cold path on the fast path's hand-overs, then the Jacobi fallback
// (after 1 and 2)
int launch_cone(hsde_handle *h, ShardDev &s, int mode, const ConePlan &pl, bool block,
                const double *in, double *out, double in_scale, cudaStream_t st, int part = 0) {
  if (pl.count == 0) return 0;
  static const int split_refresh = [] {
    const char *e = std::getenv("HSDE_SPLIT_REFRESH");
    return e ? std::atoi(e) : kSplitRefreshIters;
  }();
  static const int split_vupdate = [] {
    const char *e = std::getenv("HSDE_SPLIT_VUPDATE");
    return e ? std::atoi(e) : 1;
  }();
  static const int split_prefetch = [] {
    // L2 prefetch of the second wave's inputs by the first wave (hsde_split.cuh):
    // ~1% faster on config 4 but +18% DRAM traffic (lines evicted before use): off
    const char *e = std::getenv("HSDE_SPLIT_PREFETCH");
    return e ? std::atoi(e) : 0;
  }();
  ConeArgs ca{pl.ids, pl.count, pl.dpmax, in, out, in_scale, h->warm ? 1 : 0, pl.pscratch, pl.pstride, 0,
              split_refresh, split_vupdate};
  // cold / warm policy thresholds (hsde_split.cuh, hsde_cold.cuh)
  static const double pol_f2c = [] {
    const char *e = std::getenv("HSDE_POL_F2C");
    return e ? std::atof(e) : 0.1225;
  }();
  static const double pol_c2f = [] {
    const char *e = std::getenv("HSDE_POL_C2F");
    return e ? std::atof(e) : 0.36;
  }();
  ca.pol_f2c = pol_f2c;
  ca.pol_c2f = pol_c2f;
  if (!block) {
    const int grid = (pl.count + pl.per_block - 1) / pl.per_block;
    const int thr = pl.per_block * 32;
    if (!h->jacobi && pl.cfail && mode != CONE_HOT) {
      // warp cold path (hsde_cold.cuh), then its failures on the warp Jacobi
      // path.  (Not on the hot path: warm-started warp Jacobi is faster there,
      // e.g. config 1: 33 vs 77 us per projection; measured, tools/small_profile.py)
      ca.cfail = pl.cfail;
      const int wg = (pl.count + pl.wper_block - 1) / pl.wper_block;
      const int wt = pl.wper_block * 32;
      if (mode == CONE_HOT) k_cone_wcold<CONE_HOT><<<wg, wt, pl.wsmem, st>>>(s.P, s.S, s.W, ca);
      else if (mode == CONE_PLAIN) k_cone_wcold<CONE_PLAIN><<<wg, wt, pl.wsmem, st>>>(s.P, s.S, s.W, ca);
      else k_cone_wcold<CONE_MINEIG><<<wg, wt, pl.wsmem, st>>>(s.P, s.S, s.W, ca);
      CKL();
      ca.fail_only = 1;
    }
    if (mode == CONE_HOT) k_cone_warp<CONE_HOT><<<grid, thr, pl.smem, st>>>(s.P, s.S, s.W, ca);
    else if (mode == CONE_PLAIN) k_cone_warp<CONE_PLAIN><<<grid, thr, pl.smem, st>>>(s.P, s.S, s.W, ca);
    else k_cone_warp<CONE_MINEIG><<<grid, thr, pl.smem, st>>>(s.P, s.S, s.W, ca);
    CKL();
    return 0;
  }
  DevWork W = s.W;
  W.cstate = nullptr;  // k_cone_block does every clique (of its list)
  const int cv = h->jacobi ? 0 : pl.cold_cv;
  ca.cfail = pl.cfail;
  const bool split = mode == CONE_HOT && pl.split_smem && h->warm && h->split;
  auto cold = [&](const DevWork &Wc, const ConeArgs &a) {
    auto go = [&](auto kern) { kern<<<pl.count, kColdThreads, pl.cold_smem, st>>>(s.P, s.S, Wc, a); };
    if (mode == CONE_HOT) {
      if (cv == 1) go(k_cone_cold<CONE_HOT, 20, 3, 3>);
      else go(k_cone_cold<CONE_HOT, 24, 3, 2>);
    } else if (mode == CONE_PLAIN) {
      if (cv == 1) go(k_cone_cold<CONE_PLAIN, 20, 3, 3>);
      else go(k_cone_cold<CONE_PLAIN, 24, 3, 2>);
    } else {
      if (cv == 1) go(k_cone_cold<CONE_MINEIG, 20, 3, 3>);
      else go(k_cone_cold<CONE_MINEIG, 24, 3, 2>);
    }
    return cudaGetLastError();
  };
  if (split) {
    if (!cv) {  // (Jacobi variant) every clique, hand-overs on the Jacobi path in the same CTA
      ConeArgs co = ca;
      co.ids = s.W.corder;
      DevWork Ws = s.W;
      Ws.ccur = Ws.cnext = nullptr;
      k_cone_split<false><<<pl.count, kSplitThreads, pl.split_smem, st>>>(s.P, s.S, Ws, co);
      CKL();
      return 0;
    }
    if (part == 0 || part == 1) {  // fast path (hsde_split.cuh), scheduled by k_scalars
      ConeArgs co = ca;
      co.ids = s.W.corder;
      co.pf_ahead = split_prefetch ? 2 * h->n_sm : 0;  // two CTAs per SM resident
      if (pl.split_small) k_cone_split<true, kSplitThreadsSmall><<<pl.count, kSplitThreadsSmall, pl.split_smem, st>>>(s.P, s.S, s.W, co);
      else k_cone_split<true><<<pl.count, kSplitThreads, pl.split_smem, st>>>(s.P, s.S, s.W, co);
      CKL();
    }
    if (part == 0 || part == 2) {  // cold path on the predicted cliques
      ConeArgs c0 = ca;
      c0.cold_pass = 0;
      if (cold(s.W, c0) != cudaSuccess) CKL();
    }
    if (part == 0 || part == 3) {  // cold path on the hand-overs, then the fallback
      ConeArgs c1 = ca;
      c1.cold_pass = 1;
      if (cold(s.W, c1) != cudaSuccess) CKL();
      ca.fail_only = 1;
    } else {
      return 0;
    }
  } else if (cv && !(mode == CONE_HOT && !h->split)) {
    // tridiagonal cold path on every clique, then its failures on the Jacobi path
    DevWork Wc = s.W;
    Wc.ccur = Wc.cnext = Wc.cstate = nullptr;
    if (cold(Wc, ca) != cudaSuccess) CKL();
    ca.fail_only = 1;
  }
  if (mode == CONE_HOT) k_cone_block<CONE_HOT><<<pl.count, kConeBlock, pl.smem, st>>>(s.P, s.S, W, ca);
  else if (mode == CONE_PLAIN) k_cone_block<CONE_PLAIN><<<pl.count, kConeBlock, pl.smem, st>>>(s.P, s.S, W, ca);
  else k_cone_block<CONE_MINEIG><<<pl.count, kConeBlock, pl.smem, st>>>(s.P, s.S, W, ca);
  CKL();
  return 0;
}

// ordered dot of two device vectors into out (device scalar)
int dev_dot(hsde_handle *h, ShardDev &s, const double *a, const double *b, int64_t n, double *out) {
  const int g = grid_for(n);
  k_dot_part<<<g, kBlock, 0, h->st>>>(a, b, n, s.W.part);
  CKL();
  k_sum_parts<<<1, 1024, 0, h->st>>>(s.W.part, g, out);
  CKL();
  return 0;
}

int dev_dot_owned(hsde_handle *h, ShardDev &s, const double *a, const double *b, double *out) {
  k_dot_owned_part<<<s.grid_nc, kBlock, 0, h->st>>>(s.P, a, b, s.W.part);
  CKL();
  k_sum_parts<<<1, 1024, 0, h->st>>>(s.W.part, s.grid_nc, out);
  CKL();
  return 0;
}

// q0 = A t0 of one shard: tile partials + ordered row sums into W.qbuf (half
// passes), or row-segment partials in W.qseg (+ W.qbuf when sharded)
int launch_aq(hsde_handle *h, ShardDev &s, cudaStream_t st, int *nl, bool pdl = false) {
  const DevProblem &P = s.P;
  if (P.half) {
    // (forming the pair sums while staging each tile instead measured 24 us
    // slower: the gathers sit at the start of every CTA, 4x redundant)
    CK(launch_k(pdl, k_pair_sum, grid_for(P.n_pair), kBlock, 0, st, P, s.W.t, s.W.xq));
    CK(launch_k(pdl, k_spmv_half<false>, P.rt_ntile * P.rt_split, kBlock, sizeof(double) * P.rt_tile, st, P,
                s.W.xq, s.W.rtpart));
    CK(launch_k(pdl, k_rowsum_tiles, grid_for((int64_t)P.m * 32), kBlock, 0, st, P, s.W.rtpart, s.W.qbuf));
    *nl += 3;
    return 0;
  }
  k_spmv_seg<<<s.grid_seg, kBlock, 0, st>>>(P, s.W.t, s.W.qseg);
  CKL();
  ++*nl;
  if (h->multi()) {
    k_rowsum_seg<<<s.grid_m, kBlock, 0, st>>>(P, s.W.qseg, s.W.qbuf);
    CKL();
    ++*nl;
  }
  return 0;
}

// k_schur reads the reduced q0 from W.qbuf unless it sums row segments itself
bool q_in_buf(const hsde_handle *h, const ShardDev &s) { return s.P.half || h->multi(); }

// ua = t0 - P^{-1} A' g (+ block partials of c.ua)
int launch_ua(hsde_handle *h, ShardDev &s, cudaStream_t st, bool with_dot, bool pdl = false) {
  const DevProblem &P = s.P;
  if (P.half) {
    const size_t sm = sizeof(double) * (size_t)P.m;
    if (with_dot) CK(launch_k(pdl, k_ua_half<true>, s.grid_ua, kBlock, sm, st, P, s.W, s.W.qp));
    else CK(launch_k(pdl, k_ua_half<false>, s.grid_ua, kBlock, sm, st, P, s.W, s.W.qp));
  } else {
    if (with_dot) k_ua<true><<<s.grid_ua, kBlock, 0, st>>>(P, s.W, s.W.qp);
    else k_ua<false><<<s.grid_ua, kBlock, 0, st>>>(P, s.W, s.W.qp);
  }
  CKL();
  return 0;
}

// The inner solve of _solve_inner_parts (solver.py:203-245) on explicit
// vectors, all shards: rho (T-1 per shard, x|s|y|v) -> u12.  uy by the
// identity A ua = S^{-1} A t, or (exact_uy, single shard) the explicit CSR
// pass uy = wy - A ua of solver.py:240-241.
int inner_dist(hsde_handle *h, const std::vector<const double *> &rho,
               const std::vector<double *> &u12, bool exact_uy) {
  cudaStream_t st = h->st;
  const int G = (int)h->sh.size();
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    const DevProblem &P = s.P;
    const double *rx = rho[g], *rs = rho[g] + P.n_c, *ry = rho[g] + P.n_c + P.n_d,
                 *rv = rho[g] + P.n_c + P.n_d + P.m;
    if (h->n_sep) {
      k_zero<<<grid_for(h->n_sep), kBlock, 0, st>>>(s.W.sepbuf, h->n_sep);
      CKL();
    }
    k_rhs<false><<<s.grid_rhs + s.grid_heavy, kBlock, 0, st>>>(P, s.S, s.W, rx, rs, rv, s.grid_heavy);
    CKL();
  }
  RC(reduce(h, BUF_SEP, h->n_sep));
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    const DevProblem &P = s.P;
    const double *rx = rho[g];
    if (P.n_sep_local) {
      k_sep_finish<false><<<grid_for(P.n_sep_local), kBlock, 0, st>>>(P, s.S, s.W, rx);
      CKL();
    }
    int nl = 0;
    RC(launch_aq(h, s, st, &nl));
  }
  RC(reduce(h, BUF_Q, h->sh[0].P.m));
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    const DevProblem &P = s.P;
    const double *rs = rho[g] + P.n_c, *ry = rho[g] + P.n_c + P.n_d, *rv = ry + P.m;
    k_schur<<<s.grid_schur, kBlock, s.schur_smem, st>>>(P, s.W.qseg, q_in_buf(h, s) ? s.W.qbuf : nullptr,
                                                        ry, s.W.qp);
    CKL();
    RC(launch_ua(h, s, st, false));
    double *ua = u12[g], *ub = u12[g] + P.n_c, *uy = u12[g] + P.n_c + P.n_d, *uv = uy + P.m;
    CK(cudaMemcpyAsync(ua, s.W.ua, sizeof(double) * P.n_c, cudaMemcpyDeviceToDevice, st));
    k_slot_out<<<s.grid_nd, kBlock, 0, st>>>(P, rs, rv, ua, ub, uv);
    CKL();
    if (exact_uy) {
      k_spmv_seg<<<s.grid_seg, kBlock, 0, st>>>(P, ua, s.d_qseg2);
      CKL();
      k_uy_from_seg<<<s.grid_m, kBlock, 0, st>>>(P, s.d_qseg2, nullptr, ry, uy);
      CKL();
    } else {
      k_uy_from_seg<<<s.grid_m, kBlock, 0, st>>>(P, nullptr, s.W.qp, ry, uy);  // uy = -g
      CKL();
    }
  }
  return 0;
}

// one hot iteration (solver.py:375-395) over all shards, eager launches;
// profiling events optional (phases summed over shards)
int launch_iteration(hsde_handle *h, cudaEvent_t *ev = nullptr, int *launches = nullptr) {
  cudaStream_t st = h->st;
  const int G = (int)h->sh.size();
  const bool exact = (h->set.flags & HSDE_FLAG_EXACT_UY) != 0 && !h->multi();
  // programmatic dependent launches along the affine chain (one shard, half
  // passes, no all-reduce or event in between; not under the per-kernel profile)
  static const int pdl_env = [] {
    const char *e = std::getenv("HSDE_PDL");
    return e ? std::atoi(e) : 1;
  }();
  const bool pdl = pdl_env && !ev && G == 1 && !h->multi() && h->sh[0].P.half && !exact && h->n_sep == 0;
  int nl = 0;
  auto mark = [&](int s) {
    if (ev) cudaEventRecord(ev[s], st);
  };
  mark(PS_COUNT);
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    if (h->n_sep) {
      k_zero<<<grid_for(h->n_sep), kBlock, 0, st>>>(s.W.sepbuf, h->n_sep);
      CKL();
      ++nl;
    }
    k_rhs<true><<<s.grid_rhs + s.grid_heavy, kBlock, 0, st>>>(s.P, s.S, s.W, nullptr, nullptr, nullptr,
                                                            s.grid_heavy);
    CKL();
    ++nl;
  }
  mark(PS_RHS);
  RC(reduce(h, BUF_SEP, h->n_sep));
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    if (s.P.n_sep_local) {
      k_sep_finish<true><<<grid_for(s.P.n_sep_local), kBlock, 0, st>>>(s.P, s.S, s.W, nullptr);
      CKL();
      ++nl;
    }
    RC(launch_aq(h, s, st, &nl, pdl));
  }
  mark(PS_SPMV);
  RC(reduce(h, BUF_Q, h->sh[0].P.m));
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    CK(launch_k(pdl, k_schur, s.grid_schur, kBlock, s.schur_smem, st, s.P, s.W.qseg,
                q_in_buf(h, s) ? s.W.qbuf : nullptr, s.W.ry, s.W.qp));
    ++nl;
  }
  mark(PS_SCHUR);
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    RC(launch_ua(h, s, st, true, pdl));
    ++nl;
    if (h->multi()) {
      k_sum_parts<<<1, 1024, 0, st>>>(s.W.part, s.grid_ua, s.W.red);
      CKL();
      ++nl;
    }
    if (exact) {
      // uy = rho_y - A ua by an explicit CSR pass (solver.py:240-241)
      k_spmv_seg<<<s.grid_seg, kBlock, 0, st>>>(s.P, s.W.ua, s.d_qseg2);
      CKL();
      k_rowsum_seg<<<s.grid_m, kBlock, 0, st>>>(s.P, s.d_qseg2, s.d_tmp3);
      CKL();
      nl += 2;
    }
  }
  mark(PS_UA);
  RC(reduce(h, BUF_RED, 1));
  mark(PS_COMM);
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    CK(launch_k(pdl, k_scalars, 1, 1024, 0, st, s.P, s.S, s.W, s.grid_ua, exact ? 1 : 0, s.d_tmp3,
                h->multi() ? s.W.red : nullptr));
    ++nl;
  }
  mark(PS_SCALARS);
  // cone projections: the plans (size classes, shards) are independent, so
  // they run as parallel branches (fork / join on events; captured as graph
  // edges) -- except under the per-phase profile, which keeps them in order
  // The x update (k_xupd) touches only the x segment, the cones only s / v:
  // under graph capture it is one more parallel branch.
  struct ConeJob {
    ShardDev *s;
    const ConePlan *pl;
    bool block;
    int part;
  };
  std::vector<ConeJob> jobs;
  std::vector<int> tails;  // shards whose CTA plan needs the hand-over pass after the join
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    for (const ConePlan &wp : s.warp_plans)
      if (wp.count) jobs.push_back({&s, &wp, false, 0});
  }
  const size_t n_warp_jobs = jobs.size();
  for (int g = 0; g < G; ++g) {
    const ConePlan &bp = h->sh[g].block_plan;
    if (!bp.count) continue;
    const bool two = bp.split_smem && h->warm && h->split && bp.cold_cv && !h->jacobi;
    if (two && !ev) {  // fast path and cold path on disjoint cliques, concurrently (part 3 after the join)
      jobs.push_back({&h->sh[g], &bp, true, 2});
      jobs.push_back({&h->sh[g], &bp, true, 1});
      tails.push_back(g);
    } else {
      jobs.push_back({&h->sh[g], &bp, true, 0});
    }
  }
  nl += (int)jobs.size();
  auto launch_xupd = [&](cudaStream_t xs) -> int {
    for (int g = 0; g < G; ++g) {
      ShardDev &s = h->sh[g];
      k_xupd<<<s.grid_xupd, kBlock, 0, xs>>>(s.P, s.S, s.W);
      CKL();
      ++nl;
    }
    return 0;
  };
  const bool branch_x = !ev && !jobs.empty();
  if (branch_x) {
    // fork: k_xupd on its own branch, the cone jobs as below
    CK(cudaEventRecord(h->ev_fork, st));
    cudaStream_t xs = h->aux[hsde_handle::kAux - 1];
    CK(cudaStreamWaitEvent(xs, h->ev_fork, 0));
    RC(launch_xupd(xs));
    CK(cudaEventRecord(h->ev_xjoin, xs));
  }
  if (ev || jobs.size() <= 1) {
    if (n_warp_jobs == 0) mark(PS_CONE_WARP);
    for (size_t j = 0; j < jobs.size(); ++j) {
      RC(launch_cone(h, *jobs[j].s, CONE_HOT, *jobs[j].pl, jobs[j].block, nullptr, nullptr, 1.0, st, jobs[j].part));
      if (j + 1 == n_warp_jobs) mark(PS_CONE_WARP);
    }
  } else {
    CK(cudaEventRecord(h->ev_fork, st));
    // the largest job (CTA plan if any, else the last warp class) stays on st
    for (size_t j = 0; j + 1 < jobs.size(); ++j) {
      cudaStream_t a = h->aux[j % (hsde_handle::kAux - 1)];
      CK(cudaStreamWaitEvent(a, h->ev_fork, 0));
      RC(launch_cone(h, *jobs[j].s, CONE_HOT, *jobs[j].pl, jobs[j].block, nullptr, nullptr, 1.0, a, jobs[j].part));
    }
    RC(launch_cone(h, *jobs.back().s, CONE_HOT, *jobs.back().pl, jobs.back().block, nullptr, nullptr, 1.0,
                   st, jobs.back().part));
    for (size_t j = 0; j + 1 < jobs.size() && j < (size_t)hsde_handle::kAux - 1; ++j) {
      CK(cudaEventRecord(h->ev_join[j], h->aux[j]));
      CK(cudaStreamWaitEvent(st, h->ev_join[j], 0));
    }
    mark(PS_CONE_WARP);
  }
  for (int g : tails)
    RC(launch_cone(h, h->sh[g], CONE_HOT, h->sh[g].block_plan, true, nullptr, nullptr, 1.0, st, 3));
  nl += 2 * (int)tails.size();
  mark(PS_CONE_BLOCK);
  if (branch_x) CK(cudaStreamWaitEvent(st, h->ev_xjoin, 0));
  else RC(launch_xupd(st));
  mark(PS_XUPD);
  if (launches) *launches += nl;
  return 0;
}

int build_graph(hsde_handle *h, int iters, cudaGraphExec_t *out) {
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
  int rc = 0;
  for (int i = 0; i < iters && !rc; ++i) rc = launch_iteration(h);
  cudaError_t e = cudaStreamEndCapture(h->st, &g);
  if (rc) return rc;
  if (e != cudaSuccess) {
    h->err = std::string("capture: ") + cudaGetErrorString(e);
    return HSDE_ERR_CUDA;
  }
  e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    h->err = std::string("graph instantiate: ") + cudaGetErrorString(e);
    return HSDE_ERR_CUDA;
  }
  return 0;
}

int rebuild_graphs(hsde_handle *h) {
  if (h->g1) cudaGraphExecDestroy(h->g1);
  if (h->gci) cudaGraphExecDestroy(h->gci);
  h->g1 = h->gci = nullptr;
  RC(build_graph(h, 1, &h->g1));
  if (h->gci_len > 1) RC(build_graph(h, h->gci_len, &h->gci));
  return 0;
}

int check_err_flag(hsde_handle *h) {
  int any = 0;
  for (auto &s : h->sh) {
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, s.W.err, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (flag) {
      CK(cudaMemsetAsync(s.W.err, 0, sizeof(int), h->st));
      any = 1;
    }
  }
  if (any) {
    h->err = "batched eigendecomposition produced non-finite eigenvalues";
    return HSDE_ERR_EIGEN;
  }
  return 0;
}

int setup_cone_plans(hsde_handle *h, ShardDev &s, const int32_t *sizes, int p) {
  // warp teams in three size classes (scratch sized per class), CTA teams
  std::vector<int> wids[3], bids;
  const int wcap[3] = {8, 16, 32};
  int dpb = 2;
  // A size class with few cliques (CTA teams stay below two per SM) goes to CTA
  // teams, largest class first, down to order 8: the fast / cold paths cut the
  // projection latency that a single warp cannot hide (config 0: 20 cliques of
  // order 20; config 3: its 16 cliques of order 17-29 took 245 us as warp teams
  // and bounded the whole iteration)
  int ncls[4] = {0, 0, 0, 0};  // orders 8 (exactly), 9-16, 17-32, > 32
  auto cls_of = [](int d) { return d > 32 ? 3 : d > 16 ? 2 : d > 8 ? 1 : d == 8 ? 0 : -1; };
  for (int k = 0; k < p; ++k)
    if (cls_of(sizes[k]) >= 0) ++ncls[cls_of(sizes[k])];
  bool cta_cls[4] = {false, false, false, true};
  for (int c = 2, n_cta = ncls[3]; c >= 0; --c) {
    if (ncls[c] == 0) continue;
    if (n_cta + ncls[c] > 2 * h->n_sm) break;
    cta_cls[c] = true;
    n_cta += ncls[c];
  }
  for (int k = 0; k < p; ++k) {
    const int d = sizes[k];
    const int dp = d + (d & 1);
    const int c = cls_of(d);
    if (c < 0 || !cta_cls[c]) {
      wids[dp <= 8 ? 0 : dp <= 16 ? 1 : 2].push_back(k);
    } else {
      bids.push_back(k);
      dpb = std::max(dpb, dp);
    }
  }
  s.in_block.assign(std::max(p, 1), 0);
  for (int k : bids) s.in_block[k] = 1;
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev);
  if (maxsm <= 0) maxsm = 227 * 1024;
  for (int c = 0; c < 3; ++c) {
    ConePlan &pl = s.warp_plans[c];
    pl.count = (int)wids[c].size();
    pl.dpmax = wcap[c];
    const size_t per_warp = (size_t)jacobi_scratch_doubles(wcap[c]) * sizeof(double);
    int pb = 8;
    while (pb > 1 && per_warp * pb > (size_t)maxsm) pb >>= 1;
    pl.per_block = pb;
    pl.smem = per_warp * pb;
    if (!wids[c].empty()) RC(dupload(h, &pl.ids, wids[c].data(), wids[c].size()));
    // warp cold path: 8 warps per CTA for the small classes, 4 for d <= 32
    pl.wper_block = wcap[c] <= 16 ? 8 : 4;
    pl.wsmem = (size_t)wcold_scratch_doubles(wcap[c]) * sizeof(double) * pl.wper_block;
    if (!wids[c].empty()) {
      RC(dalloc(h, &pl.cfail, wids[c].size()));
      CK(cudaMemset(pl.cfail, 0, sizeof(int) * wids[c].size()));
    }
  }
  {
    const int sm = maxsm;  // attribute is per kernel, shared by every shard / handle
    CK(cudaFuncSetAttribute(k_cone_warp<CONE_HOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute(k_cone_warp<CONE_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute(k_cone_warp<CONE_MINEIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute(k_cone_wcold<CONE_HOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute(k_cone_wcold<CONE_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute(k_cone_wcold<CONE_MINEIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  }
  s.block_plan.count = (int)bids.size();
  s.block_plan.dpmax = dpb;
  const size_t per_blk = (size_t)jacobi_scratch_doubles(dpb) * sizeof(double);
  if (!bids.empty()) {
    if (per_blk > (size_t)maxsm) {
      h->err = "clique of order " + std::to_string(dpb) + " exceeds the shared-memory Jacobi path";
      return HSDE_ERR_ARG;
    }
    s.block_plan.smem = per_blk;
    RC(dupload(h, &s.block_plan.ids, bids.data(), bids.size()));
    s.block_plan.pstride = 5 * (int64_t)dpb * dpb;  // class split: 5 d x d regions
    RC(dalloc(h, &s.block_plan.pscratch, (size_t)bids.size() * s.block_plan.pstride));
    const int sm = maxsm;
    int dmax = 0;
    for (int k : bids) dmax = std::max(dmax, s.sizes[k]);
    // cold path variant: capacity d <= 84 / 96 (larger cliques of the plan
    // are flagged to the Jacobi launch that follows)
    int dmin = 1 << 30;
    for (int k : bids) dmin = std::min(dmin, s.sizes[k]);
    s.block_plan.cold_cv = dmin > kColdMaxD ? 0 : dmax <= 80 ? 1 : 2;
    if (s.block_plan.cold_cv) {
      s.block_plan.cold_smem = (size_t)cold_smem_doubles(std::min(dmax, kColdMaxD)) * sizeof(double);
      RC(dalloc(h, &s.block_plan.cfail, bids.size()));
      CK(cudaMemset(s.block_plan.cfail, 0, sizeof(int) * bids.size()));
      CK(cudaFuncSetAttribute(k_cone_cold<CONE_HOT, 20, 3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(cudaFuncSetAttribute(k_cone_cold<CONE_PLAIN, 20, 3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(cudaFuncSetAttribute(k_cone_cold<CONE_MINEIG, 20, 3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(cudaFuncSetAttribute(k_cone_cold<CONE_HOT, 24, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(cudaFuncSetAttribute(k_cone_cold<CONE_PLAIN, 24, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(cudaFuncSetAttribute(k_cone_cold<CONE_MINEIG, 24, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    }
    if (dmax <= kSplitMaxD) {
      s.block_plan.split_smem = std::max((size_t)split_smem_doubles(dmax) * sizeof(double), per_blk);
      s.W.cta_ids = s.block_plan.ids;  // k_scalars schedules them for k_cone_split
      s.W.cta_n = s.block_plan.count;
      s.block_plan.split_small = dmax <= kSplitSmallD;
      CK(cudaFuncSetAttribute(k_cone_split<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(cudaFuncSetAttribute(k_cone_split<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(cudaFuncSetAttribute(k_cone_split<true, kSplitThreadsSmall>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    }
    CK(cudaFuncSetAttribute(k_cone_block<CONE_HOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute(k_cone_block<CONE_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute(k_cone_block<CONE_MINEIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  }
  return 0;
}

// Partial S = A diag(p_inv) A' over the owned columns, sparse and row-wise:
// warp (i, part) walks its share of row i's CSR (ascending column l) and adds
//   S[i][j] += (a_il a_jl) p_l   for every nonzero a_jl of column l (CSC)
// into a shared-memory row (the rows j of one column are distinct: no
// conflicts); parts are summed in order by k_schur_parts_sum.  Deterministic,
// and bitwise symmetric (a_il a_jl = a_jl a_il).  Work ~ sum_l nnz(col l)^2
// instead of the dense m^2 n_c.
constexpr int kSchurParts = 8;
constexpr int kSchurBatch = 4;  // columns whose loads are in flight together

__global__ void __launch_bounds__(256) k_schur_rows(DevProblem P, int wpb, double *part) {
  extern __shared__ double srow[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w >= wpb) return;
  const int task = blockIdx.x * wpb + w;
  const int i = task / kSchurParts, sp = task - (task / kSchurParts) * kSchurParts;
  if (i >= P.m) return;
  const int m = P.m;
  double *row = srow + (size_t)w * m;
  for (int j = lane; j < m; j += 32) row[j] = 0.0;
  __syncwarp();
  const int64_t rb = P.a_rp[i], len = P.a_rp[i + 1] - rb;
  const int64_t kb = rb + len * sp / kSchurParts, ke = rb + len * (sp + 1) / kSchurParts;
  for (int64_t k0 = kb; k0 < ke; k0 += kSchurBatch) {
    int64_t cb = 0, ce = 0;
    double a = 0.0, pl = 0.0;
    if (lane < kSchurBatch && k0 + lane < ke) {
      const int l = P.a_col[k0 + lane];
      a = P.a_val[k0 + lane];  // a_il
      pl = P.p_inv[l];
      cb = P.at_cp[l];
      ce = P.at_cp[l + 1];
    }
    int jq[kSchurBatch];
    double aq[kSchurBatch], pq[kSchurBatch];
    int64_t cbq[kSchurBatch], ceq[kSchurBatch];
#pragma unroll
    for (int q = 0; q < kSchurBatch; ++q) {
      cbq[q] = __shfl_sync(0xffffffffu, cb, q);
      ceq[q] = __shfl_sync(0xffffffffu, ce, q);
      aq[q] = __shfl_sync(0xffffffffu, a, q);
      pq[q] = __shfl_sync(0xffffffffu, pl, q);
    }
    double av[kSchurBatch];
#pragma unroll
    for (int q = 0; q < kSchurBatch; ++q) {
      const int64_t e = cbq[q] + lane;
      jq[q] = e < ceq[q] ? P.at_row[e] : -1;
      av[q] = e < ceq[q] ? P.at_val[e] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kSchurBatch; ++q) {
      if (jq[q] >= 0) row[jq[q]] += (aq[q] * av[q]) * pq[q];
      __syncwarp();
      for (int64_t e = cbq[q] + 32 + lane; e < ceq[q]; e += 32)  // long columns
        row[P.at_row[e]] += (aq[q] * P.at_val[e]) * pq[q];
      __syncwarp();
    }
  }
  double *out = part + ((size_t)sp * m + i) * m;
  for (int j = lane; j < m; j += 32) out[j] = row[j];
}

__global__ void k_schur_parts_sum(const double *part, int64_t mm, double *S) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < mm;
       k += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int s = 0; s < kSchurParts; ++s) a += part[(size_t)s * mm + k];
    S[k] = a;
  }
}

// sparse row-wise partial Schur when a row of S fits in shared memory
int schur_partial_sparse(hsde_handle *h, ShardDev &s, bool *done) {
  *done = false;
  const int m = s.P.m;
  const size_t row_bytes = sizeof(double) * (size_t)m;
  const int wpb = (int)std::min<size_t>(8, (200u << 10) / std::max<size_t>(row_bytes, 1));
  if (wpb < 1 || m == 0) return 0;
  SetupTimer tick;
  RC(dalloc(h, &s.d_schur, (size_t)m * m));
  double *part = nullptr;
  CK(pool_malloc(h, (void **)&part, sizeof(double) * (size_t)kSchurParts * m * m));
  tick("    schur alloc");
  const size_t smem = row_bytes * wpb;
  CK(cudaFuncSetAttribute(k_schur_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t tasks = (int64_t)m * kSchurParts;
  k_schur_rows<<<(unsigned)((tasks + wpb - 1) / wpb), wpb * 32, smem, h->st>>>(s.P, wpb, part);
  CKL();
  tick("    schur rows");
  k_schur_parts_sum<<<grid_for((int64_t)m * m), kBlock, 0, h->st>>>(part, (int64_t)m * m, s.d_schur);
  CKL();
  CK(cudaStreamSynchronize(h->st));
  pool_free(h, part);
  tick("    schur sum+free");
  *done = true;
  return 0;
}

// Partial S = sum over owned columns of A diag(p_inv) A' (dense chunks + DGEMM)
int schur_partial_dense(hsde_handle *h, ShardDev &s) {
  const int m = s.P.m, n_c = s.P.n_c;
  RC(dalloc(h, &s.d_schur, (size_t)m * m));
  CK(cudaMemsetAsync(s.d_schur, 0, sizeof(double) * m * m, h->st));
  const size_t budget = 256ull << 20;  // bytes per densified chunk
  int wc = (int)std::max<size_t>(1, budget / (sizeof(double) * (size_t)m));
  wc = std::min(wc, std::max(n_c, 1));
  double *Dm = nullptr, *Ds = nullptr;
  CK(pool_malloc(h, (void **)&Dm, sizeof(double) * (size_t)m * wc));
  CK(pool_malloc(h, (void **)&Ds, sizeof(double) * (size_t)m * wc));
  cublasHandle_t cb;
  if (cublasCreate(&cb) != CUBLAS_STATUS_SUCCESS) {
    h->err = "cublasCreate failed";
    return HSDE_ERR_CUDA;
  }
  cublasSetStream(cb, h->st);
  const double one = 1.0;
  int rc = 0;
  for (int c0 = 0; c0 < n_c && !rc; c0 += wc) {
    const int c1 = std::min(n_c, c0 + wc);
    const int w = c1 - c0;
    CK(cudaMemsetAsync(Dm, 0, sizeof(double) * (size_t)m * w, h->st));
    CK(cudaMemsetAsync(Ds, 0, sizeof(double) * (size_t)m * w, h->st));
    k_densify<<<grid_for(w), kBlock, 0, h->st>>>(s.P, c0, c1, Dm, Ds);
    CKL();
    if (cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_T, m, m, w, &one, Ds, m, Dm, m, &one, s.d_schur, m) !=
        CUBLAS_STATUS_SUCCESS) {
      h->err = "cublasDgemm failed";
      rc = HSDE_ERR_CUDA;
    }
  }
  CK(cudaStreamSynchronize(h->st));
  cublasDestroy(cb);
  pool_free(h, Dm);
  pool_free(h, Ds);
  return rc;
}

// One cuSOLVER handle per device for the process: creating one costs up to a
// few hundred ms (module load), which every solve_decomposed call would pay.
cusolverDnHandle_t solver_handle(int dev) {
  static std::mutex mu;
  static cusolverDnHandle_t hs[64] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!hs[dev] && cusolverDnCreate(&hs[dev]) != CUSOLVER_STATUS_SUCCESS) hs[dev] = nullptr;
  return hs[dev];
}

// reduced S (in the shard's d_schur) -> S^{-1} (cuSOLVER Cholesky, potrs on I)
int schur_factor(hsde_handle *h, ShardDev &s) {
  SetupTimer tick;
  const int m = s.P.m;
  double *S = s.d_schur;
  k_add_identity<<<grid_for(m), kBlock, 0, h->st>>>(S, m);
  CKL();
  k_finite_check<<<grid_for((int64_t)m * m), kBlock, 0, h->st>>>(S, (int64_t)m * m, s.W.err);
  CKL();
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, s.W.err, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (flag) {
    CK(cudaMemset(s.W.err, 0, sizeof(int)));
    h->err = "Cholesky of the " + std::to_string(m) + " x " + std::to_string(m) +
             " reduced system failed: non-finite entries";
    return HSDE_ERR_FACTOR;
  }
  static std::mutex cs_mu;  // the shared handle is used by one setup at a time
  std::lock_guard<std::mutex> cs_lock(cs_mu);
  cusolverDnHandle_t cs = solver_handle(h->dev);
  if (!cs) {
    h->err = "cusolverDnCreate failed";
    return HSDE_ERR_CUDA;
  }
  cusolverDnSetStream(cs, h->st);
  int lwork = 0;
  cusolverDnDpotrf_bufferSize(cs, CUBLAS_FILL_MODE_LOWER, m, S, m, &lwork);
  double *work = nullptr;
  int *dinfo = nullptr;
  CK(pool_malloc(h, (void **)&work, sizeof(double) * std::max(lwork, 1)));
  CK(pool_malloc(h, (void **)&dinfo, sizeof(int)));
  tick("    potrf setup");
  cusolverDnDpotrf(cs, CUBLAS_FILL_MODE_LOWER, m, S, m, work, lwork, dinfo);
  int info = 0;
  CK(cudaMemcpyAsync(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (info != 0) {
    pool_free(h, work);
    pool_free(h, dinfo);
    h->err = "Cholesky of the " + std::to_string(m) + " x " + std::to_string(m) +
             " reduced system failed: leading minor " + std::to_string(info) + " not positive";
    return HSDE_ERR_FACTOR;
  }
  double *X = nullptr;
  RC(dalloc(h, &X, (size_t)m * m));
  k_identity<<<grid_for((int64_t)m * m), kBlock, 0, h->st>>>(X, m);
  CKL();
  cusolverDnDpotrs(cs, CUBLAS_FILL_MODE_LOWER, m, m, S, m, X, m, dinfo);
  CK(cudaStreamSynchronize(h->st));
  pool_free(h, work);
  pool_free(h, dinfo);
  k_symmetrize<<<grid_for((int64_t)m * m), kBlock, 0, h->st>>>(X, m, S);  // S^{-1}, symmetric
  CKL();
  tick("    potrf+potrs");
  s.P.sinv = S;
  s.P.schur_diag = 0;
  return 0;
}

int setup_schur(hsde_handle *h) {
  const int G = (int)h->sh.size();
  const int m = h->sh[0].P.m;
  for (auto &s : h->sh) {
    if (h->schur_diag) {
      RC(dalloc(h, &s.d_schur, std::max(m, 1)));
      k_diag_schur<<<grid_for(m), kBlock, 0, h->st>>>(s.P, s.d_schur);
      CKL();
    } else {
      bool done = false;
      RC(schur_partial_sparse(h, s, &done));
      if (!done) RC(schur_partial_dense(h, s));
    }
  }
  if (h->mode == MODE_EMULATED) {
    std::vector<double *> p(G);
    for (int g = 0; g < G; ++g) p[g] = h->sh[g].d_schur;
    RC(dupload(h, &h->d_ptrs[BUF_SCHUR], p.data(), G));
  }
  RC(reduce(h, BUF_SCHUR, h->schur_diag ? (int64_t)m : (int64_t)m * m));
  for (auto &s : h->sh) {
    if (!h->schur_diag) {
      RC(schur_factor(h, s));
      continue;
    }
    k_diag_finish<<<grid_for(m), kBlock, 0, h->st>>>(s.d_schur, m, s.W.err);
    CKL();
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, s.W.err, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (flag) {
      CK(cudaMemset(s.W.err, 0, sizeof(int)));
      h->err = "Cholesky of the " + std::to_string(m) + " x " + std::to_string(m) +
               " reduced system failed: diagonal entry not positive";
      return HSDE_ERR_FACTOR;
    }
    s.P.sinv = s.d_schur;
    s.P.schur_diag = 1;
  }
  return 0;
}

int compute_minv_zeta(hsde_handle *h) {
  const int G = (int)h->sh.size();
  std::vector<const double *> rho(G);
  std::vector<double *> out(G);
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    double *mz = nullptr;
    RC(dalloc(h, &mz, (size_t)(s.P.total - 1)));
    rho[g] = s.d_zeta;
    out[g] = mz;
  }
  // single GPU keeps the reference's explicit uy = wy - A ua (solver.py:240-241)
  RC(inner_dist(h, rho, out, !h->multi()));
  // zeta . M zeta = c . mz_x (owned) - b . mz_y (replicated: lead shard)
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    s.P.mz = out[g];
    RC(dev_dot_owned(h, s, s.P.c, out[g], s.W.red + 0));
    RC(dev_dot(h, s, s.P.b, out[g] + s.P.n_c + s.P.n_d, s.P.m, s.W.red + 1));
    if (!s.P.lead) CK(cudaMemsetAsync(s.W.red + 1, 0, sizeof(double), h->st));
  }
  RC(reduce(h, BUF_RED, 2));
  double r[2];
  CK(cudaMemcpyAsync(r, h->sh[0].W.red, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  const double zmz = r[0] - r[1];
  const double zs = 1.0 + zmz;  // solver.py:269
  if (!(zs > 0)) {
    char buf[128];
    snprintf(buf, sizeof buf, "rank-one update scale %g is not positive; data is ill-scaled", zs);
    h->err = buf;
    return HSDE_ERR_FACTOR;
  }
  for (auto &s : h->sh) {
    s.P.zmz = zmz;
    s.P.zeta_scale = zs;
  }
  h->info.zeta_scale = zs;
  return 0;
}

int init_state(hsde_handle *h) {
  for (auto &s : h->sh) {
    const int64_t T = s.P.total;
    CK(cudaMemsetAsync(s.S.u, 0, sizeof(double) * T, h->st));
    CK(cudaMemsetAsync(s.S.w, 0, sizeof(double) * T, h->st));
    const double one = 1.0;
    CK(cudaMemcpyAsync(s.S.u + T - 1, &one, sizeof(double), cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(s.S.w + T - 1, &one, sizeof(double), cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(s.d_prev_u, s.S.u, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(s.d_prev_w, s.S.w, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemsetAsync(s.W.vvalid, 0, sizeof(int) * std::max(s.P.p, 1), h->st));
    k_set_i32<<<1, 256, 0, h->st>>>(s.W.cnext, std::max(s.P.p, 1), 1);  // no basis: cold path first
    CK(cudaStreamSynchronize(h->st));
  }
  return 0;
}

// ---- per-shard construction -------------------------------------------------------

int validate(hsde_handle *h, const hsde_problem_desc *d) {
  const int m = d->m, n_c = d->n_c, p = d->p;
  const int64_t n_d = d->n_d, nnz = d->nnz;
  if (m < 0 || n_c < 0 || p < 0 || n_d < 0 || nnz < 0) {
    h->err = "negative dimension";
    return HSDE_ERR_ARG;
  }
  if (d->a_row_ptr[0] != 0 || d->a_row_ptr[m] != nnz) {
    h->err = "a_row_ptr inconsistent with nnz";
    return HSDE_ERR_ARG;
  }
  for (int i = 0; i < m; ++i) {
    if (d->a_row_ptr[i + 1] < d->a_row_ptr[i]) {
      h->err = "a_row_ptr not monotone";
      return HSDE_ERR_ARG;
    }
  }
  // column indices are checked on the device after the upload (check_csr_device)
  if (d->clique_offsets[0] != 0 || d->clique_offsets[p] != n_d) {
    h->err = "clique offsets inconsistent with n_d";
    return HSDE_ERR_ARG;
  }
  for (int k = 0; k < p; ++k) {
    const int64_t dk = d->clique_sizes[k];
    if (dk < 1 || d->clique_offsets[k + 1] - d->clique_offsets[k] != dk * dk) {
      h->err = "clique size / offset mismatch at clique " + std::to_string(k);
      return HSDE_ERR_ARG;
    }
  }
  for (int64_t j = 0; j < n_d; ++j)
    if (d->slot_cov[j] < 0 || d->slot_cov[j] >= n_c) {
      h->err = "slot_cov out of range";
      return HSDE_ERR_ARG;
    }
  if (d->n_sep_local > 0 && (!d->sep_local || !d->sep_pos)) {
    h->err = "separator lists missing";
    return HSDE_ERR_ARG;
  }
  for (int i = 0; i < d->n_sep_local; ++i)
    if (d->sep_local[i] < 0 || d->sep_local[i] >= n_c || d->sep_pos[i] < 0 ||
        d->sep_pos[i] >= d->n_sep) {
      h->err = "separator index out of range";
      return HSDE_ERR_ARG;
    }
  return 0;
}

// upload shard data (everything that does not depend on normalisation)
// a_col in range and strictly ascending within each row; first bad row or -1
__global__ void k_check_csr(const int64_t *rp, const int *col, int m, int n_c, int *bad_row) {
  for (int i = blockIdx.x; i < m; i += gridDim.x)
    for (int64_t k = rp[i] + threadIdx.x; k < rp[i + 1]; k += blockDim.x) {
      const int c = col[k];
      if (c < 0 || c >= n_c || (k > rp[i] && c <= col[k - 1])) atomicMin(bad_row, i);
    }
}

int check_csr_device(hsde_handle *h, const int64_t *rp, const int *col, int m, int n_c) {
  int *bad = nullptr;
  CK(pool_malloc(h, (void **)&bad, sizeof(int)));
  const int init = INT32_MAX;
  CK(cudaMemcpy(bad, &init, sizeof(int), cudaMemcpyHostToDevice));
  if (m > 0) k_check_csr<<<std::min(m, 148 * 8), kBlock, 0, h->st>>>(rp, col, m, n_c, bad);
  CKL();
  int hb = INT32_MAX;
  CK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  pool_free(h, bad);
  if (hb != INT32_MAX) {
    h->err = "a_col out of range or not strictly ascending in row " + std::to_string(hb);
    return HSDE_ERR_ARG;
  }
  return 0;
}

// ---- device construction of the CSC of A (rows ascending within a column)
__global__ void k_row_of(const int64_t *rp, int m, int *row_of) {
  for (int i = blockIdx.x; i < m; i += gridDim.x)
    for (int64_t k = rp[i] + threadIdx.x; k < rp[i + 1]; k += blockDim.x) row_of[k] = i;
}

__global__ void k_iota(int *x, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    x[k] = (int)k;
}

__global__ void k_col_count(const int *col, int64_t nnz, unsigned long long *cnt) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[k] + 1, 1ull);  // integer counts: order-independent
}

__global__ void k_csc_gather(const int *perm, const int *row_of, const double *val, int64_t nnz,
                             int *at_row, double *at_val) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int e = perm[k];
    at_row[k] = row_of[e];
    at_val[k] = val[e];
  }
}

__global__ void k_maxcol(const int64_t *cp, int n_c, const unsigned char *owned,
                         unsigned long long *mx) {
  unsigned long long best = 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_c; c += gridDim.x * blockDim.x)
    if (!owned || owned[c]) best = max(best, (unsigned long long)(cp[c + 1] - cp[c]));
  atomicMax(mx, best);
}

int build_csc_device(hsde_handle *h, int m, int n_c, int64_t nnz, const int64_t *rp, const int *col,
                     const double *val, int64_t **at_cp, int **at_row, double **at_val) {
  SetupTimer tick;
  RC(dalloc(h, at_cp, n_c + 1));
  RC(dalloc(h, at_row, nnz));
  RC(dalloc(h, at_val, nnz));
  tick("    csc alloc");
  unsigned long long *cnt = reinterpret_cast<unsigned long long *>(*at_cp);
  CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (n_c + 1), h->st));
  if (nnz == 0) return 0;
  if (nnz > INT32_MAX) {
    h->err = "nnz(A) above 2^31 is not supported";
    return HSDE_ERR_ARG;
  }
  const int g = 148 * 8;
  k_col_count<<<g, kBlock, 0, h->st>>>(col, nnz, cnt);
  CKL();
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, cnt, n_c + 1, h->st);
  int *row_of = nullptr, *idx = nullptr, *perm = nullptr, *keys_out = nullptr;
  void *tmp = nullptr;
  size_t tb2 = 0;
  int end_bit = 1;
  while ((1ll << end_bit) < (long long)n_c) ++end_bit;
  cub::DeviceRadixSort::SortPairs(nullptr, tb2, col, keys_out, idx, perm, (int)nnz, 0, end_bit, h->st);
  CK(pool_malloc(h, (void **)&tmp, std::max(tb, tb2)));
  CK(pool_malloc(h, (void **)&row_of, sizeof(int) * nnz));
  CK(pool_malloc(h, (void **)&idx, sizeof(int) * nnz));
  CK(pool_malloc(h, (void **)&perm, sizeof(int) * nnz));
  CK(pool_malloc(h, (void **)&keys_out, sizeof(int) * nnz));
  tick("    csc tmp alloc");
  cub::DeviceScan::InclusiveSum(tmp, tb, cnt, cnt, n_c + 1, h->st);
  k_row_of<<<std::min(m, 148 * 8), kBlock, 0, h->st>>>(rp, m, row_of);
  k_iota<<<g, kBlock, 0, h->st>>>(idx, nnz);
  CKL();
  // stable: equal columns keep CSR (row-ascending) order
  cub::DeviceRadixSort::SortPairs(tmp, tb2, col, keys_out, idx, perm, (int)nnz, 0, end_bit, h->st);
  k_csc_gather<<<g, kBlock, 0, h->st>>>(perm, row_of, val, nnz, *at_row, *at_val);
  CKL();
  CK(cudaStreamSynchronize(h->st));
  tick("    csc sort+gather");
  pool_free(h, tmp);
  pool_free(h, row_of);
  pool_free(h, idx);
  pool_free(h, perm);
  pool_free(h, keys_out);
  tick("    csc free");
  return 0;
}

// Cover lists on the device (the host loop took ~18 ms on config 4's 2.56M
// slots): cov_slot = slots sorted by covered coordinate, ascending slot within
// a coordinate (stable radix sort: bincount order, graphs.py:228), cov_ptr
// from the integer counts, p_inv = 1 / (1 + D/2) (solver.py:250) unless the
// global cover counts are given, and the heavy coordinates (> kHeavy slots)
// in ascending order.
__global__ void k_cov_finish(const unsigned long long *cnt, int n_c, int *cov_ptr, const double *cover_counts,
                             double *p_inv, unsigned char *heavy_flag) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= n_c; c += gridDim.x * blockDim.x) {
    cov_ptr[c] = (int)cnt[c];
    if (c == n_c) continue;
    const int k = (int)(cnt[c + 1] - cnt[c]);
    const double D = cover_counts ? cover_counts[c] : (double)k;
    p_inv[c] = 1.0 / (1.0 + 0.5 * D);
    heavy_flag[c] = k > kHeavy;
  }
}

int build_covers_device(hsde_handle *h, int n_c, int64_t n_d, const int *slot_cov, const double *cover_counts_d,
                        int **cov_ptr, int **cov_slot, double **p_inv, int **heavy, int *n_heavy) {
  RC(dalloc(h, cov_ptr, n_c + 1));
  RC(dalloc(h, cov_slot, std::max<int64_t>(n_d, 1)));
  RC(dalloc(h, p_inv, std::max(n_c, 1)));
  unsigned long long *cnt = nullptr;
  unsigned char *flag = nullptr;
  int *idx = nullptr, *keys_out = nullptr, *hv = nullptr, *nsel = nullptr;
  void *tmp = nullptr;
  CK(pool_malloc(h, (void **)&cnt, sizeof(unsigned long long) * (n_c + 1)));
  CK(pool_malloc(h, (void **)&flag, std::max(n_c, 1)));
  CK(pool_malloc(h, (void **)&hv, sizeof(int) * std::max(n_c, 1)));
  CK(pool_malloc(h, (void **)&nsel, sizeof(int)));
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (n_c + 1), h->st));
  const int g = 148 * 8;
  if (n_d > 0) {
    if (n_d > INT32_MAX) {
      h->err = "more than 2^31 clique slots are not supported";
      return HSDE_ERR_ARG;
    }
    k_col_count<<<g, kBlock, 0, h->st>>>(slot_cov, n_d, cnt);
    CKL();
  }
  size_t tb = 0, tb2 = 0, tb3 = 0;
  int end_bit = 1;
  while ((1ll << end_bit) < (long long)n_c) ++end_bit;
  cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, cnt, n_c + 1, h->st);
  cub::DeviceRadixSort::SortPairs(nullptr, tb2, slot_cov, keys_out, idx, *cov_slot, (int)n_d, 0, end_bit, h->st);
  cub::DeviceSelect::Flagged(nullptr, tb3, cub::CountingInputIterator<int>(0), flag, hv, nsel, n_c, h->st);
  CK(pool_malloc(h, (void **)&tmp, std::max(tb, std::max(tb2, tb3))));
  CK(pool_malloc(h, (void **)&idx, sizeof(int) * std::max<int64_t>(n_d, 1)));
  CK(pool_malloc(h, (void **)&keys_out, sizeof(int) * std::max<int64_t>(n_d, 1)));
  cub::DeviceScan::InclusiveSum(tmp, tb, cnt, cnt, n_c + 1, h->st);
  if (n_d > 0) {
    k_iota<<<g, kBlock, 0, h->st>>>(idx, n_d);
    CKL();
    cub::DeviceRadixSort::SortPairs(tmp, tb2, slot_cov, keys_out, idx, *cov_slot, (int)n_d, 0, end_bit, h->st);
  }
  k_cov_finish<<<grid_for(n_c + 1), kBlock, 0, h->st>>>(cnt, n_c, *cov_ptr, cover_counts_d, *p_inv, flag);
  CKL();
  cub::DeviceSelect::Flagged(tmp, tb3, cub::CountingInputIterator<int>(0), flag, hv, nsel, n_c, h->st);
  int nh = 0;
  CK(cudaMemcpyAsync(&nh, nsel, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  RC(dalloc(h, heavy, std::max(nh, 1)));
  if (nh) CK(cudaMemcpyAsync(*heavy, hv, sizeof(int) * nh, cudaMemcpyDeviceToDevice, h->st));
  *n_heavy = nh;
  CK(cudaStreamSynchronize(h->st));
  pool_free(h, tmp);
  pool_free(h, idx);
  pool_free(h, keys_out);
  pool_free(h, cnt);
  pool_free(h, flag);
  pool_free(h, hv);
  pool_free(h, nsel);
  return 0;
}

#include "hsde_setup_half.cuh"

int build_shard(hsde_handle *h, ShardDev &s, const hsde_problem_desc *d) {
  SetupTimer tick;
  const int m = d->m, n_c = d->n_c, p = d->p;
  const int64_t n_d = d->n_d, nnz = d->nnz;
  std::vector<unsigned char> owned(n_c, 1);
  if (d->owned)
    for (int c = 0; c < n_c; ++c) owned[c] = d->owned[c] ? 1 : 0;
  // A on the device: the CSR as given (all columns on a single shard, the
  // owned columns of a shard), then the CSC by a stable device radix sort
  int64_t *a_rp = nullptr, *at_cp_d = nullptr;
  int *a_col = nullptr, *at_row_d = nullptr;
  double *a_val = nullptr, *at_val_d = nullptr;
  std::vector<int64_t> rp(m + 1, 0);
  // (single shard) A goes up on a host thread -- staged pinned copies on their own
  // stream -- while this thread builds the segments, cover lists and small
  // uploads, none of which read A; joined before the CSC is built
  std::thread a_up;
  struct Joiner {
    std::thread &t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } a_join{a_up};
  int a_rc = 0;
  if (!d->owned) {
    rp.assign(d->a_row_ptr, d->a_row_ptr + m + 1);
    RC(dalloc(h, &a_rp, (size_t)m + 1));
    RC(dalloc(h, &a_col, (size_t)nnz));
    RC(dalloc(h, &a_val, (size_t)nnz));
    a_up = std::thread([&a_rc, h, d, a_rp, a_col, a_val, m, nnz] {
      cudaSetDevice(h->dev);
      a_rc = dcopy(h, a_rp, d->a_row_ptr, (size_t)m + 1);
      if (!a_rc) a_rc = dcopy(h, a_col, d->a_col, (size_t)nnz);
      if (!a_rc) a_rc = dcopy(h, a_val, d->a_val, (size_t)nnz);
    });
  } else {
    // CSC over all local columns (A' g is needed on every local coordinate)
    int64_t *f_rp = nullptr;
    int *f_col = nullptr;
    double *f_val = nullptr;
    CK(pool_malloc(h, (void **)&f_rp, sizeof(int64_t) * (m + 1)));
    CK(pool_malloc(h, (void **)&f_col, sizeof(int) * std::max<int64_t>(nnz, 1)));
    CK(pool_malloc(h, (void **)&f_val, sizeof(double) * std::max<int64_t>(nnz, 1)));
    CK(cudaMemcpy(f_rp, d->a_row_ptr, sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(f_col, d->a_col, sizeof(int) * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(f_val, d->a_val, sizeof(double) * nnz, cudaMemcpyHostToDevice));
    int rc = check_csr_device(h, f_rp, f_col, m, n_c);
    if (!rc) rc = build_csc_device(h, m, n_c, nnz, f_rp, f_col, f_val, &at_cp_d, &at_row_d, &at_val_d);
    pool_free(h, f_rp);
    pool_free(h, f_col);
    pool_free(h, f_val);
    RC(rc);
    // CSR over the owned columns (the only columns this shard adds into A t)
    std::vector<int> col;
    std::vector<double> val;
    col.reserve(nnz);
    val.reserve(nnz);
    for (int i = 0; i < m; ++i) {
      for (int64_t k = d->a_row_ptr[i]; k < d->a_row_ptr[i + 1]; ++k)
        if (owned[d->a_col[k]]) {
          col.push_back(d->a_col[k]);
          val.push_back(d->a_val[k]);
        }
      rp[i + 1] = (int64_t)col.size();
    }
    RC(dupload(h, &a_rp, rp.data(), m + 1));
    RC(dupload(h, &a_col, col.data(), col.size()));
    RC(dupload(h, &a_val, val.data(), val.size()));
  }
  tick("  A alloc / sharded CSR+CSC");
  // row segments
  std::vector<int> seg_row, row_seg(m + 1, 0);
  std::vector<int64_t> seg_beg;
  for (int i = 0; i < m; ++i) {
    row_seg[i] = (int)seg_row.size();
    for (int64_t k = rp[i]; k < rp[i + 1]; k += kSegNnz) {
      seg_row.push_back(i);
      seg_beg.push_back(k);
    }
  }
  row_seg[m] = (int)seg_row.size();
  tick("  host CSR+segments");
  // cover lists, cover counts D, P^{-1} and the heavy coordinates: on the device
  // (build_covers_device) after slot_cov is uploaded
  std::vector<int> sep_of;
  if (d->n_sep > 0) {
    sep_of.assign(n_c, -1);
    for (int i = 0; i < d->n_sep_local; ++i) sep_of[d->sep_local[i]] = d->sep_pos[i];
  }
  s.nc2_owned = 0;
  for (int c = 0; c < n_c; ++c)
    if (owned[c]) s.nc2_owned += d->c[c] * d->c[c];
  s.sizes.assign(d->clique_sizes, d->clique_sizes + p);
  tick("  host covers");
  // ---- device problem
  DevProblem &P = s.P;
  P.m = m;
  P.n_c = n_c;
  P.p = p;
  P.n_d = n_d;
  P.nnz = nnz;
  P.total = (int64_t)n_c + 2 * n_d + m + 1;
  P.alpha = h->set.alpha;
  P.nseg = (int)seg_row.size();
  P.n_sep = d->n_sep;
  P.n_sep_local = d->n_sep_local;
  P.lead = d->follower ? 0 : 1;
  int64_t *seg_beg_d = nullptr, *cl_off = nullptr;
  int *seg_row_d = nullptr, *row_seg_d = nullptr;
  int *cov_ptr_d = nullptr, *cov_slot_d = nullptr, *slot_cov_d = nullptr, *cl_size = nullptr;
  int *heavy_d = nullptr, *sep_of_d = nullptr, *sep_local_d = nullptr, *sep_pos_d = nullptr;
  unsigned char *owned_d = nullptr;
  double *pinv_d = nullptr;
  RC(dupload(h, &seg_row_d, seg_row.data(), seg_row.size()));
  RC(dupload(h, &seg_beg_d, seg_beg.data(), seg_beg.size()));
  RC(dupload(h, &row_seg_d, row_seg.data(), m + 1));
  RC(dupload(h, &slot_cov_d, d->slot_cov, n_d));
  int n_heavy = 0;
  {
    double *cc_d = nullptr;  // global cover counts (sharded runs), temporary
    if (d->cover_counts) {
      CK(pool_malloc(h, (void **)&cc_d, sizeof(double) * std::max(n_c, 1)));
      CK(cudaMemcpy(cc_d, d->cover_counts, sizeof(double) * n_c, cudaMemcpyHostToDevice));
    }
    RC(build_covers_device(h, n_c, n_d, slot_cov_d, cc_d, &cov_ptr_d, &cov_slot_d, &pinv_d, &heavy_d, &n_heavy));
    if (cc_d) pool_free(h, cc_d);
  }
  RC(dupload(h, &cl_off, d->clique_offsets, p + 1));
  RC(dupload(h, &cl_size, d->clique_sizes, p));
  RC(dupload(h, &s.d_c_orig, d->c, n_c));
  RC(dupload(h, &s.d_b_orig, d->b, m));
  if (d->owned) {
    RC(dupload(h, &owned_d, owned.data(), n_c));
    P.owned = owned_d;
  }
  if (d->n_sep > 0) {
    RC(dupload(h, &sep_of_d, sep_of.data(), n_c));
    RC(dupload(h, &sep_local_d, d->sep_local, d->n_sep_local));
    RC(dupload(h, &sep_pos_d, d->sep_pos, d->n_sep_local));
    P.sep_of = sep_of_d;
    P.sep_local = sep_local_d;
    P.sep_pos = sep_pos_d;
  }
  if (a_up.joinable()) {
    a_up.join();
    RC(a_rc);
    tick("  A upload (joined)");
    RC(check_csr_device(h, a_rp, a_col, m, n_c));
    RC(build_csc_device(h, m, n_c, nnz, a_rp, a_col, a_val, &at_cp_d, &at_row_d, &at_val_d));
  }
  {
    // longest owned column (diagonal-Schur test)
    unsigned long long *mx = nullptr;
    CK(pool_malloc(h, (void **)&mx, sizeof(unsigned long long)));
    CK(cudaMemset(mx, 0, sizeof(unsigned long long)));
    unsigned char *own_tmp = nullptr;
    if (d->owned) {
      CK(pool_malloc(h, (void **)&own_tmp, n_c));
      CK(cudaMemcpy(own_tmp, owned.data(), n_c, cudaMemcpyHostToDevice));
    }
    k_maxcol<<<grid_for(n_c), kBlock, 0, h->st>>>(at_cp_d, n_c, own_tmp, mx);
    CKL();
    unsigned long long hm = 0;
    CK(cudaMemcpyAsync(&hm, mx, sizeof hm, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    s.maxcol = (int64_t)hm;
    pool_free(h, mx);
    pool_free(h, own_tmp);
  }
  tick("  A CSR+CSC (device)");
  P.a_rp = a_rp;
  P.a_col = a_col;
  P.a_val = a_val;
  P.at_cp = at_cp_d;
  P.at_row = at_row_d;
  P.at_val = at_val_d;
  P.seg_row = seg_row_d;
  P.seg_beg = seg_beg_d;
  P.row_seg = row_seg_d;
  P.cov_ptr = cov_ptr_d;
  P.cov_slot = cov_slot_d;
  P.slot_cov = slot_cov_d;
  P.cl_off = cl_off;
  P.cl_size = cl_size;
  P.p_inv = pinv_d;
  P.heavy = heavy_d;
  P.n_heavy = n_heavy;
  tick("  uploads");
  RC(build_half(h, s));
  tick("  half-pass layouts");
  // state + work
  const int64_t T = P.total;
  RC(dalloc(h, &s.S.u, T));
  RC(dalloc(h, &s.S.w, T));
  RC(dalloc(h, &s.d_prev_u, T));
  RC(dalloc(h, &s.d_prev_w, T));
  RC(dalloc(h, &s.d_tmp, T));
  RC(dalloc(h, &s.d_tmp2, T));
  RC(dalloc(h, &s.d_tmp3, T));
  RC(dalloc(h, &s.d_hv, n_c));
  RC(dalloc(h, &s.W.t, n_c));
  RC(dalloc(h, &s.W.ua, n_c));
  RC(dalloc(h, &s.W.ry, m));
  RC(dalloc(h, &s.W.qseg, P.nseg));
  RC(dalloc(h, &s.d_qseg2, P.nseg));
  RC(dalloc(h, &s.W.qp, m));
  RC(dalloc(h, &s.W.uy, m));
  RC(dalloc(h, &s.W.part, kMaxParts));
  RC(dalloc(h, &s.W.scal, S_COUNT));
  RC(dalloc(h, &s.W.err, 1));
  RC(dalloc(h, &s.d_chk, 64));
  RC(dalloc(h, &s.d_mineig, std::max(p, 1)));
  RC(dalloc(h, &s.W.vstore, n_d));
  RC(dalloc(h, &s.W.vvalid, std::max(p, 1)));
  RC(dalloc(h, &s.W.ccur, std::max(p, 1)));
  RC(dalloc(h, &s.W.cnext, std::max(p, 1)));
  RC(dalloc(h, &s.W.sweeps, std::max(p, 1)));
  RC(dalloc(h, &s.W.cstate, std::max(p, 1)));
  RC(dalloc(h, &s.W.ckey, std::max(p, 1)));
  RC(dalloc(h, &s.W.corder, std::max(p, 1)));
  RC(dalloc(h, &s.W.xarg, std::max<int64_t>(n_d, 1)));
  RC(dalloc(h, &s.W.sepbuf, std::max(d->n_sep, 1)));
  RC(dalloc(h, &s.W.qbuf, std::max(m, 1)));
  RC(dalloc(h, &s.W.red, 8));
  // diagnostics buffer (Jacobi history, phase stamps): only under HSDE_DEBUG=1,
  // so production iterations carry no diagnostic stores
  s.W.dbg = nullptr;
  if (const char *e = std::getenv("HSDE_DEBUG"); e && std::atoi(e)) RC(dalloc(h, &s.W.dbg, 64));
  s.W.dbg_clique = 0;
  CK(cudaMemset(s.W.err, 0, sizeof(int)));
  CK(cudaMemset(s.W.vvalid, 0, sizeof(int) * std::max(p, 1)));
  k_set_i32<<<1, 256>>>(s.W.ccur, std::max(p, 1), 1);
  k_set_i32<<<1, 256>>>(s.W.cnext, std::max(p, 1), 1);
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(s.W.sweeps, 0, sizeof(int) * std::max(p, 1)));
  CK(cudaMemset(s.W.cstate, 0xff, sizeof(int) * std::max(p, 1)));
  CK(cudaMemset(s.W.ckey, 0, sizeof(int) * std::max(p, 1)));
  CK(cudaMemset(s.d_chk, 0, sizeof(double) * 64));
  s.grid_nc = grid_for(n_c);
  s.grid_ua = s.grid_nc;
  {
    auto env_cap = [](const char *name, int def) {
      const char *e = std::getenv(name);
      return e ? std::max(1, atoi(e)) : def;
    };
    s.grid_rhs = grid_for(n_c, env_cap("HSDE_RHS_CTAS", 148 * 8));
    s.grid_xupd = grid_for(n_c, env_cap("HSDE_XUPD_CTAS", 148 * 8));
  }
  if (P.half) {
    // two CTAs' worth of slices per SM slot (148 x 16): the second wave
    // balances the ragged slice lengths (config 4: 76 -> 68 us vs 148 x 8)
    int cap = 148 * 16;
    if (const char *e = std::getenv("HSDE_UA_CTAS")) cap = std::max(1, std::min(kMaxParts, atoi(e)));
    s.grid_ua = std::max(1, std::min(cap, (P.n_slice + 7) / 8));
    const int sm = (int)(sizeof(double) * (size_t)m);
    if (sm > 48 * 1024) {
      CK(cudaFuncSetAttribute(k_ua_half<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(cudaFuncSetAttribute(k_ua_half<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    }
  }
  s.grid_nd = grid_for(n_d);
  s.grid_m = grid_for(m);
  s.grid_T = grid_for(T);
  s.grid_heavy = (P.n_heavy + (kBlock / 32) - 1) / (kBlock / 32);
  s.grid_seg = std::max(1, (int)((P.nseg * 32LL + kBlock - 1) / kBlock));
  s.schur_smem = sizeof(double) * std::max(m, 1);
  s.grid_schur = 1;
  if (s.schur_smem > 48 * 1024) {
    if (cudaFuncSetAttribute(k_schur, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)s.schur_smem) != cudaSuccess) {
      h->err = "m too large for the shared-memory Schur apply";
      return HSDE_ERR_ARG;
    }
  }
  RC(setup_cone_plans(h, s, d->clique_sizes, p));
  return 0;
}

// normalised data (after the global |c| is known)
int set_data(hsde_handle *h, ShardDev &s, const hsde_problem_desc *d, double sc, double sb) {
  const int m = d->m, n_c = d->n_c;
  const int64_t n_d = d->n_d;
  std::vector<double> cint(n_c), bint(m);
  for (int c = 0; c < n_c; ++c) cint[c] = sc == 1.0 ? d->c[c] : sc * d->c[c];
  for (int i = 0; i < m; ++i) bint[i] = sb == 1.0 ? d->b[i] : sb * d->b[i];
  double *c_d = nullptr, *b_d = nullptr;
  RC(dupload(h, &c_d, cint.data(), n_c));
  RC(dupload(h, &b_d, bint.data(), m));
  s.P.c = c_d;
  s.P.b = b_d;
  const double consts[4] = {sb, sc, 1.0, 0.0};
  RC(dupload(h, &s.d_consts, consts, 4));
  // zeta = (c, 0, -b, 0) (solver.py:264): zero on the device, two segments copied
  RC(dalloc(h, &s.d_zeta, (size_t)(s.P.total - 1)));
  CK(cudaMemsetAsync(s.d_zeta, 0, sizeof(double) * (size_t)(s.P.total - 1), h->st));
  std::vector<double> nb(m);
  for (int i = 0; i < m; ++i) nb[i] = -bint[i];
  CK(cudaMemcpyAsync(s.d_zeta, c_d, sizeof(double) * n_c, cudaMemcpyDeviceToDevice, h->st));
  CK(cudaMemcpyAsync(s.d_zeta + n_c + n_d, nb.data(), sizeof(double) * m, cudaMemcpyHostToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
  return 0;
}

int create_impl(const hsde_problem_desc *descs, int nshards, const hsde_settings *st,
                const hsde_comm *comm, hsde_handle *h) {
  cudaError_t e = cudaSetDevice(h->dev);
  if (e != cudaSuccess) {
    h->err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
    return HSDE_ERR_CUDA;
  }
  if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess) {
    h->err = "stream create failed";
    return HSDE_ERR_CUDA;
  }
  retain_pool(h->dev);
  if (int n = 0; cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, h->dev) == cudaSuccess && n > 0) h->n_sm = n;
  for (int a = 0; a < hsde_handle::kAux; ++a) {
    if (cudaStreamCreateWithFlags(&h->aux[a], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_join[a], cudaEventDisableTiming) != cudaSuccess) {
      h->err = "aux stream / event create failed";
      return HSDE_ERR_CUDA;
    }
  }
  if (cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_xjoin, cudaEventDisableTiming) != cudaSuccess) {
    h->err = "event create failed";
    return HSDE_ERR_CUDA;
  }
  if (comm && comm->world >= 1) {  // explicit communicator: NCCL (a 1-rank comm is valid)
    if (nshards != 1) {
      h->err = "NCCL mode takes exactly one shard per rank";
      return HSDE_ERR_ARG;
    }
    h->mode = MODE_NCCL;
    h->world = comm->world;
    h->rank = comm->rank;
    ncclUniqueId id;
    static_assert(sizeof(id.internal) == HSDE_NCCL_ID_BYTES, "nccl id size");
    memcpy(id.internal, comm->nccl_id, HSDE_NCCL_ID_BYTES);
    ncclResult_t r = ncclCommInitRank(&h->nccl, comm->world, id, comm->rank);
    if (r != ncclSuccess) {
      h->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      return HSDE_ERR_CUDA;
    }
  } else if (nshards > 1) {
    h->mode = MODE_EMULATED;
  }
  SetupTimer tick;
  tick("context+stream");
  const int m = descs[0].m;
  h->n_sep = descs[0].n_sep;
  for (int g = 0; g < nshards; ++g) {
    RC(validate(h, &descs[g]));
    if (descs[g].m != m || descs[g].n_sep != h->n_sep) {
      h->err = "shards disagree on m or the separator count";
      return HSDE_ERR_ARG;
    }
  }
  tick("validate");
  h->sh.resize(nshards);
  for (int g = 0; g < nshards; ++g) RC(build_shard(h, h->sh[g], &descs[g]));
  tick("build_shard");
  if (h->mode == MODE_EMULATED) {
    const int bufs[] = {BUF_SEP, BUF_Q, BUF_RED, BUF_CHK, BUF_MINEIG};
    for (int b : bufs) {
      std::vector<double *> p(nshards);
      for (int g = 0; g < nshards; ++g) p[g] = buf_ptr(h->sh[g], b);
      RC(dupload(h, &h->d_ptrs[b], p.data(), nshards));
    }
  }
  // ---- global scalars: |c|^2 over owners; diagonal-Schur test (each owned
  // column has <= 1 nonzero on every shard; reduced as a count of violators)
  for (auto &s : h->sh) {
    const double v[2] = {s.nc2_owned, s.maxcol > 1 ? 1.0 : 0.0};
    CK(cudaMemcpy(s.W.red, v, sizeof v, cudaMemcpyHostToDevice));
  }
  RC(reduce(h, BUF_RED, 2));
  double gv[2];
  CK(cudaMemcpyAsync(gv, h->sh[0].W.red, sizeof gv, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  h->schur_diag = gv[1] == 0.0;
  for (auto &s : h->sh)
    s.grid_schur = h->schur_diag ? grid_for(m, 64)
                                 : std::min(148 * 8, std::max(1, (m + 1) / ((kBlock / 32) / kSchurSplit)));
  const double *bsrc = descs[0].b;
  double nb2 = 0;
  for (int i = 0; i < m; ++i) nb2 += bsrc[i] * bsrc[i];
  double sc = 1.0, sb = 1.0;
  if (st->normalize) {
    const double ncn = std::sqrt(gv[0]), nbn = std::sqrt(nb2);
    sc = ncn > 0 ? 1.0 / ncn : 1.0;  // solver.py:659-665
    sb = nbn > 0 ? 1.0 / nbn : 1.0;
  }
  for (int g = 0; g < nshards; ++g) RC(set_data(h, h->sh[g], &descs[g], sc, sb));
  tick("set_data");
  // norms of the iterated data (residual denominators, solver.py:417-423)
  {
    double nci = 0;  // |c|^2 of the iterated (scaled) c over the owners, on the host
    for (int g = 0; g < nshards; ++g) {
      const hsde_problem_desc &dg = descs[g];
      for (int c = 0; c < dg.n_c; ++c) {
        if (dg.owned && !dg.owned[c]) continue;
        const double ci = sc == 1.0 ? dg.c[c] : sc * dg.c[c];
        nci += ci * ci;
      }
    }
    double *red = h->sh[0].W.red;
    for (auto &s : h->sh) CK(cudaMemset(s.W.red, 0, sizeof(double)));
    CK(cudaMemcpy(red, &nci, sizeof(double), cudaMemcpyHostToDevice));
    if (h->mode == MODE_NCCL) {
      RC(reduce(h, BUF_RED, 1));
      CK(cudaMemcpyAsync(&nci, red, sizeof(double), cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
    }
    h->norm_c = std::sqrt(nci);
    double nbi = 0;
    for (int i = 0; i < m; ++i) {
      const double bi = sb == 1.0 ? bsrc[i] : sb * bsrc[i];
      nbi += bi * bi;
    }
    h->norm_b = std::sqrt(nbi);
  }
  tick("norms");
  if (h->factor) {
    RC(setup_schur(h));
    tick("setup_schur");
    RC(compute_minv_zeta(h));
    tick("minv_zeta");
  } else {
    for (auto &s : h->sh) {
      s.P.schur_diag = 1;
      s.P.sinv = s.P.p_inv;  // unused placeholder
      s.P.mz = s.d_zeta;
      s.P.zeta_scale = 1.0;
    }
  }
  RC(init_state(h));
  tick("init_state");
  int maxd = 0;
  for (auto &s : h->sh)
    for (int d : s.sizes) maxd = std::max(maxd, d);
  h->info.total = h->sh[0].P.total;
  h->info.n_c = descs[0].n_c;
  h->info.m = m;
  h->info.p = descs[0].p;
  h->info.n_d = descs[0].n_d;
  h->info.nnz = descs[0].nnz;
  h->info.sigma_c = sc;
  h->info.sigma_b = sb;
  h->info.schur_diagonal = h->schur_diag ? 1 : 0;
  h->info.max_clique = maxd;
  h->info.n_shards = nshards;
  h->info.mode = h->mode;
  h->info.half_passes = 1;
  for (auto &s : h->sh) h->info.half_passes &= s.P.half;
  if (h->factor) {
    // graph of check_interval - 1 iterations: hsde_iterate(check_interval)
    // = one replay + snapshot + the single-iteration graph
    h->gci_len = std::max(1, st->check_interval - 1);
    RC(rebuild_graphs(h));
    tick("graphs");
  }
  return 0;
}

}  // namespace

extern "C" {

const char *hsde_last_error(const hsde_t *h) { return h ? h->err.c_str() : g_create_error.c_str(); }

int hsde_nccl_unique_id(uint8_t *out) {
  if (!out) return HSDE_ERR_ARG;
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    g_create_error = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
    return HSDE_ERR_CUDA;
  }
  memcpy(out, id.internal, HSDE_NCCL_ID_BYTES);
  return HSDE_OK;
}

int hsde_create_sharded(const hsde_problem_desc *descs, int32_t nshards, const hsde_settings *s,
                        const hsde_comm *comm, hsde_t **out) {
  g_create_error.clear();
  if (!descs || !s || !out || nshards < 1) {
    g_create_error = "null argument";
    return HSDE_ERR_ARG;
  }
  *out = nullptr;
  if (!(s->alpha >= 1.0 && s->alpha < 2.0)) {
    g_create_error = "alpha must lie in [1, 2)";
    return HSDE_ERR_ARG;
  }
  hsde_handle *h = new hsde_handle();
  h->set = *s;
  h->dev = s->device;
  h->factor = !(s->flags & HSDE_FLAG_NO_FACTOR);
  h->warm = !(s->flags & HSDE_FLAG_COLD_EIG);
  h->split = !(s->flags & HSDE_FLAG_NO_SPLIT);
  h->jacobi = (s->flags & HSDE_FLAG_JACOBI) != 0;
  h->h_chk = pinned_slot_acquire();
  if (!h->h_chk) {
    g_create_error = "cudaHostAlloc failed";
    delete h;
    return HSDE_ERR_CUDA;
  }
  const int rc = create_impl(descs, nshards, s, comm, h);
  if (rc) {
    g_create_error = h->err;
    hsde_destroy(h);
    return rc;
  }
  *out = h;
  return HSDE_OK;
}

int hsde_create(const hsde_problem_desc *desc, const hsde_settings *settings, hsde_t **out) {
  return hsde_create_sharded(desc, 1, settings, nullptr, out);
}

void hsde_destroy(hsde_t *h) {
  if (!h) return;
  SetupTimer tick;
  cudaSetDevice(h->dev);
  if (h->st) cudaStreamSynchronize(h->st);
  tick("destroy: sync");
  if (h->g1) cudaGraphExecDestroy(h->g1);
  if (h->gci) cudaGraphExecDestroy(h->gci);
  tick("destroy: graphs");
  if (h->nccl) ncclCommDestroy(h->nccl);
  for (void *p : h->bufs) pool_free(h, p);
  if (h->st) cudaStreamSynchronize(h->st);
  tick("destroy: pool frees");
  pinned_slot_release(h->h_chk);
  for (int a = 0; a < hsde_handle::kAux; ++a) {
    if (h->aux[a]) cudaStreamDestroy(h->aux[a]);
    if (h->ev_join[a]) cudaEventDestroy(h->ev_join[a]);
  }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_xjoin) cudaEventDestroy(h->ev_xjoin);
  if (h->st) cudaStreamDestroy(h->st);
  tick("destroy: streams");
  delete h;
}

int hsde_info(const hsde_t *h, hsde_info_t *out) {
  if (!h || !out) return HSDE_ERR_ARG;
  *out = h->info;
  return HSDE_OK;
}

int hsde_shard_total(const hsde_t *h, int32_t g, int64_t *total) {
  if (!h || !total || g < 0 || g >= (int)h->sh.size()) return HSDE_ERR_ARG;
  *total = h->sh[g].P.total;
  return HSDE_OK;
}

int hsde_set_state_shard(hsde_t *h, int32_t g, const double *u, const double *w) {
  if (!h || !u || !w || g < 0 || g >= (int)h->sh.size()) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  ShardDev &s = h->sh[g];
  const int64_t T = s.P.total;
  CK(cudaMemcpyAsync(s.S.u, u, sizeof(double) * T, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(s.S.w, w, sizeof(double) * T, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(s.d_prev_u, s.S.u, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
  CK(cudaMemcpyAsync(s.d_prev_w, s.S.w, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
  CK(cudaMemsetAsync(s.W.vvalid, 0, sizeof(int) * std::max(s.P.p, 1), h->st));
    k_set_i32<<<1, 256, 0, h->st>>>(s.W.cnext, std::max(s.P.p, 1), 1);  // no basis: cold path first
  CK(cudaStreamSynchronize(h->st));
  return HSDE_OK;
}

int hsde_get_state_shard(hsde_t *h, int32_t g, double *u, double *w) {
  if (!h || g < 0 || g >= (int)h->sh.size()) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  ShardDev &s = h->sh[g];
  const int64_t T = s.P.total;
  if (u) CK(cudaMemcpyAsync(u, s.S.u, sizeof(double) * T, cudaMemcpyDeviceToHost, h->st));
  if (w) CK(cudaMemcpyAsync(w, s.S.w, sizeof(double) * T, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return HSDE_OK;
}

// H' vt with vt = (u_v / sigma_c) / tau, one thread per covered coordinate
// summing its slots in ascending order: the reference's unscale, divide and
// np.bincount (solver.py:668-687, 575-585; graphs.py:251) in the same order
__global__ void k_report_hv(DevProblem P, const double *u, double sc, double tau, double *hv) {
  const int64_t vo = P.n_c + P.n_d + P.m;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < P.n_c; l += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int e = P.cov_ptr[l]; e < P.cov_ptr[l + 1]; ++e) {
      const double v = sc == 1.0 ? u[vo + P.cov_slot[e]] : u[vo + P.cov_slot[e]] / sc;
      acc += v / tau;
    }
    hv[l] = acc;
  }
}

int hsde_report_vectors(hsde_t *h, double tau, double *x, double *y, double *hv) {
  if (!h || h->sh.size() != 1 || !(tau > 0.0)) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  ShardDev &s = h->sh[0];
  const DevProblem &P = s.P;
  if (x) CK(cudaMemcpyAsync(x, s.S.u, sizeof(double) * P.n_c, cudaMemcpyDeviceToHost, h->st));
  if (y) CK(cudaMemcpyAsync(y, s.S.u + P.n_c + P.n_d, sizeof(double) * P.m, cudaMemcpyDeviceToHost, h->st));
  if (hv) {
    k_report_hv<<<grid_for(P.n_c), kBlock, 0, h->st>>>(P, s.S.u, h->info.sigma_c, tau, s.d_hv);
    CKL();
    CK(cudaMemcpyAsync(hv, s.d_hv, sizeof(double) * P.n_c, cudaMemcpyDeviceToHost, h->st));
  }
  CK(cudaStreamSynchronize(h->st));
  return HSDE_OK;
}

int hsde_set_state(hsde_t *h, const double *u, const double *w) {
  return hsde_set_state_shard(h, 0, u, w);
}

int hsde_get_state(hsde_t *h, double *u, double *w) { return hsde_get_state_shard(h, 0, u, w); }

int hsde_reset_state(hsde_t *h) {
  if (!h) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  return init_state(h);
}

int hsde_set_alpha(hsde_t *h, double alpha) {
  if (!h || !(alpha >= 1.0 && alpha < 2.0)) return HSDE_ERR_ARG;
  if (alpha == h->sh[0].P.alpha) return HSDE_OK;
  cudaSetDevice(h->dev);
  CK(cudaStreamSynchronize(h->st));
  for (auto &s : h->sh) s.P.alpha = alpha;
  h->set.alpha = alpha;
  return h->factor ? rebuild_graphs(h) : 0;
}

int hsde_iterate(hsde_t *h, int32_t k) {
  if (!h || k < 0 || !h->factor) return HSDE_ERR_ARG;
  if (k == 0) return HSDE_OK;
  cudaSetDevice(h->dev);
  for (auto &s : h->sh) {
    k_prep_ry<<<s.grid_m, kBlock, 0, h->st>>>(s.P, s.S, s.W);
    CKL();
  }
  int left = k - 1;  // the last iteration runs after the snapshot
  while (h->gci && left >= h->gci_len) {
    CK(cudaGraphLaunch(h->gci, h->st));
    left -= h->gci_len;
  }
  while (left > 0) {
    CK(cudaGraphLaunch(h->g1, h->st));
    --left;
  }
  for (auto &s : h->sh) {
    const int64_t T = s.P.total;
    CK(cudaMemcpyAsync(s.d_prev_u, s.S.u, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(s.d_prev_w, s.S.w, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
  }
  CK(cudaGraphLaunch(h->g1, h->st));
  return HSDE_OK;
}

int hsde_sync(hsde_t *h) {
  if (!h) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  CK(cudaStreamSynchronize(h->st));
  return check_err_flag(h);
}

// Residual sums of the stacked states (all shards) into d_chk[0..5]:
// |A xt - b|^2 (lead), |H xt - st|^2, |st|^2, |A' yt + H' vt - c|^2 (owned),
// c.xt (owned), b.yt (lead).  The caller reduces d_chk across shards.
static int residual_sums(hsde_t *h, const std::vector<const double *> &us) {
  cudaStream_t st = h->st;
  const int G = (int)h->sh.size();
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    const DevProblem &P = s.P;
    const int64_t T = P.total;
    const double *u = us[g];
    double *ut = s.d_tmp2;
    k_div_copy<<<s.grid_T, kBlock, 0, st>>>(u, u + T - 1, 1.0, T - 1, ut);  // solver.py:413-416
    CKL();
    const double *xt = ut, *stv = ut + P.n_c, *yt = ut + P.n_c + P.n_d, *vt = yt + P.m;
    k_spmv_seg<<<s.grid_seg, kBlock, 0, st>>>(P, xt, s.d_qseg2);
    CKL();
    k_rowsum_seg<<<s.grid_m, kBlock, 0, st>>>(P, s.d_qseg2, s.W.qbuf);
    CKL();
    double *pa = s.W.part, *pb = s.W.part + 2048;
    k_cons_part<<<s.grid_nd, kBlock, 0, st>>>(P, xt, stv, pa, pb);
    CKL();
    k_sum_parts<<<1, 1024, 0, st>>>(pa, s.grid_nd, s.d_chk + 1);
    k_sum_parts<<<1, 1024, 0, st>>>(pb, s.grid_nd, s.d_chk + 2);
    CKL();
    if (h->n_sep) {
      k_zero<<<grid_for(h->n_sep), kBlock, 0, st>>>(s.W.sepbuf, h->n_sep);
      CKL();
    }
    k_pull<<<s.grid_nc + s.grid_heavy, kBlock, 0, st>>>(P, s.W, vt, s.d_hv, s.grid_nc);
    CKL();
    RC(dev_dot_owned(h, s, P.c, xt, s.d_chk + 4));
    RC(dev_dot(h, s, P.b, yt, P.m, s.d_chk + 5));
    if (!P.lead) CK(cudaMemsetAsync(s.d_chk + 5, 0, sizeof(double), st));
  }
  RC(reduce(h, BUF_Q, h->sh[0].P.m));
  RC(reduce(h, BUF_SEP, h->n_sep));
  for (int g = 0; g < G; ++g) {
    ShardDev &s = h->sh[g];
    const DevProblem &P = s.P;
    const double *yt = s.d_tmp2 + P.n_c + P.n_d;
    if (P.n_sep_local) {
      k_sep_store<<<grid_for(P.n_sep_local), kBlock, 0, st>>>(P, s.W, s.d_hv);
      CKL();
    }
    k_dres_part<<<s.grid_nc, kBlock, 0, st>>>(P, yt, s.d_hv, P.c, s.W.part);
    CKL();
    k_sum_parts<<<1, 1024, 0, st>>>(s.W.part, s.grid_nc, s.d_chk + 3);
    CKL();
    if (P.lead) {
      k_rowres_part<<<s.grid_m, kBlock, 0, st>>>(P, nullptr, s.W.qbuf, P.b, s.W.part);
      CKL();
      k_sum_parts<<<1, 1024, 0, st>>>(s.W.part, s.grid_m, s.d_chk + 0);
      CKL();
    } else {
      CK(cudaMemsetAsync(s.d_chk + 0, 0, sizeof(double), st));
    }
  }
  return 0;
}

static void finish_residuals(const hsde_t *h, const double *v, double *out3) {
  const double pa = std::sqrt(v[0]) / (1.0 + h->norm_b);
  const double pc = std::sqrt(v[1]) / (1.0 + std::sqrt(v[2]));
  const double dres = std::sqrt(v[3]) / (1.0 + h->norm_c);
  const double ctx = v[4], bty = v[5];
  const double gap = std::fabs(ctx - bty) / (1.0 + std::fabs(ctx) + std::fabs(bty));
  out3[0] = std::max(pa, pc);
  out3[1] = dres;
  out3[2] = gap;
}

int hsde_check(hsde_t *h, double *out) {
  if (!h || !out) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  cudaStream_t st = h->st;
  std::vector<const double *> us;
  for (auto &s : h->sh) {
    // merit |u - prev.u| + |w - prev.w| (solver.py:721-723)
    k_merit_part<<<s.grid_T, kBlock, 0, st>>>(s.P, s.S.u, s.d_prev_u, s.W.part);
    CKL();
    k_sum_parts<<<1, 1024, 0, st>>>(s.W.part, s.grid_T, s.d_chk + 10);
    k_merit_part<<<s.grid_T, kBlock, 0, st>>>(s.P, s.S.w, s.d_prev_w, s.W.part);
    CKL();
    k_sum_parts<<<1, 1024, 0, st>>>(s.W.part, s.grid_T, s.d_chk + 11);
    CKL();
    us.push_back(s.S.u);
  }
  RC(residual_sums(h, us));
  RC(reduce(h, BUF_CHK, 12));
  ShardDev &s0 = h->sh[0];
  const int64_t T0 = s0.P.total;
  CK(cudaMemcpyAsync(h->h_chk, s0.d_chk, 12 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h->h_chk + 12, s0.S.u + T0 - 1, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h->h_chk + 13, s0.S.w + T0 - 1, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double *v = h->h_chk;
  const double tau = v[12], kappa = v[13];
  double r3[3];
  if (tau > h->set.infeas_tau_tol) {
    finish_residuals(h, v, r3);
  } else {
    r3[0] = r3[1] = r3[2] = std::numeric_limits<double>::infinity();
  }
  out[0] = r3[0];
  out[1] = r3[1];
  out[2] = r3[2];
  out[3] = tau;
  out[4] = kappa;
  out[5] = std::sqrt(v[10]) + std::sqrt(v[11]);
  out[6] = h->norm_b;
  out[7] = h->norm_c;
  return check_err_flag(h);
}

int hsde_residuals(hsde_t *h, const double *u, double *out3) {
  if (!h || !u || !out3) return HSDE_ERR_ARG;
  if (h->multi()) {
    h->err = "hsde_residuals: single-shard handles only";
    return HSDE_ERR_ARG;
  }
  cudaSetDevice(h->dev);
  ShardDev &s = h->sh[0];
  const int64_t T = s.P.total;
  if (!(u[T - 1] > h->set.infeas_tau_tol)) {
    char buf[64];
    snprintf(buf, sizeof buf, "tau = %g is numerically zero", u[T - 1]);
    h->err = buf;
    return HSDE_ERR_TAUZERO;
  }
  CK(cudaMemcpyAsync(s.d_tmp, u, sizeof(double) * T, cudaMemcpyHostToDevice, h->st));
  std::vector<const double *> us{s.d_tmp};
  RC(residual_sums(h, us));
  CK(cudaMemcpyAsync(h->h_chk, s.d_chk, 16 * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  finish_residuals(h, h->h_chk, out3);
  return HSDE_OK;
}

int hsde_certificate(hsde_t *h, double *out) {
  if (!h || !out) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  cudaStream_t st = h->st;
  const int G = (int)h->sh.size();
  const double nan = std::numeric_limits<double>::quiet_NaN();
  for (int i = 0; i < HSDE_CERT_LEN; ++i) out[i] = nan;
  // unscale (solver.py:668-687): x, s / sigma_b ; y, v / sigma_c ; then b.y, c.x
  for (auto &s : h->sh) {
    const DevProblem &P = s.P;
    double *uu = s.d_tmp;
    k_div_copy<<<s.grid_T, kBlock, 0, st>>>(s.S.u, s.d_consts + 0, 1.0, P.n_c + P.n_d, uu);
    k_div_copy<<<s.grid_T, kBlock, 0, st>>>(s.S.u + P.n_c + P.n_d, s.d_consts + 1, 1.0, P.m + P.n_d,
                                            uu + P.n_c + P.n_d);
    CKL();
    RC(dev_dot(h, s, s.d_b_orig, uu + P.n_c + P.n_d, P.m, s.d_chk + 20));
    if (!P.lead) CK(cudaMemsetAsync(s.d_chk + 20, 0, sizeof(double), st));
    RC(dev_dot_owned(h, s, s.d_c_orig, uu, s.d_chk + 21));
  }
  RC(reduce(h, BUF_CHK, 2, 20));
  CK(cudaMemcpyAsync(h->h_chk, h->sh[0].d_chk + 20, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double by = h->h_chk[0], cx = h->h_chk[1];
  out[0] = by;
  out[1] = cx;
  // min clique eigenvalue over all shards of the stacked blocks
  auto min_eig = [&](const std::vector<const double *> &blocks, double *res) -> int {
    for (int g = 0; g < G; ++g) {
      ShardDev &s = h->sh[g];
      for (const ConePlan &wp : s.warp_plans)
        RC(launch_cone(h, s, CONE_MINEIG, wp, false, blocks[g], s.d_mineig, 1.0, st));
      RC(launch_cone(h, s, CONE_MINEIG, s.block_plan, true, blocks[g], s.d_mineig, 1.0, st));
    }
    double mn = std::numeric_limits<double>::infinity();
    for (auto &s : h->sh) {
      std::vector<double> me(s.P.p);
      if (s.P.p)
        CK(cudaMemcpyAsync(me.data(), s.d_mineig, sizeof(double) * s.P.p, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (double e : me) mn = std::min(mn, e);
    }
    if (h->mode == MODE_NCCL) {
      CK(cudaMemcpyAsync(h->sh[0].d_mineig, &mn, sizeof(double), cudaMemcpyHostToDevice, st));
      RC(reduce(h, BUF_MINEIG, 1, 0, /*min=*/true));
      CK(cudaMemcpyAsync(&mn, h->sh[0].d_mineig, sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    *res = mn;
    return 0;
  };
  if (by > 0) {
    // yt = y / by, vt = v / by ; |A' yt + H' vt| ; min eig of vt blocks
    std::vector<const double *> vts;
    for (auto &s : h->sh) {
      const DevProblem &P = s.P;
      double *y = s.d_tmp + P.n_c + P.n_d, *t2 = s.d_tmp2;
      k_div_copy<<<s.grid_T, kBlock, 0, st>>>(y, s.d_chk + 20, 1.0, P.m + P.n_d, t2);
      CKL();
      if (h->n_sep) {
        k_zero<<<grid_for(h->n_sep), kBlock, 0, st>>>(s.W.sepbuf, h->n_sep);
        CKL();
      }
      k_pull<<<s.grid_nc + s.grid_heavy, kBlock, 0, st>>>(P, s.W, t2 + P.m, s.d_hv, s.grid_nc);
      CKL();
      vts.push_back(t2 + P.m);
    }
    RC(reduce(h, BUF_SEP, h->n_sep));
    for (auto &s : h->sh) {
      const DevProblem &P = s.P;
      if (P.n_sep_local) {
        k_sep_store<<<grid_for(P.n_sep_local), kBlock, 0, st>>>(P, s.W, s.d_hv);
        CKL();
      }
      k_dres_part<<<s.grid_nc, kBlock, 0, st>>>(P, s.d_tmp2, s.d_hv, nullptr, s.W.part);
      CKL();
      k_sum_parts<<<1, 1024, 0, st>>>(s.W.part, s.grid_nc, s.d_chk + 22);
      CKL();
    }
    RC(reduce(h, BUF_CHK, 1, 22));
    double mn;
    RC(min_eig(vts, &mn));
    CK(cudaMemcpyAsync(h->h_chk + 22, h->sh[0].d_chk + 22, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out[2] = std::sqrt(h->h_chk[22]);
    out[3] = mn;
  }
  if (cx < 0) {
    // xt = x / (-cx), st = s / (-cx) ; |A xt| ; |H xt - st| ; min eig of H xt
    std::vector<const double *> hxs;
    for (auto &s : h->sh) {
      const DevProblem &P = s.P;
      double *t2 = s.d_tmp2;
      k_div_copy<<<s.grid_T, kBlock, 0, st>>>(s.d_tmp, s.d_chk + 21, -1.0, P.n_c + P.n_d, t2);
      CKL();
      const double *xt = t2, *stv = t2 + P.n_c;
      k_spmv_seg<<<s.grid_seg, kBlock, 0, st>>>(P, xt, s.d_qseg2);
      k_rowsum_seg<<<s.grid_m, kBlock, 0, st>>>(P, s.d_qseg2, s.W.qbuf);
      CKL();
      double *pa = s.W.part, *pb = s.W.part + 2048;
      k_cons_part<<<s.grid_nd, kBlock, 0, st>>>(P, xt, stv, pa, pb);
      k_sum_parts<<<1, 1024, 0, st>>>(pa, s.grid_nd, s.d_chk + 24);
      CKL();
      double *hx = s.d_tmp3;
      k_gather<<<s.grid_nd, kBlock, 0, st>>>(P, xt, hx);
      CKL();
      hxs.push_back(hx);
    }
    RC(reduce(h, BUF_Q, h->sh[0].P.m));
    for (auto &s : h->sh) {
      const DevProblem &P = s.P;
      if (P.lead) {
        k_rowres_part<<<s.grid_m, kBlock, 0, st>>>(P, nullptr, s.W.qbuf, nullptr, s.W.part);
        k_sum_parts<<<1, 1024, 0, st>>>(s.W.part, s.grid_m, s.d_chk + 23);
        CKL();
      } else {
        CK(cudaMemsetAsync(s.d_chk + 23, 0, sizeof(double), st));
      }
    }
    RC(reduce(h, BUF_CHK, 2, 23));
    double mn;
    RC(min_eig(hxs, &mn));
    CK(cudaMemcpyAsync(h->h_chk + 23, h->sh[0].d_chk + 23, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out[4] = std::sqrt(h->h_chk[23]);
    out[5] = std::sqrt(h->h_chk[24]);
    out[6] = mn;
  }
  return check_err_flag(h);
}

int hsde_affine_project(hsde_t *h, const double *w, double *u) {
  if (!h || !w || !u || !h->factor || h->multi()) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  ShardDev &s = h->sh[0];
  const DevProblem &P = s.P;
  cudaStream_t st = h->st;
  const int64_t T = P.total;
  double *dw = s.d_tmp, *rho = s.d_tmp2, *du = s.d_tmp3;
  CK(cudaMemcpyAsync(dw, w, sizeof(double) * T, cudaMemcpyHostToDevice, st));
  k_rho<<<s.grid_T, kBlock, 0, st>>>(P, dw, rho);  // solver.py:301
  CKL();
  RC(inner_dist(h, {rho}, {du}, true));
  RC(dev_dot(h, s, s.d_zeta, du, T - 1, s.W.scal + S_ZU));             // :315
  k_shift_apply<<<s.grid_T, kBlock, 0, st>>>(P, du, s.W.scal + S_ZU);  // :316
  CKL();
  RC(dev_dot(h, s, s.d_zeta, du, T - 1, s.W.scal + S_UTAU));
  k_tau_out<<<1, 32, 0, st>>>(dw, T, s.W.scal + S_UTAU, du);           // :317
  CKL();
  CK(cudaMemcpyAsync(u, du, sizeof(double) * T, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return HSDE_OK;
}

int hsde_solve_inner(hsde_t *h, const double *w12, double *u12) {
  if (!h || !w12 || !u12 || !h->factor || h->multi()) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  ShardDev &s = h->sh[0];
  const int64_t T = s.P.total;
  CK(cudaMemcpyAsync(s.d_tmp2, w12, sizeof(double) * (T - 1), cudaMemcpyHostToDevice, h->st));
  RC(inner_dist(h, {s.d_tmp2}, {s.d_tmp3}, true));
  CK(cudaMemcpyAsync(u12, s.d_tmp3, sizeof(double) * (T - 1), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return HSDE_OK;
}

int hsde_project_cone(hsde_t *h, const double *in, double *out) {
  if (!h || !in || !out || h->multi()) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  ShardDev &s = h->sh[0];
  const DevProblem &P = s.P;
  const int64_t T = P.total;
  cudaStream_t st = h->st;
  CK(cudaMemcpyAsync(s.d_tmp, in, sizeof(double) * T, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(s.d_tmp2, s.d_tmp, sizeof(double) * T, cudaMemcpyDeviceToDevice, st));
  const double *sin = s.d_tmp + P.n_c;
  double *sout = s.d_tmp2 + P.n_c;
  for (const ConePlan &wp : s.warp_plans) RC(launch_cone(h, s, CONE_PLAIN, wp, false, sin, sout, 1.0, st));
  RC(launch_cone(h, s, CONE_PLAIN, s.block_plan, true, sin, sout, 1.0, st));
  k_tau_clamp<<<1, 32, 0, st>>>(s.d_tmp, T, s.d_tmp2);
  CKL();
  CK(cudaMemcpyAsync(out, s.d_tmp2, sizeof(double) * T, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return check_err_flag(h);
}

int hsde_get_minv_zeta(hsde_t *h, double *out) {
  if (!h || !out || !h->factor) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  CK(cudaMemcpy(out, h->sh[0].P.mz, sizeof(double) * (h->sh[0].P.total - 1), cudaMemcpyDeviceToHost));
  return HSDE_OK;
}

int hsde_time_iterations(hsde_t *h, int32_t k, float *ms) {
  if (!h || !ms || k < 1) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaStreamSynchronize(h->st));
  CK(cudaEventRecord(a, h->st));
  RC(hsde_iterate(h, k));
  CK(cudaEventRecord(b, h->st));
  CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return check_err_flag(h);
}

int hsde_profile_iterations(hsde_t *h, int32_t k, float *ms, int32_t *launches) {
  if (!h || !ms || k < 1) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  // one event set per iteration, one synchronisation at the end: the host
  // runs ahead of the device, so the intervals hold kernel time and not the
  // launch latency an idle device would add after a per-iteration sync
  std::vector<cudaEvent_t> ev((size_t)k * (PS_COUNT + 1));
  for (auto &e : ev) CK(cudaEventCreate(&e));
  for (int i = 0; i < HSDE_PROFILE_SLOTS; ++i) ms[i] = 0.f;
  int nl = 0;
  for (auto &s : h->sh) {
    k_prep_ry<<<s.grid_m, kBlock, 0, h->st>>>(s.P, s.S, s.W);
    CKL();
    ++nl;
  }
  const int order[] = {PS_COUNT, PS_RHS, PS_SPMV, PS_SCHUR, PS_UA, PS_COMM, PS_SCALARS,
                       PS_CONE_WARP, PS_CONE_BLOCK, PS_XUPD};
  for (int it = 0; it < k; ++it) RC(launch_iteration(h, ev.data() + (size_t)it * (PS_COUNT + 1), &nl));
  CK(cudaStreamSynchronize(h->st));
  for (int it = 0; it < k; ++it) {
    cudaEvent_t *e = ev.data() + (size_t)it * (PS_COUNT + 1);
    for (int q = 1; q < 10; ++q) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, e[order[q - 1]], e[order[q]]));
      ms[order[q]] += t;
    }
  }
  for (auto &e : ev) cudaEventDestroy(e);
  if (launches) *launches = nl;
  return check_err_flag(h);
}

int hsde_stats(hsde_t *h, double *out) {
  if (!h || !out) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  double sum = 0, mx = 0, sum_big = 0, n_big = 0, n = 0, n_done = 0, n_hand = 0, n_fp = 0, n_res = 0,
         n_why[4] = {0, 0, 0, 0}, n_cold = 0, n_fail = 0;
  for (auto &s : h->sh) {
    std::vector<int> sw(std::max(s.P.p, 1)), cs(std::max(s.P.p, 1));
    std::vector<int> cf(std::max(s.block_plan.count, 1), 0);
    CK(cudaMemcpyAsync(sw.data(), s.W.sweeps, sizeof(int) * sw.size(), cudaMemcpyDeviceToHost, h->st));
    CK(cudaMemcpyAsync(cs.data(), s.W.cstate, sizeof(int) * cs.size(), cudaMemcpyDeviceToHost, h->st));
    if (s.block_plan.cfail)
      CK(cudaMemcpyAsync(cf.data(), s.block_plan.cfail, sizeof(int) * s.block_plan.count, cudaMemcpyDeviceToHost,
                         h->st));
    CK(cudaStreamSynchronize(h->st));
    const bool split_ran = s.block_plan.split_smem && h->warm && h->split;
    const bool cold_ran = s.block_plan.cold_cv && !h->jacobi;
    for (int i = 0; i < s.block_plan.count; ++i) n_fail += cf[i] != 0;
    for (int k = 0; k < s.P.p; ++k) {
      const bool big = s.in_block[k] != 0;  // CTA team (order > 32, or a small class with few cliques)
      // final states: 0 fast path, 16 fast path after Jacobi sweeps (resumed),
      // 33 cold / Jacobi path (no basis), 34..37 after a hand-over (reason + 34)
      const bool resumed = big && split_ran && cs[k] == SPLIT_DONE + 16;
      const bool fast = big && split_ran && (cs[k] == SPLIT_DONE || resumed);
      n_res += resumed;
      if (big && split_ran) {
        n_done += fast;
        const int why = cs[k] - (SPLIT_DONE + 32 + SPLIT_HANDOFF);
        n_hand += why >= 0 && why <= 3;
        if (why >= 0 && why <= 3) ++n_why[why];
      }
      if (fast) {  // no Jacobi solve; sweeps holds -(fixed-point iterations)
        n_fp -= sw[k];
        continue;
      }
      if (big && cold_ran) {
        n_cold += 1;
        continue;
      }
      sum += sw[k];
      n += 1;
      mx = std::max(mx, (double)sw[k]);
      if (big) {
        sum_big += sw[k];
        n_big += 1;
      }
    }
  }
  int nbig = 0;
  for (auto &s : h->sh)
    for (int k = 0; k < s.P.p; ++k) nbig += s.in_block[k] != 0;
  out[4] = nbig ? n_done / nbig : 0.0;
  out[5] = nbig ? n_hand / nbig : 0.0;
  out[6] = n_done ? n_fp / n_done : 0.0;
  for (int i = 0; i < 3; ++i) out[7 + i] = nbig ? n_why[i] / nbig : 0.0;
  out[10] = nbig ? n_res / nbig : 0.0;
  out[11] = nbig ? n_why[3] / nbig : 0.0;
  out[12] = nbig ? (n_cold - n_fail) / nbig : 0.0;
  out[13] = nbig ? n_fail / nbig : 0.0;
  out[0] = n ? sum / n : 0.0;
  out[1] = mx;
  out[2] = n_big ? sum_big / n_big : 0.0;
  out[3] = h->warm ? 1.0 : 0.0;
  return HSDE_OK;
}

int hsde_debug_jacobi(hsde_t *h, int32_t clique, double *out64) {
  if (!h || !out64) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  ShardDev &s = h->sh[0];
  if (!s.W.dbg) {
    h->err = "hsde_debug_jacobi: diagnostics are off (create the handle with HSDE_DEBUG=1 in the environment)";
    return HSDE_ERR_ARG;
  }
  CK(cudaStreamSynchronize(h->st));
  CK(cudaMemcpy(out64, s.W.dbg, 64 * sizeof(double), cudaMemcpyDeviceToHost));
  CK(cudaMemset(s.W.dbg + 23, 0, sizeof(double)));  // k_cone_split hand-over record counter
  if (clique != s.W.dbg_clique) {
    s.W.dbg_clique = clique;
    if (h->factor) RC(rebuild_graphs(h));
  }
  return HSDE_OK;
}

const char *hsde_profile_name(int32_t slot) {
  if (slot < 0 || slot >= HSDE_PROFILE_SLOTS) return "";
  return kProfNames[slot];
}

}  // extern "C"
