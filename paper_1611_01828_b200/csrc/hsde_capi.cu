// hsde_capi.cu -- C ABI (include/hsde.h) over the sm_100a kernels.
//
// Host responsibilities: validate and derive the device layout once
// (CSC of A, row segments, cover lists, P^{-1}, normalisation), assemble and
// factor the m x m Schur matrix S = I + A P^{-1} A' on the device
// (solver.py:248-283: dense chunks + cuBLAS DGEMM, cuSOLVER Cholesky, explicit
// S^{-1}), solve M zeta with the device inner solve, capture the iteration
// as a CUDA graph, and run the residual / certificate reductions.

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/hsde.h"
#include "hsde_kernels.cuh"

using namespace hsde;

namespace {

std::string g_create_error;

enum ProfSlot {
  PS_PREP = 0, PS_RHS, PS_SPMV, PS_SCHUR, PS_UA, PS_SCALARS, PS_CONE_WARP, PS_CONE_BLOCK,
  PS_XUPD, PS_SNAPSHOT, PS_COUNT
};
const char *kProfNames[HSDE_PROFILE_SLOTS] = {
    "k_prep_ry", "k_rhs", "k_spmv_seg", "k_schur", "k_ua", "k_scalars", "k_cone_warp",
    "k_cone_block", "k_xupd", "snapshot", "", "", "", "", "", ""};

struct ConePlan {
  int *ids = nullptr;
  int count = 0;
  int dpmax = 0;
  size_t smem = 0;
  double *gscratch = nullptr;  // when the scratch exceeds shared memory
  int per_block = 0;           // warps per CTA (warp plan)
};

}  // namespace

struct hsde_handle {
  int dev = 0;
  cudaStream_t st = nullptr;
  hsde_settings set{};
  hsde_info_t info{};
  DevProblem P{};
  DevState S{};
  DevWork W{};
  std::vector<void *> bufs;
  std::string err;
  ConePlan warp_plan, block_plan;
  // extra device buffers
  double *d_zeta = nullptr;       // [T-1] (c, 0, -b, 0) normalised
  double *d_prev_u = nullptr, *d_prev_w = nullptr;
  double *d_tmp = nullptr, *d_tmp2 = nullptr, *d_tmp3 = nullptr;  // [T] scratch
  double *d_qseg2 = nullptr;
  double *d_c_orig = nullptr, *d_b_orig = nullptr;
  double *d_consts = nullptr;     // [0] sigma_b [1] sigma_c [2] 1.0
  double *d_chk = nullptr;        // [64] check sums
  double *d_mineig = nullptr;     // [p]
  double *h_chk = nullptr;        // pinned [64]
  int grid_heavy = 0;
  int grid_nc = 1, grid_nd = 1, grid_m = 1, grid_T = 1, grid_seg = 1, grid_schur = 1;
  size_t schur_smem = 0;
  double norm_b = 0, norm_c = 0;  // of the iterated (normalised) data
  // graphs
  cudaGraphExec_t g1 = nullptr, gci = nullptr;
  int gci_len = 0;
  bool factor = true;
  bool warm = true;               // warm-started eigensolves (HSDE_FLAG_COLD_EIG clears)
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

namespace {

template <class T>
int dalloc(hsde_handle *h, T **p, size_t n) {
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T));
  if (e != cudaSuccess) {
    h->err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
    return HSDE_ERR_CUDA;
  }
  h->bufs.push_back(q);
  *p = static_cast<T *>(q);
  return 0;
}

template <class T>
int dupload(hsde_handle *h, T **p, const T *src, size_t n) {
  int rc = dalloc(h, p, n);
  if (rc) return rc;
  if (n) {
    cudaError_t e = cudaMemcpy(*p, src, n * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      h->err = std::string("cudaMemcpy H2D: ") + cudaGetErrorString(e);
      return HSDE_ERR_CUDA;
    }
  }
  return 0;
}

int grid_for(int64_t n, int cap = 148 * 8) {
  int64_t g = (n + kBlock - 1) / kBlock;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// densify columns [c0, c1) of A (CSC) into Dm (m x w, col-major) and Ds = Dm diag(p_inv)
__global__ void k_densify(DevProblem P, int c0, int c1, double *Dm, double *Ds) {
  const int64_t w = c1 - c0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < w;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int l = c0 + (int)k;
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

// cone launches
int launch_cone(hsde_handle *h, int mode, const ConePlan &pl, bool block, const double *in,
                double *out, double in_scale, cudaStream_t st) {
  if (pl.count == 0) return 0;
  ConeArgs ca{pl.ids, pl.count, pl.dpmax, in, out, in_scale, h->warm ? 1 : 0};
  if (!block) {
    const int grid = (pl.count + pl.per_block - 1) / pl.per_block;
    const int thr = pl.per_block * 32;
    if (mode == CONE_HOT) k_cone_warp<CONE_HOT><<<grid, thr, pl.smem, st>>>(h->P, h->S, h->W, ca);
    else if (mode == CONE_PLAIN) k_cone_warp<CONE_PLAIN><<<grid, thr, pl.smem, st>>>(h->P, h->S, h->W, ca);
    else k_cone_warp<CONE_MINEIG><<<grid, thr, pl.smem, st>>>(h->P, h->S, h->W, ca);
  } else {
    if (mode == CONE_HOT) k_cone_block<CONE_HOT><<<pl.count, kConeBlock, pl.smem, st>>>(h->P, h->S, h->W, ca);
    else if (mode == CONE_PLAIN) k_cone_block<CONE_PLAIN><<<pl.count, kConeBlock, pl.smem, st>>>(h->P, h->S, h->W, ca);
    else k_cone_block<CONE_MINEIG><<<pl.count, kConeBlock, pl.smem, st>>>(h->P, h->S, h->W, ca);
  }
  CKL();
  return 0;
}

// The inner solve of _solve_inner_parts (solver.py:203-245) on explicit vectors:
// rho (T-1, layout x|s|y|v) -> u12 (T-1).  uy by the explicit CSR pass.
int inner_explicit(hsde_handle *h, const double *rho, double *u12, cudaStream_t st) {
  const DevProblem &P = h->P;
  const double *rx = rho, *rs = rho + P.n_c, *ry = rho + P.n_c + P.n_d,
               *rv = rho + P.n_c + P.n_d + P.m;
  k_rhs<false><<<h->grid_nc + h->grid_heavy, kBlock, 0, st>>>(P, h->S, h->W, rx, rs, ry, rv, h->grid_nc);
  CKL();
  k_spmv_seg<<<h->grid_seg, kBlock, 0, st>>>(P, h->W.t, h->W.qseg);
  CKL();
  k_schur<<<h->grid_schur, kBlock, h->schur_smem, st>>>(P, h->W.qseg, h->W.qp);
  CKL();
  k_ua<false><<<h->grid_nc, kBlock, 0, st>>>(P, h->W, h->W.qp);
  CKL();
  double *ua = u12, *ub = u12 + P.n_c, *uy = u12 + P.n_c + P.n_d, *uv = uy + P.m;
  CK(cudaMemcpyAsync(ua, h->W.ua, sizeof(double) * P.n_c, cudaMemcpyDeviceToDevice, st));
  k_slot_out<<<h->grid_nd, kBlock, 0, st>>>(P, rs, rv, ua, ub, uv);
  CKL();
  k_spmv_seg<<<h->grid_seg, kBlock, 0, st>>>(P, ua, h->d_qseg2);
  CKL();
  k_uy_from_seg<<<h->grid_m, kBlock, 0, st>>>(P, h->d_qseg2, ry, uy);
  CKL();
  return 0;
}

// ordered dot of two device vectors into out (device scalar)
int dev_dot(hsde_handle *h, const double *a, const double *b, int64_t n, double *out,
            cudaStream_t st) {
  const int g = grid_for(n);
  k_dot_part<<<g, kBlock, 0, st>>>(a, b, n, h->W.part);
  CKL();
  k_sum_parts<<<1, 1024, 0, st>>>(h->W.part, g, out);
  CKL();
  return 0;
}

// one hot iteration (solver.py:375-395), eager launches; prof events optional
int launch_iteration(hsde_handle *h, cudaStream_t st, cudaEvent_t *ev = nullptr, int *launches = nullptr) {
  const DevProblem &P = h->P;
  int slot = 0;
  auto mark = [&](int s) {
    if (ev) cudaEventRecord(ev[s], st);
    slot = s;
  };
  (void)slot;
  if (ev) cudaEventRecord(ev[PS_COUNT], st);
  k_rhs<true><<<h->grid_nc + h->grid_heavy, kBlock, 0, st>>>(P, h->S, h->W, nullptr, nullptr, nullptr,
                                                             nullptr, h->grid_nc);
  CKL();
  mark(PS_RHS);
  k_spmv_seg<<<h->grid_seg, kBlock, 0, st>>>(P, h->W.t, h->W.qseg);
  CKL();
  mark(PS_SPMV);
  k_schur<<<h->grid_schur, kBlock, h->schur_smem, st>>>(P, h->W.qseg, h->W.qp);
  CKL();
  mark(PS_SCHUR);
  k_ua<true><<<h->grid_nc, kBlock, 0, st>>>(P, h->W, h->W.qp);
  CKL();
  const bool exact = (h->set.flags & HSDE_FLAG_EXACT_UY) != 0;
  if (exact) {
    // uy = rho_y - A ua by an explicit CSR pass (solver.py:240-241)
    k_spmv_seg<<<h->grid_seg, kBlock, 0, st>>>(P, h->W.ua, h->d_qseg2);
    CKL();
    k_rowsum_seg<<<h->grid_m, kBlock, 0, st>>>(P, h->d_qseg2, h->d_tmp3);
    CKL();
  }
  mark(PS_UA);
  k_scalars<<<1, 1024, 0, st>>>(P, h->S, h->W, h->grid_nc, exact ? 1 : 0, h->d_tmp3);
  CKL();
  mark(PS_SCALARS);
  if (launch_cone(h, CONE_HOT, h->warp_plan, false, nullptr, nullptr, 1.0, st)) return HSDE_ERR_CUDA;
  mark(PS_CONE_WARP);
  if (launch_cone(h, CONE_HOT, h->block_plan, true, nullptr, nullptr, 1.0, st)) return HSDE_ERR_CUDA;
  mark(PS_CONE_BLOCK);
  k_xupd<<<h->grid_nc, kBlock, 0, st>>>(P, h->S, h->W);
  CKL();
  mark(PS_XUPD);
  if (launches) *launches += 6 + (h->warp_plan.count > 0) + (h->block_plan.count > 0) + (exact ? 2 : 0);
  return 0;
}

int build_graph(hsde_handle *h, int iters, cudaGraphExec_t *out) {
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
  int rc = 0;
  for (int i = 0; i < iters && !rc; ++i) rc = launch_iteration(h, h->st);
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

int check_err_flag(hsde_handle *h) {
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, h->W.err, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (flag) {
    CK(cudaMemsetAsync(h->W.err, 0, sizeof(int), h->st));
    h->err = "batched eigendecomposition produced non-finite eigenvalues";
    return HSDE_ERR_EIGEN;
  }
  return 0;
}

int setup_cone_plans(hsde_handle *h, const int32_t *sizes, int p) {
  std::vector<int> wids, bids;
  int dpw = 2, dpb = 2;
  for (int k = 0; k < p; ++k) {
    const int d = sizes[k];
    const int dp = d + (d & 1);
    if (d <= 32) {
      wids.push_back(k);
      dpw = std::max(dpw, dp);
    } else {
      bids.push_back(k);
      dpb = std::max(dpb, dp);
    }
  }
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev);
  if (maxsm <= 0) maxsm = 227 * 1024;
  // warp plan
  h->warp_plan.count = (int)wids.size();
  h->warp_plan.dpmax = dpw;
  const size_t per_warp = (size_t)jacobi_scratch_doubles(dpw) * sizeof(double);
  int pb = 8;
  while (pb > 1 && per_warp * pb > (size_t)maxsm) pb >>= 1;
  h->warp_plan.per_block = pb;
  h->warp_plan.smem = per_warp * pb;
  if (!wids.empty()) {
    if (dupload(h, &h->warp_plan.ids, wids.data(), wids.size())) return HSDE_ERR_CUDA;
    CK(cudaFuncSetAttribute(k_cone_warp<CONE_HOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->warp_plan.smem));
    CK(cudaFuncSetAttribute(k_cone_warp<CONE_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->warp_plan.smem));
    CK(cudaFuncSetAttribute(k_cone_warp<CONE_MINEIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->warp_plan.smem));
  }
  h->block_plan.count = (int)bids.size();
  h->block_plan.dpmax = dpb;
  const size_t per_blk = (size_t)jacobi_scratch_doubles(dpb) * sizeof(double);
  if (!bids.empty()) {
    if (per_blk > (size_t)maxsm) {
      h->err = "clique of order " + std::to_string(dpb) + " exceeds the shared-memory Jacobi path";
      return HSDE_ERR_ARG;
    }
    h->block_plan.smem = per_blk;
    if (dupload(h, &h->block_plan.ids, bids.data(), bids.size())) return HSDE_ERR_CUDA;
    CK(cudaFuncSetAttribute(k_cone_block<CONE_HOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per_blk));
    CK(cudaFuncSetAttribute(k_cone_block<CONE_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per_blk));
    CK(cudaFuncSetAttribute(k_cone_block<CONE_MINEIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per_blk));
  }
  return 0;
}

// Dense Schur S = I + A P^{-1} A' (solver.py:250-255) -> S^{-1}
int setup_schur_dense(hsde_handle *h) {
  const int m = h->P.m;
  const int n_c = h->P.n_c;
  double *S = nullptr, *X = nullptr;
  if (dalloc(h, &S, (size_t)m * m)) return HSDE_ERR_CUDA;
  CK(cudaMemsetAsync(S, 0, sizeof(double) * m * m, h->st));
  // chunked dense GEMM
  const size_t budget = 256ull << 20;  // bytes per densified chunk
  int wc = (int)std::max<size_t>(1, budget / (sizeof(double) * (size_t)m));
  wc = std::min(wc, std::max(n_c, 1));
  double *Dm = nullptr, *Ds = nullptr;
  CK(cudaMalloc(&Dm, sizeof(double) * (size_t)m * wc));
  CK(cudaMalloc(&Ds, sizeof(double) * (size_t)m * wc));
  cublasHandle_t cb;
  if (cublasCreate(&cb) != CUBLAS_STATUS_SUCCESS) {
    h->err = "cublasCreate failed";
    return HSDE_ERR_CUDA;
  }
  cublasSetStream(cb, h->st);
  const double one = 1.0;
  for (int c0 = 0; c0 < n_c; c0 += wc) {
    const int c1 = std::min(n_c, c0 + wc);
    const int w = c1 - c0;
    CK(cudaMemsetAsync(Dm, 0, sizeof(double) * (size_t)m * w, h->st));
    CK(cudaMemsetAsync(Ds, 0, sizeof(double) * (size_t)m * w, h->st));
    k_densify<<<grid_for(w), kBlock, 0, h->st>>>(h->P, c0, c1, Dm, Ds);
    CKL();
    // S += Ds * Dm'
    if (cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_T, m, m, w, &one, Ds, m, Dm, m, &one, S, m) !=
        CUBLAS_STATUS_SUCCESS) {
      h->err = "cublasDgemm failed";
      cublasDestroy(cb);
      return HSDE_ERR_CUDA;
    }
  }
  cublasDestroy(cb);
  k_add_identity<<<grid_for(m), kBlock, 0, h->st>>>(S, m);
  CKL();
  CK(cudaStreamSynchronize(h->st));
  cudaFree(Dm);
  cudaFree(Ds);
  // finite check (cho_factor on non-finite data fails: solver.py:254-259)
  k_finite_check<<<grid_for((int64_t)m * m), kBlock, 0, h->st>>>(S, (int64_t)m * m, h->W.err);
  CKL();
  int flag = 0;
  CK(cudaMemcpy(&flag, h->W.err, sizeof(int), cudaMemcpyDeviceToHost));
  if (flag) {
    CK(cudaMemset(h->W.err, 0, sizeof(int)));
    h->err = "Cholesky of the " + std::to_string(m) + " x " + std::to_string(m) +
             " reduced system failed: non-finite entries";
    return HSDE_ERR_FACTOR;
  }
  // Cholesky (lower) and explicit inverse via potrs on the identity
  cusolverDnHandle_t cs;
  if (cusolverDnCreate(&cs) != CUSOLVER_STATUS_SUCCESS) {
    h->err = "cusolverDnCreate failed";
    return HSDE_ERR_CUDA;
  }
  cusolverDnSetStream(cs, h->st);
  int lwork = 0;
  cusolverDnDpotrf_bufferSize(cs, CUBLAS_FILL_MODE_LOWER, m, S, m, &lwork);
  double *work = nullptr;
  int *dinfo = nullptr;
  CK(cudaMalloc(&work, sizeof(double) * std::max(lwork, 1)));
  CK(cudaMalloc(&dinfo, sizeof(int)));
  cusolverDnDpotrf(cs, CUBLAS_FILL_MODE_LOWER, m, S, m, work, lwork, dinfo);
  int info = 0;
  CK(cudaMemcpyAsync(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (info != 0) {
    cudaFree(work);
    cudaFree(dinfo);
    cusolverDnDestroy(cs);
    h->err = "Cholesky of the " + std::to_string(m) + " x " + std::to_string(m) +
             " reduced system failed: leading minor " + std::to_string(info) + " not positive";
    return HSDE_ERR_FACTOR;
  }
  if (dalloc(h, &X, (size_t)m * m)) return HSDE_ERR_CUDA;
  k_identity<<<grid_for((int64_t)m * m), kBlock, 0, h->st>>>(X, m);
  CKL();
  cusolverDnDpotrs(cs, CUBLAS_FILL_MODE_LOWER, m, m, S, m, X, m, dinfo);
  CK(cudaStreamSynchronize(h->st));
  cudaFree(work);
  cudaFree(dinfo);
  cusolverDnDestroy(cs);
  // S^{-1} symmetrised, row-major == col-major
  k_symmetrize<<<grid_for((int64_t)m * m), kBlock, 0, h->st>>>(X, m, S);
  CKL();
  h->P.sinv = S;
  h->P.schur_diag = 0;
  return 0;
}

int compute_minv_zeta(hsde_handle *h) {
  const DevProblem &P = h->P;
  double *mz = nullptr;
  if (dalloc(h, &mz, (size_t)(P.total - 1))) return HSDE_ERR_CUDA;
  int rc = inner_explicit(h, h->d_zeta, mz, h->st);
  if (rc) return rc;
  h->P.mz = mz;
  rc = dev_dot(h, h->d_zeta, mz, P.total - 1, h->d_chk, h->st);
  if (rc) return rc;
  double zmz = 0;
  CK(cudaMemcpyAsync(&zmz, h->d_chk, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  const double zs = 1.0 + zmz;  // solver.py:269
  if (!(zs > 0)) {
    char buf[128];
    snprintf(buf, sizeof buf, "rank-one update scale %g is not positive; data is ill-scaled", zs);
    h->err = buf;
    return HSDE_ERR_FACTOR;
  }
  h->P.zmz = zmz;
  h->P.zeta_scale = zs;
  h->info.zeta_scale = zs;
  return 0;
}

int init_state(hsde_handle *h) {
  const int64_t T = h->P.total;
  CK(cudaMemsetAsync(h->S.u, 0, sizeof(double) * T, h->st));
  CK(cudaMemsetAsync(h->S.w, 0, sizeof(double) * T, h->st));
  const double one = 1.0;
  CK(cudaMemcpyAsync(h->S.u + T - 1, &one, sizeof(double), cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->S.w + T - 1, &one, sizeof(double), cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->d_prev_u, h->S.u, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
  CK(cudaMemcpyAsync(h->d_prev_w, h->S.w, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
  CK(cudaMemsetAsync(h->W.vvalid, 0, sizeof(int) * std::max(h->P.p, 1), h->st));
  CK(cudaStreamSynchronize(h->st));
  return 0;
}

}  // namespace

extern "C" {

const char *hsde_last_error(const hsde_t *h) { return h ? h->err.c_str() : g_create_error.c_str(); }

int hsde_create(const hsde_problem_desc *d, const hsde_settings *s, hsde_t **out) {
  g_create_error.clear();
  if (!d || !s || !out) {
    g_create_error = "null argument";
    return HSDE_ERR_ARG;
  }
  *out = nullptr;
  if (d->m < 0 || d->n_c < 0 || d->p < 0 || d->n_d < 0 || d->nnz < 0) {
    g_create_error = "negative dimension";
    return HSDE_ERR_ARG;
  }
  if (!(s->alpha >= 1.0 && s->alpha < 2.0)) {
    g_create_error = "alpha must lie in [1, 2)";
    return HSDE_ERR_ARG;
  }
  hsde_handle *h = new hsde_handle();
  h->set = *s;
  h->dev = s->device;
  h->factor = !(s->flags & HSDE_FLAG_NO_FACTOR);
  h->warm = !(s->flags & HSDE_FLAG_COLD_EIG);
  auto fail = [&](int rc) {
    g_create_error = h->err;
    hsde_destroy(h);
    return rc;
  };
  cudaError_t e = cudaSetDevice(h->dev);
  if (e != cudaSuccess) {
    h->err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
    return fail(HSDE_ERR_CUDA);
  }
  if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess) {
    h->err = "stream create failed";
    return fail(HSDE_ERR_CUDA);
  }
  const int m = d->m, n_c = d->n_c, p = d->p;
  const int64_t n_d = d->n_d, nnz = d->nnz;
  // ---- validate
  if (d->a_row_ptr[0] != 0 || d->a_row_ptr[m] != nnz) {
    h->err = "a_row_ptr inconsistent with nnz";
    return fail(HSDE_ERR_ARG);
  }
  for (int i = 0; i < m; ++i) {
    if (d->a_row_ptr[i + 1] < d->a_row_ptr[i]) {
      h->err = "a_row_ptr not monotone";
      return fail(HSDE_ERR_ARG);
    }
    for (int64_t k = d->a_row_ptr[i]; k < d->a_row_ptr[i + 1]; ++k) {
      const int c = d->a_col[k];
      if (c < 0 || c >= n_c || (k > d->a_row_ptr[i] && c <= d->a_col[k - 1])) {
        h->err = "a_col out of range or not strictly ascending in row " + std::to_string(i);
        return fail(HSDE_ERR_ARG);
      }
    }
  }
  if (d->clique_offsets[0] != 0 || d->clique_offsets[p] != n_d) {
    h->err = "clique offsets inconsistent with n_d";
    return fail(HSDE_ERR_ARG);
  }
  int maxd = 0;
  for (int k = 0; k < p; ++k) {
    const int64_t dk = d->clique_sizes[k];
    if (dk < 1 || d->clique_offsets[k + 1] - d->clique_offsets[k] != dk * dk) {
      h->err = "clique size / offset mismatch at clique " + std::to_string(k);
      return fail(HSDE_ERR_ARG);
    }
    maxd = std::max<int>(maxd, (int)dk);
  }
  for (int64_t j = 0; j < n_d; ++j)
    if (d->slot_cov[j] < 0 || d->slot_cov[j] >= n_c) {
      h->err = "slot_cov out of range";
      return fail(HSDE_ERR_ARG);
    }
  // ---- derived host structures
  // CSC (transpose) by counting sort; rows ascending within a column
  std::vector<int64_t> at_cp(n_c + 1, 0);
  for (int64_t k = 0; k < nnz; ++k) at_cp[d->a_col[k] + 1]++;
  for (int c = 0; c < n_c; ++c) at_cp[c + 1] += at_cp[c];
  std::vector<int> at_row(nnz);
  std::vector<double> at_val(nnz);
  {
    std::vector<int64_t> pos(at_cp.begin(), at_cp.end() - 1);
    for (int i = 0; i < m; ++i)
      for (int64_t k = d->a_row_ptr[i]; k < d->a_row_ptr[i + 1]; ++k) {
        const int64_t q = pos[d->a_col[k]]++;
        at_row[q] = i;
        at_val[q] = d->a_val[k];
      }
  }
  int64_t maxcol = 0;
  for (int c = 0; c < n_c; ++c) maxcol = std::max(maxcol, at_cp[c + 1] - at_cp[c]);
  // row segments
  std::vector<int> seg_row, row_seg(m + 1, 0);
  std::vector<int64_t> seg_beg;
  for (int i = 0; i < m; ++i) {
    row_seg[i] = (int)seg_row.size();
    for (int64_t k = d->a_row_ptr[i]; k < d->a_row_ptr[i + 1]; k += kSegNnz) {
      seg_row.push_back(i);
      seg_beg.push_back(k);
    }
  }
  row_seg[m] = (int)seg_row.size();
  // cover lists (stable by slot) and cover counts D
  std::vector<int> cov_ptr(n_c + 1, 0), cov_slot(n_d);
  for (int64_t j = 0; j < n_d; ++j) cov_ptr[d->slot_cov[j] + 1]++;
  for (int c = 0; c < n_c; ++c) cov_ptr[c + 1] += cov_ptr[c];
  {
    std::vector<int> pos(cov_ptr.begin(), cov_ptr.end() - 1);
    for (int64_t j = 0; j < n_d; ++j) cov_slot[pos[d->slot_cov[j]]++] = (int)j;
  }
  std::vector<int> heavy;
  for (int c = 0; c < n_c; ++c)
    if (cov_ptr[c + 1] - cov_ptr[c] > kHeavy) heavy.push_back(c);
  std::vector<double> p_inv(n_c);
  for (int c = 0; c < n_c; ++c)
    p_inv[c] = 1.0 / (1.0 + 0.5 * (double)(cov_ptr[c + 1] - cov_ptr[c]));  // solver.py:250
  // normalisation (solver.py:659-665)
  double nc2 = 0, nb2 = 0;
  for (int c = 0; c < n_c; ++c) nc2 += d->c[c] * d->c[c];
  for (int i = 0; i < m; ++i) nb2 += d->b[i] * d->b[i];
  double sc = 1.0, sb = 1.0;
  if (s->normalize) {
    const double ncn = std::sqrt(nc2), nbn = std::sqrt(nb2);
    sc = ncn > 0 ? 1.0 / ncn : 1.0;
    sb = nbn > 0 ? 1.0 / nbn : 1.0;
  }
  std::vector<double> cint(n_c), bint(m);
  for (int c = 0; c < n_c; ++c) cint[c] = sc == 1.0 ? d->c[c] : sc * d->c[c];
  for (int i = 0; i < m; ++i) bint[i] = sb == 1.0 ? d->b[i] : sb * d->b[i];
  double nci = 0, nbi = 0;
  for (int c = 0; c < n_c; ++c) nci += cint[c] * cint[c];
  for (int i = 0; i < m; ++i) nbi += bint[i] * bint[i];
  h->norm_c = std::sqrt(nci);
  h->norm_b = std::sqrt(nbi);
  // diagonal Schur detection: no two rows share a column
  const bool sdiag = maxcol <= 1;
  // ---- device problem
  DevProblem &P = h->P;
  P.m = m;
  P.n_c = n_c;
  P.p = p;
  P.n_d = n_d;
  P.nnz = nnz;
  P.total = (int64_t)n_c + 2 * n_d + m + 1;
  P.alpha = s->alpha;
  P.nseg = (int)seg_row.size();
  int rc = 0;
  int64_t *a_rp = nullptr, *at_cp_d = nullptr, *seg_beg_d = nullptr, *cl_off = nullptr;
  int *a_col = nullptr, *at_row_d = nullptr, *seg_row_d = nullptr, *row_seg_d = nullptr;
  int *cov_ptr_d = nullptr, *cov_slot_d = nullptr, *slot_cov_d = nullptr, *cl_size = nullptr;
  double *a_val = nullptr, *at_val_d = nullptr, *c_d = nullptr, *b_d = nullptr, *pinv_d = nullptr;
  if ((rc = dupload(h, &a_rp, d->a_row_ptr, m + 1)) || (rc = dupload(h, &a_col, d->a_col, nnz)) ||
      (rc = dupload(h, &a_val, d->a_val, nnz)) || (rc = dupload(h, &at_cp_d, at_cp.data(), n_c + 1)) ||
      (rc = dupload(h, &at_row_d, at_row.data(), nnz)) || (rc = dupload(h, &at_val_d, at_val.data(), nnz)) ||
      (rc = dupload(h, &seg_row_d, seg_row.data(), seg_row.size())) ||
      (rc = dupload(h, &seg_beg_d, seg_beg.data(), seg_beg.size())) ||
      (rc = dupload(h, &row_seg_d, row_seg.data(), m + 1)) ||
      (rc = dupload(h, &cov_ptr_d, cov_ptr.data(), n_c + 1)) ||
      (rc = dupload(h, &cov_slot_d, cov_slot.data(), n_d)) ||
      (rc = dupload(h, &slot_cov_d, d->slot_cov, n_d)) ||
      (rc = dupload(h, &cl_off, d->clique_offsets, p + 1)) ||
      (rc = dupload(h, &cl_size, d->clique_sizes, p)) || (rc = dupload(h, &c_d, cint.data(), n_c)) ||
      (rc = dupload(h, &b_d, bint.data(), m)) || (rc = dupload(h, &pinv_d, p_inv.data(), n_c)) ||
      (rc = dupload(h, &h->d_c_orig, d->c, n_c)) || (rc = dupload(h, &h->d_b_orig, d->b, m)))
    return fail(rc);
  int *heavy_d = nullptr;
  if ((rc = dupload(h, &heavy_d, heavy.data(), heavy.size()))) return fail(rc);
  P.heavy = heavy_d;
  P.n_heavy = (int)heavy.size();
  h->grid_heavy = (P.n_heavy + (kBlock / 32) - 1) / (kBlock / 32);
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
  P.c = c_d;
  P.b = b_d;
  P.p_inv = pinv_d;
  const double consts[4] = {sb, sc, 1.0, 0.0};
  if ((rc = dupload(h, &h->d_consts, consts, 4))) return fail(rc);
  // zeta (solver.py:264)
  {
    std::vector<double> z(P.total - 1, 0.0);
    for (int c = 0; c < n_c; ++c) z[c] = cint[c];
    for (int i = 0; i < m; ++i) z[n_c + n_d + i] = -bint[i];
    if ((rc = dupload(h, &h->d_zeta, z.data(), z.size()))) return fail(rc);
  }
  // state + work
  const int64_t T = P.total;
  if ((rc = dalloc(h, &h->S.u, T)) || (rc = dalloc(h, &h->S.w, T)) ||
      (rc = dalloc(h, &h->d_prev_u, T)) || (rc = dalloc(h, &h->d_prev_w, T)) ||
      (rc = dalloc(h, &h->d_tmp, T)) || (rc = dalloc(h, &h->d_tmp2, T)) ||
      (rc = dalloc(h, &h->d_tmp3, T)) || (rc = dalloc(h, &h->W.t, n_c)) ||
      (rc = dalloc(h, &h->W.ua, n_c)) || (rc = dalloc(h, &h->W.ry, m)) ||
      (rc = dalloc(h, &h->W.qseg, P.nseg)) || (rc = dalloc(h, &h->d_qseg2, P.nseg)) ||
      (rc = dalloc(h, &h->W.qp, m)) || (rc = dalloc(h, &h->W.uy, m)) ||
      (rc = dalloc(h, &h->W.part, kMaxParts)) || (rc = dalloc(h, &h->W.scal, S_COUNT)) ||
      (rc = dalloc(h, &h->W.err, 1)) || (rc = dalloc(h, &h->d_chk, 64)) ||
      (rc = dalloc(h, &h->d_mineig, std::max(p, 1))) || (rc = dalloc(h, &h->W.vstore, n_d)) ||
      (rc = dalloc(h, &h->W.vvalid, std::max(p, 1))) || (rc = dalloc(h, &h->W.sweeps, std::max(p, 1))))
    return fail(rc);
  if (cudaMemset(h->W.vvalid, 0, sizeof(int) * std::max(p, 1)) != cudaSuccess ||
      cudaMemset(h->W.sweeps, 0, sizeof(int) * std::max(p, 1)) != cudaSuccess)
    return fail(HSDE_ERR_CUDA);
  if (cudaMemset(h->W.err, 0, sizeof(int)) != cudaSuccess) return fail(HSDE_ERR_CUDA);
  if (cudaMallocHost(&h->h_chk, 64 * sizeof(double)) != cudaSuccess) {
    h->err = "cudaMallocHost failed";
    return fail(HSDE_ERR_CUDA);
  }
  h->grid_nc = grid_for(n_c);
  h->grid_nd = grid_for(n_d);
  h->grid_m = grid_for(m);
  h->grid_T = grid_for(T);
  h->grid_seg = std::max(1, (int)((P.nseg * 32LL + kBlock - 1) / kBlock));
  h->schur_smem = sizeof(double) * std::max(m, 1);
  h->grid_schur = sdiag ? grid_for(m, 64) : std::min(148 * 2, std::max(1, (m + 7) / 8));
  if (h->schur_smem > 48 * 1024) {
    if (cudaFuncSetAttribute(k_schur, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)h->schur_smem) != cudaSuccess) {
      h->err = "m too large for the shared-memory Schur apply";
      return fail(HSDE_ERR_ARG);
    }
  }
  if ((rc = setup_cone_plans(h, d->clique_sizes, p))) return fail(rc);
  // ---- Schur complement (solver.py:250-255)
  if (h->factor) {
    if (sdiag) {
      std::vector<double> sinv(m);
      for (int i = 0; i < m; ++i) {
        double sii = 0.0;
        for (int64_t k = d->a_row_ptr[i]; k < d->a_row_ptr[i + 1]; ++k)
          sii += (d->a_val[k] * p_inv[d->a_col[k]]) * d->a_val[k];
        sii += 1.0;
        if (!(sii > 0) || !std::isfinite(sii)) {
          h->err = "Cholesky of the " + std::to_string(m) + " x " + std::to_string(m) +
                   " reduced system failed: diagonal entry not positive";
          return fail(HSDE_ERR_FACTOR);
        }
        sinv[i] = 1.0 / sii;
      }
      double *sinv_d = nullptr;
      if ((rc = dupload(h, &sinv_d, sinv.data(), m))) return fail(rc);
      P.sinv = sinv_d;
      P.schur_diag = 1;
    } else if ((rc = setup_schur_dense(h))) {
      return fail(rc);
    }
    if ((rc = compute_minv_zeta(h))) return fail(rc);
  } else {
    P.schur_diag = 1;
    P.sinv = pinv_d;  // unused placeholder
    P.mz = h->d_zeta;
    P.zeta_scale = 1.0;
  }
  if ((rc = init_state(h))) return fail(rc);
  // info
  h->info.total = T;
  h->info.n_c = n_c;
  h->info.m = m;
  h->info.p = p;
  h->info.n_d = n_d;
  h->info.nnz = nnz;
  h->info.sigma_c = sc;
  h->info.sigma_b = sb;
  h->info.schur_diagonal = sdiag ? 1 : 0;
  h->info.max_clique = maxd;
  if (h->factor) {
    if ((rc = build_graph(h, 1, &h->g1))) return fail(rc);
    // graph of check_interval - 1 iterations: hsde_iterate(check_interval)
    // = one replay + snapshot + the single-iteration graph
    h->gci_len = std::max(1, s->check_interval - 1);
    if (h->gci_len > 1 && (rc = build_graph(h, h->gci_len, &h->gci))) return fail(rc);
  }
  *out = h;
  return HSDE_OK;
}

void hsde_destroy(hsde_t *h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  if (h->st) cudaStreamSynchronize(h->st);
  if (h->g1) cudaGraphExecDestroy(h->g1);
  if (h->gci) cudaGraphExecDestroy(h->gci);
  for (void *p : h->bufs) cudaFree(p);
  if (h->h_chk) cudaFreeHost(h->h_chk);
  if (h->st) cudaStreamDestroy(h->st);
  delete h;
}

int hsde_info(const hsde_t *h, hsde_info_t *out) {
  if (!h || !out) return HSDE_ERR_ARG;
  *out = h->info;
  return HSDE_OK;
}

int hsde_set_state(hsde_t *h, const double *u, const double *w) {
  if (!h || !u || !w) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  const int64_t T = h->P.total;
  CK(cudaMemcpyAsync(h->S.u, u, sizeof(double) * T, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->S.w, w, sizeof(double) * T, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->d_prev_u, h->S.u, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
  CK(cudaMemcpyAsync(h->d_prev_w, h->S.w, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
  CK(cudaMemsetAsync(h->W.vvalid, 0, sizeof(int) * std::max(h->P.p, 1), h->st));
  CK(cudaStreamSynchronize(h->st));
  return HSDE_OK;
}

int hsde_get_state(hsde_t *h, double *u, double *w) {
  if (!h) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  const int64_t T = h->P.total;
  if (u) CK(cudaMemcpyAsync(u, h->S.u, sizeof(double) * T, cudaMemcpyDeviceToHost, h->st));
  if (w) CK(cudaMemcpyAsync(w, h->S.w, sizeof(double) * T, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return HSDE_OK;
}

int hsde_reset_state(hsde_t *h) {
  if (!h) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  return init_state(h);
}

int hsde_set_alpha(hsde_t *h, double alpha) {
  if (!h || !(alpha >= 1.0 && alpha < 2.0)) return HSDE_ERR_ARG;
  if (alpha == h->P.alpha) return HSDE_OK;
  cudaSetDevice(h->dev);
  CK(cudaStreamSynchronize(h->st));
  h->P.alpha = alpha;
  h->set.alpha = alpha;
  if (h->g1) cudaGraphExecDestroy(h->g1);
  if (h->gci) cudaGraphExecDestroy(h->gci);
  h->g1 = h->gci = nullptr;
  int rc = build_graph(h, 1, &h->g1);
  if (!rc && h->gci_len > 1) rc = build_graph(h, h->gci_len, &h->gci);
  return rc;
}

int hsde_iterate(hsde_t *h, int32_t k) {
  if (!h || k < 0 || !h->factor) return HSDE_ERR_ARG;
  if (k == 0) return HSDE_OK;
  cudaSetDevice(h->dev);
  const int64_t T = h->P.total;
  k_prep_ry<<<h->grid_m, kBlock, 0, h->st>>>(h->P, h->S, h->W);
  CKL();
  int left = k - 1;  // the last iteration runs after the snapshot
  while (h->gci && left >= h->gci_len) {
    CK(cudaGraphLaunch(h->gci, h->st));
    left -= h->gci_len;
  }
  while (left > 0) {
    CK(cudaGraphLaunch(h->g1, h->st));
    --left;
  }
  CK(cudaMemcpyAsync(h->d_prev_u, h->S.u, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
  CK(cudaMemcpyAsync(h->d_prev_w, h->S.w, sizeof(double) * T, cudaMemcpyDeviceToDevice, h->st));
  CK(cudaGraphLaunch(h->g1, h->st));
  return HSDE_OK;
}

int hsde_sync(hsde_t *h) {
  if (!h) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  CK(cudaStreamSynchronize(h->st));
  return check_err_flag(h);
}

// residual sums of a stacked vector `u` (device) into d_chk[base..base+6]:
// |A xt - b|^2, |H xt - st|^2, |st|^2, |A' yt + H' vt - c|^2, c.xt, b.yt
static int residual_sums(hsde_t *h, const double *u, int base) {
  const DevProblem &P = h->P;
  cudaStream_t st = h->st;
  const int64_t T = P.total;
  double *ut = h->d_tmp2;
  // tilde = u / tau (solver.py:413-416)
  k_div_copy<<<h->grid_T, kBlock, 0, st>>>(u, u + T - 1, 1.0, T - 1, ut);
  CKL();
  const double *xt = ut, *stv = ut + P.n_c, *yt = ut + P.n_c + P.n_d, *vt = yt + P.m;
  double *chk = h->d_chk + base;
  k_spmv_seg<<<h->grid_seg, kBlock, 0, st>>>(P, xt, h->d_qseg2);
  CKL();
  k_rowres_part<<<h->grid_m, kBlock, 0, st>>>(P, h->d_qseg2, P.b, h->W.part);
  CKL();
  k_sum_parts<<<1, 1024, 0, st>>>(h->W.part, h->grid_m, chk + 0);
  CKL();
  double *pa = h->W.part, *pb = h->W.part + 2048;
  k_cons_part<<<h->grid_nd, kBlock, 0, st>>>(P, xt, stv, pa, pb);
  CKL();
  k_sum_parts<<<1, 1024, 0, st>>>(pa, h->grid_nd, chk + 1);
  k_sum_parts<<<1, 1024, 0, st>>>(pb, h->grid_nd, chk + 2);
  CKL();
  k_dres_part<<<h->grid_nc, kBlock, 0, st>>>(P, yt, vt, P.c, h->W.part);
  CKL();
  k_sum_parts<<<1, 1024, 0, st>>>(h->W.part, h->grid_nc, chk + 3);
  CKL();
  if (dev_dot(h, P.c, xt, P.n_c, chk + 4, st)) return HSDE_ERR_CUDA;
  if (dev_dot(h, P.b, yt, P.m, chk + 5, st)) return HSDE_ERR_CUDA;
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
  const DevProblem &P = h->P;
  const int64_t T = P.total;
  cudaStream_t st = h->st;
  // merit |u - prev.u| + |w - prev.w| (solver.py:721-723)
  k_diff2_part<<<h->grid_T, kBlock, 0, st>>>(h->S.u, h->d_prev_u, T, h->W.part);
  CKL();
  k_sum_parts<<<1, 1024, 0, st>>>(h->W.part, h->grid_T, h->d_chk + 10);
  k_diff2_part<<<h->grid_T, kBlock, 0, st>>>(h->S.w, h->d_prev_w, T, h->W.part);
  CKL();
  k_sum_parts<<<1, 1024, 0, st>>>(h->W.part, h->grid_T, h->d_chk + 11);
  CK(cudaMemcpyAsync(h->d_chk + 12, h->S.u + T - 1, sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(h->d_chk + 13, h->S.w + T - 1, sizeof(double), cudaMemcpyDeviceToDevice, st));
  int rc = residual_sums(h, h->S.u, 0);
  if (rc) return rc;
  CK(cudaMemcpyAsync(h->h_chk, h->d_chk, 16 * sizeof(double), cudaMemcpyDeviceToHost, st));
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
  cudaSetDevice(h->dev);
  const int64_t T = h->P.total;
  if (!(u[T - 1] > h->set.infeas_tau_tol)) {
    char buf[64];
    snprintf(buf, sizeof buf, "tau = %g is numerically zero", u[T - 1]);
    h->err = buf;
    return HSDE_ERR_TAUZERO;
  }
  CK(cudaMemcpyAsync(h->d_tmp, u, sizeof(double) * T, cudaMemcpyHostToDevice, h->st));
  int rc = residual_sums(h, h->d_tmp, 0);
  if (rc) return rc;
  CK(cudaMemcpyAsync(h->h_chk, h->d_chk, 16 * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  finish_residuals(h, h->h_chk, out3);
  return HSDE_OK;
}

int hsde_certificate(hsde_t *h, double *out) {
  if (!h || !out) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  const DevProblem &P = h->P;
  cudaStream_t st = h->st;
  const int64_t T = P.total;
  const double nan = std::numeric_limits<double>::quiet_NaN();
  for (int i = 0; i < HSDE_CERT_LEN; ++i) out[i] = nan;
  // unscale (solver.py:668-687): x, s / sigma_b ; y, v / sigma_c
  double *uu = h->d_tmp;
  k_div_copy<<<h->grid_T, kBlock, 0, st>>>(h->S.u, h->d_consts + 0, 1.0, P.n_c + P.n_d, uu);
  k_div_copy<<<h->grid_T, kBlock, 0, st>>>(h->S.u + P.n_c + P.n_d, h->d_consts + 1, 1.0,
                                            P.m + P.n_d, uu + P.n_c + P.n_d);
  CKL();
  const double *x = uu, *y = uu + P.n_c + P.n_d;
  if (dev_dot(h, h->d_b_orig, y, P.m, h->d_chk + 20, st)) return HSDE_ERR_CUDA;
  if (dev_dot(h, h->d_c_orig, x, P.n_c, h->d_chk + 21, st)) return HSDE_ERR_CUDA;
  CK(cudaMemcpyAsync(h->h_chk, h->d_chk + 20, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double by = h->h_chk[0], cx = h->h_chk[1];
  out[0] = by;
  out[1] = cx;
  double *t2 = h->d_tmp2;
  if (by > 0) {
    // yt = y / by, vt = v / by ; |A' yt + H' vt| ; min eig of vt blocks
    k_div_copy<<<h->grid_T, kBlock, 0, st>>>(y, h->d_chk + 20, 1.0, P.m + P.n_d, t2);
    CKL();
    const double *yt = t2, *vt = t2 + P.m;
    k_dres_part<<<h->grid_nc, kBlock, 0, st>>>(P, yt, vt, nullptr, h->W.part);
    CKL();
    k_sum_parts<<<1, 1024, 0, st>>>(h->W.part, h->grid_nc, h->d_chk + 22);
    CKL();
    if (launch_cone(h, CONE_MINEIG, h->warp_plan, false, vt, h->d_mineig, 1.0, st)) return HSDE_ERR_CUDA;
    if (launch_cone(h, CONE_MINEIG, h->block_plan, true, vt, h->d_mineig, 1.0, st)) return HSDE_ERR_CUDA;
    std::vector<double> me(P.p);
    CK(cudaMemcpyAsync(h->h_chk + 22, h->d_chk + 22, sizeof(double), cudaMemcpyDeviceToHost, st));
    if (P.p) CK(cudaMemcpyAsync(me.data(), h->d_mineig, sizeof(double) * P.p, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double mn = std::numeric_limits<double>::infinity();
    for (double e : me) mn = std::min(mn, e);
    out[2] = std::sqrt(h->h_chk[22]);
    out[3] = mn;
  }
  if (cx < 0) {
    // xt = x / (-cx), st = s / (-cx) ; |A xt| ; |H xt - st| ; min eig of H xt
    k_div_copy<<<h->grid_T, kBlock, 0, st>>>(x, h->d_chk + 21, -1.0, P.n_c + P.n_d, t2);
    CKL();
    const double *xt = t2, *stv = t2 + P.n_c;
    k_spmv_seg<<<h->grid_seg, kBlock, 0, st>>>(P, xt, h->d_qseg2);
    k_rowres_part<<<h->grid_m, kBlock, 0, st>>>(P, h->d_qseg2, nullptr, h->W.part);
    k_sum_parts<<<1, 1024, 0, st>>>(h->W.part, h->grid_m, h->d_chk + 23);
    CKL();
    double *pa = h->W.part, *pb = h->W.part + 2048;
    k_cons_part<<<h->grid_nd, kBlock, 0, st>>>(P, xt, stv, pa, pb);
    k_sum_parts<<<1, 1024, 0, st>>>(pa, h->grid_nd, h->d_chk + 24);
    CKL();
    double *hx = h->d_tmp3;
    k_gather<<<h->grid_nd, kBlock, 0, st>>>(P, xt, hx);
    CKL();
    if (launch_cone(h, CONE_MINEIG, h->warp_plan, false, hx, h->d_mineig, 1.0, st)) return HSDE_ERR_CUDA;
    if (launch_cone(h, CONE_MINEIG, h->block_plan, true, hx, h->d_mineig, 1.0, st)) return HSDE_ERR_CUDA;
    std::vector<double> me(P.p);
    CK(cudaMemcpyAsync(h->h_chk + 23, h->d_chk + 23, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (P.p) CK(cudaMemcpyAsync(me.data(), h->d_mineig, sizeof(double) * P.p, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double mn = std::numeric_limits<double>::infinity();
    for (double e : me) mn = std::min(mn, e);
    out[4] = std::sqrt(h->h_chk[23]);
    out[5] = std::sqrt(h->h_chk[24]);
    out[6] = mn;
  }
  (void)T;
  return check_err_flag(h);
}

int hsde_affine_project(hsde_t *h, const double *w, double *u) {
  if (!h || !w || !u || !h->factor) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  const DevProblem &P = h->P;
  cudaStream_t st = h->st;
  const int64_t T = P.total;
  double *dw = h->d_tmp, *rho = h->d_tmp2, *du = h->d_tmp3;
  CK(cudaMemcpyAsync(dw, w, sizeof(double) * T, cudaMemcpyHostToDevice, st));
  k_rho<<<h->grid_T, kBlock, 0, st>>>(P, dw, rho);  // solver.py:301
  CKL();
  int rc = inner_explicit(h, rho, du, st);
  if (rc) return rc;
  if ((rc = dev_dot(h, h->d_zeta, du, T - 1, h->W.scal + S_ZU, st))) return rc;  // :315
  k_shift_apply<<<h->grid_T, kBlock, 0, st>>>(P, du, h->W.scal + S_ZU);         // :316
  CKL();
  if ((rc = dev_dot(h, h->d_zeta, du, T - 1, h->W.scal + S_UTAU, st))) return rc;
  k_tau_out<<<1, 32, 0, st>>>(dw, T, h->W.scal + S_UTAU, du);                    // :317
  CKL();
  CK(cudaMemcpyAsync(u, du, sizeof(double) * T, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return HSDE_OK;
}

int hsde_solve_inner(hsde_t *h, const double *w12, double *u12) {
  if (!h || !w12 || !u12 || !h->factor) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  const int64_t T = h->P.total;
  CK(cudaMemcpyAsync(h->d_tmp2, w12, sizeof(double) * (T - 1), cudaMemcpyHostToDevice, h->st));
  int rc = inner_explicit(h, h->d_tmp2, h->d_tmp3, h->st);
  if (rc) return rc;
  CK(cudaMemcpyAsync(u12, h->d_tmp3, sizeof(double) * (T - 1), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return HSDE_OK;
}

int hsde_project_cone(hsde_t *h, const double *in, double *out) {
  if (!h || !in || !out) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  const DevProblem &P = h->P;
  const int64_t T = P.total;
  cudaStream_t st = h->st;
  CK(cudaMemcpyAsync(h->d_tmp, in, sizeof(double) * T, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(h->d_tmp2, h->d_tmp, sizeof(double) * T, cudaMemcpyDeviceToDevice, st));
  const double *sin = h->d_tmp + P.n_c;
  double *sout = h->d_tmp2 + P.n_c;
  if (launch_cone(h, CONE_PLAIN, h->warp_plan, false, sin, sout, 1.0, st)) return HSDE_ERR_CUDA;
  if (launch_cone(h, CONE_PLAIN, h->block_plan, true, sin, sout, 1.0, st)) return HSDE_ERR_CUDA;
  k_tau_clamp<<<1, 32, 0, st>>>(h->d_tmp, T, h->d_tmp2);
  CKL();
  CK(cudaMemcpyAsync(out, h->d_tmp2, sizeof(double) * T, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return check_err_flag(h);
}

int hsde_get_minv_zeta(hsde_t *h, double *out) {
  if (!h || !out || !h->factor) return HSDE_ERR_ARG;
  cudaSetDevice(h->dev);
  CK(cudaMemcpy(out, h->P.mz, sizeof(double) * (h->P.total - 1), cudaMemcpyDeviceToHost));
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
  int rc = hsde_iterate(h, k);
  if (rc) return rc;
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
  cudaEvent_t ev[PS_COUNT + 1];
  for (auto &e : ev) CK(cudaEventCreate(&e));
  for (int i = 0; i < HSDE_PROFILE_SLOTS; ++i) ms[i] = 0.f;
  int nl = 0;
  k_prep_ry<<<h->grid_m, kBlock, 0, h->st>>>(h->P, h->S, h->W);
  CKL();
  ++nl;
  for (int it = 0; it < k; ++it) {
    // record all slot events so unused slots have zero duration
    for (int s = 0; s <= PS_COUNT; ++s) CK(cudaEventRecord(ev[s], h->st));
    int rc = launch_iteration(h, h->st, ev, &nl);
    if (rc) return rc;
    CK(cudaEventSynchronize(ev[PS_XUPD]));
    const int order[] = {PS_COUNT, PS_RHS, PS_SPMV, PS_SCHUR, PS_UA, PS_SCALARS, PS_CONE_WARP,
                         PS_CONE_BLOCK, PS_XUPD};
    for (int q = 1; q < 9; ++q) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, ev[order[q - 1]], ev[order[q]]));
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
  std::vector<int> sw(std::max(h->P.p, 1));
  CK(cudaMemcpyAsync(sw.data(), h->W.sweeps, sizeof(int) * sw.size(), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  double sum = 0, mx = 0, sum_big = 0, n_big = 0;
  std::vector<int> sizes(h->P.p);
  if (h->P.p) CK(cudaMemcpy(sizes.data(), h->P.cl_size, sizeof(int) * h->P.p, cudaMemcpyDeviceToHost));
  for (int k = 0; k < h->P.p; ++k) {
    sum += sw[k];
    mx = std::max(mx, (double)sw[k]);
    if (sizes[k] > 32) {
      sum_big += sw[k];
      n_big += 1;
    }
  }
  out[0] = h->P.p ? sum / h->P.p : 0.0;
  out[1] = mx;
  out[2] = n_big ? sum_big / n_big : 0.0;
  out[3] = h->warm ? 1.0 : 0.0;
  return HSDE_OK;
}

const char *hsde_profile_name(int32_t slot) {
  if (slot < 0 || slot >= HSDE_PROFILE_SLOTS) return "";
  return kProfNames[slot];
}

}  // extern "C"
