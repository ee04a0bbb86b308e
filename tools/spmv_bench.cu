// Microbenchmark of the two sparse passes over A (m x n_c, ~2% dense, the
// BASELINE config-4 shape): y = A' g (pull over columns, k_ua) and q = A t
// (k_spmv_seg), in several storage layouts.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/spmv_bench tools/spmv_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// ---- A' g: per-thread column loop (current k_ua)
__global__ void k_csc_thread(int n, const int64_t *cp, const int *row, const double *val, const double *g,
                             double *out) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < n; l += gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int64_t e = cp[l]; e < cp[l + 1]; ++e) a += val[e] * __ldg(g + row[e]);
    out[l] = a;
  }
}

// ---- A' g: warp per 32-column slice, segmented scan over the contiguous nnz
// range; key = row | lane << 11 (16 bit) -- g staged in shared memory
template <class K, int SHIFT>
__global__ void __launch_bounds__(256) k_csc_segscan(int n, int m, const int64_t *cp, const K *key,
                                                      const double *val, const double *g, double *out) {
  extern __shared__ double sg[];
  __shared__ double acc[8][33];
  for (int i = threadIdx.x; i < m; i += blockDim.x) sg[i] = g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nsl = (n + 31) >> 5;
  for (int sl = blockIdx.x * 8 + w; sl < nsl; sl += gridDim.x * 8) {
    const int l0 = sl * 32;
    const int64_t b = cp[l0], e = cp[min(l0 + 32, n)];
    acc[w][lane] = 0.0;
    __syncwarp();
    for (int64_t base = b; base < e; base += 128) {
      double v[4];
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t k = base + u * 32 + lane;
        if (k < e) {
          const unsigned kk = key[k];
          v[u] = val[k] * sg[kk & ((1u << SHIFT) - 1)];
          c[u] = kk >> SHIFT;
        } else {
          v[u] = 0.0;
          c[u] = 32;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double t = __shfl_up_sync(0xffffffffu, v[u], o);
          const int tc = __shfl_up_sync(0xffffffffu, c[u], o);
          if (lane >= o && tc == c[u]) v[u] += t;
        }
        const int nc = __shfl_down_sync(0xffffffffu, c[u], 1);
        if ((lane == 31 || nc != c[u]) && c[u] < 32) acc[w][c[u]] += v[u];
        __syncwarp();
      }
    }
    if (l0 + lane < n) out[l0 + lane] = acc[w][lane];
    __syncwarp();
  }
}

// ---- segmented streaming over one group's contiguous element range [b, e):
// key = gather index (low SHIFT bits) | segment (high bits, < 32); the run
// sums are added to acc[segment] (per-warp shared array), in element order.
template <int U, class K, int SHIFT>
__device__ __forceinline__ void seg_stream(const K *__restrict__ key, const double *__restrict__ val,
                                           const double *__restrict__ gs, int64_t b, int64_t e,
                                           double *acc, int lane) {
  for (int64_t base = b; base < e; base += 32 * U) {
    double v[U];
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = base + u * 32 + lane;
      if (k < e) {
        const unsigned kk = __ldcs(key + k);
        v[u] = __ldcs(val + k) * gs[kk & ((1u << SHIFT) - 1)];
        c[u] = kk >> SHIFT;
      } else {
        v[u] = 0.0;
        c[u] = 32;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, v[u], o);
        const int tc = __shfl_up_sync(0xffffffffu, c[u], o);
        if (lane >= o && tc == c[u]) v[u] += t;
      }
      const int nc = __shfl_down_sync(0xffffffffu, c[u], 1);
      if ((lane == 31 || nc != c[u]) && c[u] < 32) acc[c[u]] += v[u];
      __syncwarp();
    }
  }
}

template <int U, int NW>
__global__ void __launch_bounds__(NW * 32) k_csc_seg2(int n, int m, const int64_t *cp, const uint16_t *key,
                                                       const double *val, const double *g, double *out) {
  extern __shared__ double sg[];
  __shared__ double acc[NW][32];
  for (int i = threadIdx.x; i < m; i += blockDim.x) sg[i] = g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nsl = (n + 31) >> 5;
  int sl = blockIdx.x * NW + w;
  int64_t nb = sl < nsl ? cp[sl * 32] : 0, ne = sl < nsl ? cp[min(sl * 32 + 32, n)] : 0;
  for (; sl < nsl; sl += gridDim.x * NW) {
    const int64_t b = nb, e = ne;
    const int nx = sl + gridDim.x * NW;
    if (nx < nsl) {  // prefetch the next slice's range
      nb = cp[nx * 32];
      ne = cp[min(nx * 32 + 32, n)];
    }
    acc[w][lane] = 0.0;
    __syncwarp();
    seg_stream<U, uint16_t, 11>(key, val, sg, b, e, acc[w], lane);
    const int l = sl * 32 + lane;
    if (l < n) out[l] = acc[w][lane];
    __syncwarp();
  }
}

// ---- A' g, SELL-32: slice s of 32 columns, element k of lane j at
// sb[s] + 32 k + j (padded with zeros to the slice's longest column)
template <class K>
__global__ void __launch_bounds__(256) k_sell_col(int n, int m, const int64_t *sb, const K *idx,
                                                   const double *val, const double *g, double *out) {
  extern __shared__ double sg[];
  for (int i = threadIdx.x; i < m; i += blockDim.x) sg[i] = g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nsl = (n + 31) >> 5;
  for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < nsl; sl += (gridDim.x * blockDim.x) >> 5) {
    const int64_t b = sb[sl], e = sb[sl + 1];
    double a0 = 0.0, a1 = 0.0;
    int64_t k = b + lane;
#pragma unroll 4
    for (; k + 32 < e; k += 64) {
      a0 += __ldcs(val + k) * sg[__ldcs(idx + k)];
      a1 += __ldcs(val + k + 32) * sg[__ldcs(idx + k + 32)];
    }
    if (k < e) a0 += __ldcs(val + k) * sg[__ldcs(idx + k)];
    const int l = sl * 32 + lane;
    if (l < n) out[l] = a0 + a1;
  }
}

// ---- A t, row-SELL tiles: tile t of W columns, row group gr of 32 rows;
// element k of lane j (row 32 gr + j) at tb[t G + gr] + 32 k + j, local column
// index (16 bit) into the staged x tile; part[row * ntile + t]
template <int W>
__global__ void __launch_bounds__(256) k_sell_row(int n, int m, int ntile, const int64_t *tb,
                                                   const uint16_t *lcol, const double *val,
                                                   const double *x, double *part, int rg) {
  __shared__ double xs[W];
  const int G = (m + 31) >> 5;
  const int t = blockIdx.x / rg, rr = blockIdx.x - t * rg;
  const int c0 = t * W, wn = min(W, n - c0);
  for (int i = threadIdx.x; i < wn; i += blockDim.x) xs[i] = x[c0 + i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int gr = rr * (blockDim.x >> 5) + (threadIdx.x >> 5); gr < G; gr += rg * (blockDim.x >> 5)) {
    const int64_t b = tb[(int64_t)t * G + gr], e = tb[(int64_t)t * G + gr + 1];
    double a0 = 0.0, a1 = 0.0;
    int64_t k = b + lane;
#pragma unroll 4
    for (; k + 32 < e; k += 64) {
      a0 += __ldcs(val + k) * xs[__ldcs(lcol + k)];
      a1 += __ldcs(val + k + 32) * xs[__ldcs(lcol + k + 32)];
    }
    if (k < e) a0 += __ldcs(val + k) * xs[__ldcs(lcol + k)];
    const int r = gr * 32 + lane;
    if (r < m) part[(int64_t)r * ntile + t] = a0 + a1;
  }
}

// ---- A t: row-split CSR, global gather (current k_spmv_seg)
__global__ void k_csr_seg(int nseg, const int *seg_row, const int64_t *seg_beg, const int64_t *rp,
                          const int *col, const double *val, const double *x, double *qseg) {
  const int lane = threadIdx.x & 31;
  const int seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (seg >= nseg) return;
  const int r = seg_row[seg];
  const int64_t b = seg_beg[seg];
  const int64_t e = min(b + (int64_t)2048, rp[r + 1]);
  double acc = 0.0;
  for (int64_t k = b + lane; k < e; k += 32) acc += val[k] * __ldg(x + col[k]);
  acc = warp_sum(acc);
  if (lane == 0) qseg[seg] = acc;
}

// ---- A t: column tiles of W, x tile staged in shared memory; tile-local CSR
// (row-major within the tile), 16-bit local column; one warp per (tile,row).
// part[row * ntile + tile]
template <int W>
__global__ void __launch_bounds__(512) k_csr_tiled(int n, int m, int ntile, int rgroups, const int64_t *trp,
                                                    const uint16_t *lcol, const double *val,
                                                    const double *x, double *part) {
  __shared__ double xs[W];
  const int tile = blockIdx.x / rgroups, rg = blockIdx.x - tile * rgroups;
  const int c0 = tile * W;
  const int wn = min(W, n - c0);
  for (int i = threadIdx.x; i < wn; i += blockDim.x) xs[i] = x[c0 + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int rows_per = (m + rgroups - 1) / rgroups;
  const int r0 = rg * rows_per, r1 = min(m, r0 + rows_per);
  const int64_t *tp = trp + (int64_t)tile * (m + 1);
  for (int r = r0 + w; r < r1; r += nw) {
    const int64_t b = tp[r], e = tp[r + 1];
    double acc = 0.0;
#pragma unroll 4
    for (int64_t k = b + lane; k < e; k += 32) acc += val[k] * xs[lcol[k]];
    acc = warp_sum(acc);
    if (lane == 0) part[(int64_t)r * ntile + tile] = acc;
  }
}

__global__ void k_rowsum(int m, int ntile, const double *part, double *q) {
  const int lane = threadIdx.x & 31;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= m) return;
  double a = 0.0;
  for (int t = lane; t < ntile; t += 32) a += part[(int64_t)r * ntile + t];
  a = warp_sum(a);
  if (lane == 0) q[r] = a;
}

__global__ void k_stream(const double2 *a, int64_t n2, double *out) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; k + 3 * stride < n2; k += 4 * stride) {
    const double2 x0 = __ldcs(a + k), x1 = __ldcs(a + k + stride), x2 = __ldcs(a + k + 2 * stride),
                  x3 = __ldcs(a + k + 3 * stride);
    acc += x0.x + x0.y + x1.x + x1.y + x2.x + x2.y + x3.x + x3.y;
  }
  for (; k < n2; k += stride) acc += a[k].x + a[k].y;
  if (acc == 12345.0) out[0] = acc;
}

template <class F>
float timeit(F f, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char **argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 1000;
  const int n = argc > 2 ? atoi(argv[2]) : 1921600;
  const double dens = argc > 3 ? atof(argv[3]) : 0.02;
  std::mt19937_64 rng(1);
  std::binomial_distribution<int> bin(m, dens);
  std::normal_distribution<double> nd;
  // CSC
  std::vector<int64_t> cp(n + 1, 0);
  std::vector<int> row;
  std::vector<double> val;
  std::vector<int> pick(m);
  for (int i = 0; i < m; ++i) pick[i] = i;
  for (int l = 0; l < n; ++l) {
    int k = bin(rng);
    for (int j = 0; j < k; ++j) std::swap(pick[j], pick[j + rng() % (m - j)]);
    std::vector<int> rs(pick.begin(), pick.begin() + k);
    std::sort(rs.begin(), rs.end());
    for (int r : rs) { row.push_back(r); val.push_back(nd(rng)); }
    cp[l + 1] = row.size();
  }
  const int64_t nnz = row.size();
  printf("m %d n %d nnz %lld\n", m, n, (long long)nnz);
  std::vector<uint16_t> key16(nnz);
  std::vector<uint32_t> key32(nnz);
  for (int l = 0; l < n; ++l)
    for (int64_t e = cp[l]; e < cp[l + 1]; ++e) {
      key16[e] = (uint16_t)(row[e] | ((l & 31) << 11));
      key32[e] = (uint32_t)row[e] | ((uint32_t)(l & 31) << 27);
    }
  // CSR
  std::vector<int64_t> rp(m + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) rp[row[e] + 1]++;
  for (int i = 0; i < m; ++i) rp[i + 1] += rp[i];
  std::vector<int> col(nnz);
  std::vector<double> rval(nnz);
  {
    std::vector<int64_t> pos(rp.begin(), rp.end() - 1);
    for (int l = 0; l < n; ++l)
      for (int64_t e = cp[l]; e < cp[l + 1]; ++e) {
        const int64_t q = pos[row[e]]++;
        col[q] = l;
        rval[q] = val[e];
      }
  }
  std::vector<int> seg_row;
  std::vector<int64_t> seg_beg;
  for (int i = 0; i < m; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; k += 2048) { seg_row.push_back(i); seg_beg.push_back(k); }
  // tiled CSR (W = 4096)
  constexpr int W = 4096;
  const int ntile = (n + W - 1) / W;
  std::vector<int64_t> trp((int64_t)ntile * (m + 1));
  std::vector<uint16_t> lcol(nnz);
  std::vector<double> tval(nnz);
  {
    int64_t o = 0;
    std::vector<int64_t> cur(m);
    for (int i = 0; i < m; ++i) cur[i] = rp[i];
    for (int t = 0; t < ntile; ++t) {
      const int cend = std::min(n, (t + 1) * W);
      for (int i = 0; i < m; ++i) {
        trp[(int64_t)t * (m + 1) + i] = o;
        while (cur[i] < rp[i + 1] && col[cur[i]] < cend) {
          lcol[o] = (uint16_t)(col[cur[i]] - t * W);
          tval[o] = rval[cur[i]];
          ++o;
          ++cur[i];
        }
      }
      trp[(int64_t)t * (m + 1) + m] = o;
    }
  }
  std::vector<double> g(m), x(n);
  for (auto &v : g) v = nd(rng);
  for (auto &v : x) v = nd(rng);
  // reference results
  std::vector<double> ref_y(n, 0.0), ref_q(m, 0.0);
  for (int l = 0; l < n; ++l)
    for (int64_t e = cp[l]; e < cp[l + 1]; ++e) {
      ref_y[l] += val[e] * g[row[e]];
      ref_q[row[e]] += val[e] * x[l];
    }
  auto up = [](auto &v) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    T *p;
    CK(cudaMalloc(&p, sizeof(T) * std::max<size_t>(v.size(), 1)));
    CK(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return p;
  };
  int64_t *d_cp = up(cp), *d_rp = up(rp), *d_segb = up(seg_beg), *d_trp = up(trp);
  int *d_row = up(row), *d_col = up(col), *d_segr = up(seg_row);
  double *d_val = up(val), *d_rval = up(rval), *d_tval = up(tval), *d_g = up(g), *d_x = up(x);
  uint16_t *d_k16 = up(key16), *d_lcol = up(lcol);
  uint32_t *d_k32 = up(key32);
  double *d_y, *d_q, *d_part;
  CK(cudaMalloc(&d_y, sizeof(double) * n));
  CK(cudaMalloc(&d_q, sizeof(double) * std::max<size_t>(seg_row.size(), m)));
  CK(cudaMalloc(&d_part, sizeof(double) * (size_t)ntile * m));
  std::vector<double> hy(n), hq(m);
  auto chk_y = [&](const char *name, float ms, double bytes) {
    CK(cudaMemcpy(hy.data(), d_y, sizeof(double) * n, cudaMemcpyDeviceToHost));
    double err = 0, nr = 0;
    for (int l = 0; l < n; ++l) { err = std::max(err, fabs(hy[l] - ref_y[l])); nr = std::max(nr, fabs(ref_y[l])); }
    printf("%-28s %8.1f us  %7.0f GB/s  maxerr %.2e\n", name, ms * 1e3, bytes / ms / 1e6, err / nr);
  };
  const int nsm = 148;
  const double base_y = 8.0 * n * 2;  // out + (counted once) overhead
  float ms;
  ms = timeit([&] { k_csc_thread<<<nsm * 8, 256>>>(n, d_cp, d_row, d_val, d_g, d_y); });
  chk_y("csc thread (int32 row)", ms, nnz * 12.0 + 8.0 * n + 8.0 * n);
  for (int blocks : {nsm * 4, nsm * 8, nsm * 16}) {
    ms = timeit([&] { k_csc_segscan<uint16_t, 11><<<blocks, 256, m * 8>>>(n, m, d_cp, d_k16, d_val, d_g, d_y); });
    char nm[64];
    snprintf(nm, 64, "csc segscan key16 g=%d", blocks);
    chk_y(nm, ms, nnz * 10.0 + 8.0 * n + 8.0 * n);
  }
  {
    auto run = [&](auto kern, int blocks, int nthr, const char *nm) {
      ms = timeit([&] { kern<<<blocks, nthr, m * 8>>>(n, m, d_cp, d_k16, d_val, d_g, d_y); });
      chk_y(nm, ms, nnz * 10.0 + 8.0 * n + 8.0 * n);
    };
    run(k_csc_seg2<4, 8>, nsm * 8, 256, "seg2 U4 NW8 g8");
    run(k_csc_seg2<8, 8>, nsm * 8, 256, "seg2 U8 NW8 g8");
    run(k_csc_seg2<8, 8>, nsm * 4, 256, "seg2 U8 NW8 g4");
    run(k_csc_seg2<8, 16>, nsm * 4, 512, "seg2 U8 NW16 g4");
    run(k_csc_seg2<16, 8>, nsm * 8, 256, "seg2 U16 NW8 g8");
    run(k_csc_seg2<8, 4>, nsm * 16, 128, "seg2 U8 NW4 g16");
  }
  ms = timeit([&] { k_csc_segscan<uint32_t, 27><<<nsm * 8, 256, m * 8>>>(n, m, d_cp, d_k32, d_val, d_g, d_y); });
  chk_y("csc segscan key32", ms, nnz * 12.0 + 8.0 * n + 8.0 * n);
  // CSR
  auto chk_q = [&](const char *name, float ms, double bytes, bool from_seg) {
    if (from_seg) {
      std::vector<double> qs(seg_row.size());
      CK(cudaMemcpy(qs.data(), d_q, sizeof(double) * qs.size(), cudaMemcpyDeviceToHost));
      std::fill(hq.begin(), hq.end(), 0.0);
      for (size_t s = 0; s < qs.size(); ++s) hq[seg_row[s]] += qs[s];
    } else {
      CK(cudaMemcpy(hq.data(), d_q, sizeof(double) * m, cudaMemcpyDeviceToHost));
    }
    double err = 0, nr = 0;
    for (int i = 0; i < m; ++i) { err = std::max(err, fabs(hq[i] - ref_q[i])); nr = std::max(nr, fabs(ref_q[i])); }
    printf("%-28s %8.1f us  %7.0f GB/s  maxerr %.2e\n", name, ms * 1e3, bytes / ms / 1e6, err / nr);
  };
  const int nseg = seg_row.size();
  ms = timeit([&] { k_csr_seg<<<(nseg * 32 + 255) / 256, 256>>>(nseg, d_segr, d_segb, d_rp, d_col, d_rval, d_x, d_q); });
  chk_q("csr seg (global gather)", ms, nnz * 12.0 + 8.0 * n, true);
  for (int rg : {1, 2, 4, 8}) {
    ms = timeit([&] {
      k_csr_tiled<W><<<ntile * rg, 512>>>(n, m, ntile, rg, d_trp, d_lcol, d_tval, d_x, d_part);
      k_rowsum<<<(m * 32 + 255) / 256, 256>>>(m, ntile, d_part, d_q);
    });
    char nm[64];
    snprintf(nm, 64, "csr tiled W=4096 rg=%d", rg);
    chk_q(nm, ms, nnz * 10.0 + 8.0 * n, false);
  }
  for (int g : {nsm * 2, nsm * 4, nsm * 8, nsm * 16}) {
    ms = timeit([&] { k_stream<<<g, 256>>>((const double2 *)d_val, nnz / 2, d_y); });
    printf("stream read val g=%d  %8.1f us  %7.0f GB/s\n", g, ms * 1e3, nnz * 8.0 / ms / 1e6);
  }
  {
    // SELL-32 columns
    const int nsl = (n + 31) / 32;
    std::vector<int64_t> sb(nsl + 1, 0);
    for (int sl = 0; sl < nsl; ++sl) {
      int64_t w = 0;
      for (int l = sl * 32; l < std::min(n, sl * 32 + 32); ++l) w = std::max(w, cp[l + 1] - cp[l]);
      sb[sl + 1] = sb[sl] + 32 * w;
    }
    std::vector<uint16_t> si(sb[nsl], 0);
    std::vector<double> sv(sb[nsl], 0.0);
    for (int l = 0; l < n; ++l) {
      const int sl = l / 32, j = l % 32;
      for (int64_t e = cp[l]; e < cp[l + 1]; ++e) {
        si[sb[sl] + 32 * (e - cp[l]) + j] = (uint16_t)row[e];
        sv[sb[sl] + 32 * (e - cp[l]) + j] = val[e];
      }
    }
    printf("SELL col padding %.3f\n", (double)sb[nsl] / nnz);
    int64_t *d_sb = up(sb);
    uint16_t *d_si = up(si);
    double *d_sv = up(sv);
    for (int blocks : {nsm * 4, nsm * 8, nsm * 16}) {
      ms = timeit([&] { k_sell_col<uint16_t><<<blocks, 256, m * 8>>>(n, m, d_sb, d_si, d_sv, d_g, d_y); });
      char nm[64];
      snprintf(nm, 64, "SELL-32 col g=%d", blocks);
      chk_y(nm, ms, sb[nsl] * 10.0 + 8.0 * n);
    }
    // row-SELL tiles
    constexpr int W2 = 4096;
    const int nt2 = (n + W2 - 1) / W2, G = (m + 31) / 32;
    std::vector<std::vector<std::pair<int, double>>> cell((size_t)nt2 * m);
    for (int l = 0; l < n; ++l)
      for (int64_t e = cp[l]; e < cp[l + 1]; ++e)
        cell[(size_t)(l / W2) * m + row[e]].push_back({l % W2, val[e]});
    std::vector<int64_t> tb((size_t)nt2 * G + 1, 0);
    for (int t = 0; t < nt2; ++t)
      for (int gr = 0; gr < G; ++gr) {
        size_t w = 0;
        for (int r = gr * 32; r < std::min(m, gr * 32 + 32); ++r) w = std::max(w, cell[(size_t)t * m + r].size());
        tb[(size_t)t * G + gr + 1] = tb[(size_t)t * G + gr] + 32 * (int64_t)w;
      }
    const int64_t tot = tb[(size_t)nt2 * G];
    std::vector<uint16_t> ti(tot, 0);
    std::vector<double> tv(tot, 0.0);
    for (int t = 0; t < nt2; ++t)
      for (int r = 0; r < m; ++r) {
        const auto &c = cell[(size_t)t * m + r];
        const int64_t base = tb[(size_t)t * G + r / 32];
        for (size_t k = 0; k < c.size(); ++k) {
          ti[base + 32 * k + r % 32] = (uint16_t)c[k].first;
          tv[base + 32 * k + r % 32] = c[k].second;
        }
      }
    printf("row-SELL padding %.3f\n", (double)tot / nnz);
    int64_t *d_tb = up(tb);
    uint16_t *d_ti = up(ti);
    double *d_tv = up(tv);
    for (int rg : {1, 2, 4}) {
      ms = timeit([&] {
        k_sell_row<W2><<<nt2 * rg, 256>>>(n, m, nt2, d_tb, d_ti, d_tv, d_x, d_part, rg);
        k_rowsum<<<(m * 32 + 255) / 256, 256>>>(m, nt2, d_part, d_q);
      });
      char nm[64];
      snprintf(nm, 64, "row-SELL W=4096 rg=%d (+rowsum)", rg);
      chk_q(nm, ms, tot * 10.0 + 8.0 * n, false);
    }
    ms = timeit([&] { k_rowsum<<<(m * 32 + 255) / 256, 256>>>(m, nt2, d_part, d_q); });
    printf("rowsum only %.1f us\n", ms * 1e3);
  }
  // pure streaming reference: read val once
  ms = timeit([&] { k_csc_thread<<<nsm * 8, 256>>>(0, d_cp, d_row, d_val, d_g, d_y); });
  printf("empty launch %.1f us\n", ms * 1e3);
  return 0;
}
