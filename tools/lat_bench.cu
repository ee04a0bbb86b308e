// Single-warp dependent-chain latencies on the B200 (clock64): DFMA, DADD,
// double shuffle, shared-memory load chain, double division, sqrt, and a
// __syncthreads round trip.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double *out, long long *cyc, double a, double b, int n) {
  __shared__ double sh[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sh[i] = 1.0 + i * 1e-9; idx[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  double x = threadIdx.x * 1e-3 + 1.0;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  t1 = clock64(); cyc[0] = (t1 - t0) / n;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + b;
  t1 = clock64(); cyc[1] = (t1 - t0) / n;
  // shuffle chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + b;
  t1 = clock64(); cyc[2] = (t1 - t0) / n;
  // LDS pointer chase
  int p = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = idx[p];
  t1 = clock64(); cyc[3] = (t1 - t0) / n;
  // division chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = b / x + a;
  t1 = clock64(); cyc[4] = (t1 - t0) / n;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + a;
  t1 = clock64(); cyc[5] = (t1 - t0) / n;
  // syncthreads
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); cyc[6] = (t1 - t0) / n;
  // LDS double dependent: x = sh[(int)x & 1023]
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sh[p & 1023] * x, p += 1;
  t1 = clock64(); cyc[7] = (t1 - t0) / n;
  // drcp chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x) + a;
  t1 = clock64(); cyc[8] = (t1 - t0) / n;
  out[threadIdx.x] = x + p;
}

int main() {
  double *out; long long *cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  for (int threads : {32, 384}) {
    k_lat<<<1, threads>>>(out, cyc, 0.999999, 1e-7, 1000);
    cudaDeviceSynchronize();
    printf("threads %d: dfma %lld dadd %lld shfl+dadd %lld lds-chase %lld ddiv+dadd %lld dsqrt+dadd %lld syncthreads %lld lds*dmul %lld drcp+dadd %lld\n",
           threads, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cyc[7], cyc[8]);
  }
  return 0;
}
