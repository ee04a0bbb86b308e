// DMMA (mma.sync m8n8k4 f64) latency / throughput microbenchmark.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_bench tools/dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double *out, long long *cyc, int iters) {
  double d[CH][2];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
  double a = 1.0000001, b = 0.9999999;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
void run(int blocks, int threads) {
  double *o; long long *c;
  cudaMalloc(&o, sizeof(double) * blocks * threads);
  cudaMalloc(&c, sizeof(long long));
  const int iters = 4096;
  k<CH><<<blocks, threads>>>(o, c, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH><<<blocks, threads>>>(o, c, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long cyc; cudaMemcpy(&cyc, c, sizeof(cyc), cudaMemcpyDeviceToHost);
  double flops = 512.0 * CH * iters * (blocks * threads / 32);
  printf("chains %d blocks %d threads %d: %.1f cycles/dmma/warp-chain, %.2f TFLOP/s\n", CH, blocks, threads,
         (double)cyc / iters, flops / ms / 1e9);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<1>(1, 32); run<4>(1, 32); run<8>(1, 32);
  run<1>(1, 128); run<4>(1, 128); run<4>(1, 256); run<4>(1, 512);
  run<4>(148, 128); run<4>(148, 256); run<4>(148, 512); run<8>(148, 512); run<4>(296, 384);
  return 0;
}
