// Probe: DMMA (mma.sync m8n8k4 f64) throughput on B200, and whether it overlaps DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int NF, int NM>
__global__ void k(double* out, int iters, double s) {
  double a[8], c0[4], c1[4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) c0[j] = c1[j] = 0;
  double x = threadIdx.x * 1e-4, y = 1.0 - x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < NF; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fma(a[j], s, 1e-9);
#pragma unroll
    for (int r = 0; r < NM; ++r)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(c0[j], c1[j], x, y);
  }
  double t = 0;
  for (int j = 0; j < 8; ++j) t += a[j];
  for (int j = 0; j < 4; ++j) t += c0[j] + c1[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int NF, int NM>
float run(double* d, int iters) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<NF, NM><<<148 * 4, 256>>>(d, iters, 0.999999);
  cudaEventRecord(a);
  k<NF, NM><<<148 * 4, 256>>>(d, iters, 0.999999);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fl_f = 2.0 * NF * 8 * iters * 148.0 * 4 * 256;            // per-thread FMAs
  double fl_m = 2.0 * NM * 4 * 256.0 * iters * 148 * 4 * 256 / 32;  // 256 FMA per warp-mma
  printf("NF=%d NM=%d: %.3f ms  dfma %.1f TF  dmma %.1f TF\n", NF, NM, ms, fl_f / ms * 1e-9,
         fl_m / ms * 1e-9);
  return ms;
}
int main() {
  double* d; cudaMalloc(&d, 148 * 4 * 256 * 8);
  int it = 2000;
  run<4, 0>(d, it);
  run<0, 4>(d, it);
  run<4, 4>(d, it);
  run<4, 1>(d, it);
  run<4, 2>(d, it);
  run<2, 4>(d, it);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
