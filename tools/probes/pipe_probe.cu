// Probe: do F2I.F64 / I2F.F64 / DSETP share the FP64 pipe with DFMA on B200? (tools only)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters, double s) {
  double a[8];
  int acc = 0;
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[j] = fma(a[j], s, 1e-9);
      if (MODE == 1) acc += __double2int_rn(a[j] * 0.5);          // DMUL + F2I
      if (MODE == 2) a[j] += (double)(it + j);                      // I2F + DADD
      if (MODE == 3) acc += (a[j] < -5.0) ? 1 : 0;                  // DSETP
      if (MODE == 4) acc += __double2int_rn(a[j]);                  // F2I only
    }
  }
  double t = 0;
  for (int j = 0; j < 8; ++j) t += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t + acc;
}
template <int MODE>
float run(double* d, int iters) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<MODE><<<148 * 4, 256>>>(d, iters, 0.999999);
  cudaEventRecord(a);
  k<MODE><<<148 * 4, 256>>>(d, iters, 0.999999);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  double* d; cudaMalloc(&d, 148 * 4 * 256 * 8);
  int it = 4000;
  printf("dfma only        %.3f ms\n", run<0>(d, it));
  printf("+dmul+f2i        %.3f ms\n", run<1>(d, it));
  printf("+i2f+dadd        %.3f ms\n", run<2>(d, it));
  printf("+dsetp           %.3f ms\n", run<3>(d, it));
  printf("+f2i only        %.3f ms\n", run<4>(d, it));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
