// synth.cu — deterministic synthetic plasma cells for tests and the benchmark (not the
// compression path). Counter-based: particle p of cell c of species s depends only on
// (seed, s, p), so any shard regenerates identical data. Electrons (s=0): thermal core
// (unit variance) + a colder beam whose drift, density fraction and temperature vary
// smoothly with the cell index; ions (s=1): colder core plus a
// weak hot tail. Box-Muller on splitmix64 uniforms, FP64.
#include <algorithm>

#include "common.cuh"
#include "ctx.cuh"

namespace vdfcg {

VDFCG_DEV uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

VDFCG_DEV double u01(uint64_t h) { return (static_cast<double>(h >> 11) + 0.5) * 0x1.0p-53; }

__global__ void synth_kernel(int d, int n_cells, const int64_t* __restrict__ offsets,
                             int64_t cell_base, uint64_t seed, int species,
                             double* __restrict__ u, double* __restrict__ v,
                             double* __restrict__ w) {
  const int64_t p0 = offsets[0];
  const int64_t n = offsets[n_cells] - p0;
  const uint64_t key = splitmix64(seed ^ (0x5851F42D4C957F2DULL * (species + 1)));
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = p0 + q;  // global particle index
    int lo = 0, hi = n_cells - 1;  // cell owning p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (offsets[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const double cg = static_cast<double>(cell_base + lo);
    const double ph1 = 0.0123 * cg, ph2 = 0.00731 * cg;
    const uint64_t h0 = splitmix64(key + 4 * static_cast<uint64_t>(p));
    const uint64_t h1 = splitmix64(h0 + 1), h2 = splitmix64(h0 + 2), h3 = splitmix64(h0 + 3),
                   h4 = splitmix64(h0 + 4);
    const double r1 = sqrt(-2.0 * log(u01(h1))), a1 = 6.283185307179586 * u01(h2);
    const double r2 = sqrt(-2.0 * log(u01(h3))), a2 = 6.283185307179586 * u01(h4);
    const double z0 = r1 * cos(a1), z1 = r1 * sin(a1), z2 = r2 * cos(a2);
    double m0 = 0, m1 = 0, m2 = 0, s0 = 1, s1 = 1, s2 = 1;
    const double sel = u01(h0);
    if (species == 0) {
      const double fb = 0.2 + 0.08 * sin(ph2);
      if (sel < fb) {
        m0 = 2.6 + 0.5 * sin(ph1);
        m1 = 0.6 * cos(ph2);
        const double sb = 0.45 + 0.1 * cos(ph1);
        s0 = s1 = s2 = sb;
      }
    } else {
      s0 = s1 = s2 = 0.3;
      if (sel < 0.1) {
        m0 = 0.3 * sin(ph1);
        s0 = s1 = s2 = 0.6;
      }
    }
    u[q] = m0 + s0 * z0;
    v[q] = m1 + s1 * z1;
    if (d == 3) w[q] = m2 + s2 * z2;
  }
}

void launch_synth(vdfcg_ctx* ctx, int d, int n_cells, const int64_t* offsets, int64_t cell_base,
                  uint64_t seed, int species, double* u, double* v, double* w) {
  VDFCG_LAUNCH(ctx, "synth",
               synth_kernel<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(d, n_cells, offsets, cell_base,
                                                                        seed, species, u, v, w));
}

// ---------------------------------------------------------------- peak probe
// 8 independent FMA chains per thread, 64K iterations: issue-bound FMA throughput.
template <class T>
__global__ void __launch_bounds__(256) fma_probe_kernel(T seed, int iters, T* sink) {
  T a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + T(threadIdx.x + k);
  const T b = T(0.999999), c = T(1e-7);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  T s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == T(-12345)) *sink = s;  // keep the work alive
}

template <class T>
static double probe(vdfcg_ctx* ctx) {
  T* sink = arena<T>(ctx, 1);
  const int blocks = ctx->sm_count * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t a, b;
  VDFCG_CUDA(cudaEventCreate(&a));
  VDFCG_CUDA(cudaEventCreate(&b));
  fma_probe_kernel<T><<<blocks, threads, 0, ctx->stream>>>(T(1), iters, sink);  // warm-up
  double best = 0.0;
  for (int r = 0; r < 5; ++r) {
    VDFCG_CUDA(cudaEventRecord(a, ctx->stream));
    fma_probe_kernel<T><<<blocks, threads, 0, ctx->stream>>>(T(1), iters, sink);
    VDFCG_CUDA(cudaEventRecord(b, ctx->stream));
    VDFCG_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    VDFCG_CUDA(cudaEventElapsedTime(&ms, a, b));
    const double flops = 2.0 * 8.0 * double(iters) * blocks * threads;
    best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

double probe_fp64(vdfcg_ctx* ctx) { return probe<double>(ctx); }
double probe_fp32(vdfcg_ctx* ctx) { return probe<float>(ctx); }

}  // namespace vdfcg
