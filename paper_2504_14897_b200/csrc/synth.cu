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

// ---------------------------------------------------------------- reference generator
// synthdata.cpp:54-86 on the device, drawing from the reference's own stream (rng.hpp:17-48):
// ONE mt19937_64(seed); uniform() = (x >> 11)·2⁻⁵³; normal() = Box-Muller that returns
// r·cos and keeps r·sin as the spare for the next call. Per particle: one selection
// uniform, then d normals. The engine is sequential, so a single CTA produces the uniform
// stream: the in-place 312-word twist splits into two data-parallel halves (i < 156 reads
// only untouched words; i >= 156 reads the words the first half just wrote, and i = 311
// reads the new word 0, exactly as the sequential loop does). The transform is one thread
// per particle at a closed-form stream offset, so it is embarrassingly parallel.
constexpr int kMtN = 312, kMtM = 156;

VDFCG_DEV uint64_t mt_twist(uint64_t upper_src, uint64_t lower_src) {
  const uint64_t xx = (upper_src & 0xFFFFFFFF80000000ULL) | (lower_src & 0x7FFFFFFFULL);
  return (xx >> 1) ^ ((xx & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
}

VDFCG_DEV double mt_uniform(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return static_cast<double>(y >> 11) * 0x1.0p-53;
}

// Thread t < 156 keeps the pair (mt[t], mt[t + 156]) in registers. The sequential twist
// gives  mt'[t] = mt[t+156] ^ T(mt[t], mt[t+1])  and  mt'[t+156] = mt'[t] ^ T(mt[t+156],
// mt[t+157]), where mt[312] means the NEW word 0 (the loop wraps after updating it), so a
// thread needs only its right neighbour's old pair: one double-buffered shared-memory
// exchange and ONE barrier per 312 words. Thread 155 recomputes the new word 0 itself.
// The single CTA stores the raw (untempered) words; tempering and the 53-bit conversion run
// in the all-SM transform, which keeps the serial kernel to the twist itself.
__global__ void __launch_bounds__(kMtM) mt_stream_kernel(uint64_t seed, int64_t count,
                                                        uint64_t* __restrict__ out) {
  __shared__ uint64_t sh[2][2][kMtM];  // [buffer][low half / high half][t]
  const int t = threadIdx.x;
  if (t == 0) {  // std::mersenne_twister_engine seeding, into buffer 1 (read on block 0)
    uint64_t x = seed;
    sh[1][0][0] = x;
    for (int i = 1; i < kMtN; ++i) {
      x = 6364136223846793005ULL * (x ^ (x >> 62)) + i;
      sh[1][i / kMtM][i % kMtM] = x;
    }
  }
  __syncthreads();
  uint64_t A = sh[1][0][t], B = sh[1][1][t];
  int p = 0;
  for (int64_t base = 0; base < count; base += kMtN) {
    sh[p][0][t] = A;
    sh[p][1][t] = B;
    __syncthreads();
    uint64_t A1, B1;
    if (t + 1 < kMtM) {
      A1 = sh[p][0][t + 1];
      B1 = sh[p][1][t + 1];
    } else {
      A1 = sh[p][1][0];                                        // mt[156]
      B1 = sh[p][1][0] ^ mt_twist(sh[p][0][0], sh[p][0][1]);   // new mt[0]
    }
    A = B ^ mt_twist(A, A1);
    B = A ^ mt_twist(B, B1);
    if (base + t < count) out[base + t] = A;
    if (base + t + kMtM < count) out[base + t + kMtM] = B;
    p ^= 1;
  }
}

// Stream offsets (normal call j = n·d + a pairs up as q = j/2; pair q is opened by the
// particle floor(2q/d) after its selection uniform): selection uniform of particle n at
// n + 2·ceil(n·d/2); pair q's two uniforms at floor(2q/d) + 1 + 2q.
__global__ void generate_kernel(int d, int m, int64_t n, const uint64_t* __restrict__ uni,
                                const double* __restrict__ par, double* __restrict__ vel) {
  // par: cdf[m], mean[m][d], chol[m][3][3] (row-major lower factor)
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j0 = r * d;
    const double u = mt_uniform(uni[r + 2 * ((j0 + 1) >> 1)]);
    int k = 0;
    while (k + 1 < m && u >= par[k]) ++k;
    double z[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < d; ++a) {
      const int64_t j = j0 + a, q = j >> 1;
      const int64_t pos = (2 * q) / d + 1 + 2 * q;
      const double u1 = 1.0 - mt_uniform(uni[pos]);
      const double u2 = mt_uniform(uni[pos + 1]);
      const double rad = sqrt(-2.0 * log(u1));
      const double ang = 6.283185307179586 * u2;  // 2.0 * M_PI * u2 (2·π folds exactly)
      z[a] = (j & 1) ? rad * sin(ang) : rad * cos(ang);
    }
    const double* mean = par + m + k * d;
    const double* L = par + m + m * d + k * 9;
    for (int a = 0; a < d; ++a) {
      double s = 0.0;  // no FMA contraction: the reference builds without -march
      for (int b = 0; b < d; ++b) s = __dadd_rn(s, __dmul_rn(L[a * 3 + b], z[b]));
      vel[static_cast<int64_t>(a) * n + r] = __dadd_rn(mean[a], s);
    }
  }
}

void launch_mt_serial(vdfcg_ctx* ctx, uint64_t seed, int64_t count, uint64_t* out) {
  VDFCG_LAUNCH(ctx, "mt19937_64_stream", mt_stream_kernel<<<1, kMtM, 0, ctx->stream>>>(seed, count, out));
}

bool launch_mt_stream_jump(vdfcg_ctx* ctx, uint64_t seed, int64_t count, uint64_t* out);  // mtjump.cu

void launch_generate(vdfcg_ctx* ctx, int d, int m, int64_t n, uint64_t seed, uint64_t* uniforms,
                     int64_t n_uniforms, const double* params, double* vel) {
  // long streams: base window + one CTA per 2^18-word chunk (GF(2) jump-ahead, mtjump.cu);
  // short ones: the single-CTA twist
  if (!launch_mt_stream_jump(ctx, seed, n_uniforms, uniforms)) launch_mt_serial(ctx, seed, n_uniforms, uniforms);
  const int grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>((n + 255) / 256, static_cast<int64_t>(ctx->sm_count) * 16)));
  VDFCG_LAUNCH(ctx, "generate",
               generate_kernel<<<grid, 256, 0, ctx->stream>>>(d, m, n, uniforms, params, vel));
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
