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

__global__ void synth_kernel(int d, int n_cells, const int64_t* __restrict__ offsets, uint64_t seed,
                             int species, double* __restrict__ u, double* __restrict__ v,
                             double* __restrict__ w) {
  const int64_t n = offsets[n_cells];
  const uint64_t key = splitmix64(seed ^ (0x5851F42D4C957F2DULL * (species + 1)));
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = n_cells - 1;  // cell owning p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (offsets[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const double ph1 = 0.0123 * lo, ph2 = 0.00731 * lo;
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
    u[p] = m0 + s0 * z0;
    v[p] = m1 + s1 * z1;
    if (d == 3) w[p] = m2 + s2 * z2;
  }
}

void launch_synth(vdfcg_ctx* ctx, int d, int n_cells, const int64_t* offsets, uint64_t seed,
                  int species, double* u, double* v, double* w) {
  VDFCG_LAUNCH(ctx, "synth",
               synth_kernel<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(d, n_cells, offsets, seed,
                                                                        species, u, v, w));
}

}  // namespace vdfcg
