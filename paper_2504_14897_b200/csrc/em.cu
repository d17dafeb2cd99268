// em.cu — K5: the batched weighted-EM fitter (sm_100a, FP64 CUDA cores).
//
// Cells: one CTA of G warps owns one fit at a time and pulls the next one from an
// atomic queue (persistent grid). A single point set (vdfcg_fit) runs on a thread-block
// cluster of up to 16 CTAs that split its points and combine partial statistics through
// distributed shared memory; every CTA runs the same deterministic protocol.
// Per fit, entirely on-device (wgmm.cpp:364-423):
//   prologue   normalize over the non-empty bins (wgmm.cpp:78-100), temperature
//              (wgmm.cpp:22-25), seeded init or warm start (wgmm.cpp:136-191)
//   iteration  lanes of warp 0 factor every component (LLT + in-place repair,
//              wgmm.cpp:197-229) into a pre-scaled affine form; all threads stream the
//              points once: log2-domain log-densities, per-point log-sum-exp (table exp2 /
//              log), responsibilities and the weighted sufficient statistics about the
//              frame origin in registers; fixed-order warp reduce-scatter + cross-warp
//              (+ cross-CTA) reduction (bitwise reproducible); M-step per component lane
//              (Eq. 9; an exact second pass centred on the new mean where the raw-moment
//              form would cost precision), collapse test by a Cholesky-determinant
//              certificate with the full eigen/repair path near the threshold
//              (wgmm.cpp:300-315); thread 0 runs degenerate removal, scheduled pruning and
//              the convergence test (wgmm.cpp:386-417) on the E-step log-likelihood
//   epilogue   denormalize (wgmm.cpp:102-120) and write parameters + diagnostics.
// Points never leave L1/L2 between iterations of a fit; parameters live in shared memory.
#include <cub/block/block_reduce.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>

#include "common.cuh"
#include "em.cuh"
#include "em_dev.cuh"
#include "em_kernel_api.cuh"
#include "linalg.cuh"

namespace vdfcg {

// Single point-set prologue (vdfcg_fit): validate, normalize, z, temperature, distinct.
template <int D>
__global__ void __launch_bounds__(1024) fit_prologue_kernel(const double* __restrict__ x,
                                                            const double* __restrict__ w,
                                                            int64_t n, double total_weight,
                                                            EmConfig cfg, double* __restrict__ z,
                                                            Frame* frame) {
  __shared__ double s_min[32][3], s_max[32][3], s_sum[32][7];
  __shared__ int s_flags[2];
  __shared__ double s_list[kMaxK][3];
  __shared__ int s_count;
  __shared__ double s_off[3], s_scale[3];
  __shared__ int s_status, s_axis;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    s_flags[0] = 0;
    s_flags[1] = 0;
    s_status = 0;
    s_axis = -1;
  }
  __syncthreads();
  // WeightedPoints::validate (histogram.cpp:20-26) + bounding box
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = dinf();
    hi[a] = -dinf();
  }
  bool neg = false, pos = false;
  for (int64_t p = threadIdx.x; p < n; p += blockDim.x) {
    const double wt = w[p];
    neg |= !(wt >= 0.0);
    pos |= wt > 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double v = x[a * n + p];
      lo[a] = fmin(lo[a], v);
      hi[a] = fmax(hi[a], v);
    }
  }
  if (neg) atomicOr(&s_flags[0], 1);
  if (pos) atomicOr(&s_flags[1], 1);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lo[a] = warp_min(lo[a]);
    hi[a] = warp_max(hi[a]);
    if (lane == 0) {
      s_min[warp][a] = lo[a];
      s_max[warp][a] = hi[a];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Frame F{};
    F.total = total_weight;
    if (n == 0) {
      s_status = VDFCG_INVALID_ARGUMENT;
      s_axis = kMsgEmpty;
    } else if (s_flags[0]) {
      s_status = VDFCG_INVALID_ARGUMENT;
      s_axis = kMsgNegWeight;
    } else if (!s_flags[1]) {
      s_status = VDFCG_INVALID_ARGUMENT;
      s_axis = kMsgNoPosWeight;
    } else {
      for (int a = 0; a < D; ++a) {
        double l = s_min[0][a], h = s_max[0][a];
        for (int g = 1; g < G; ++g) {
          l = fmin(l, s_min[g][a]);
          h = fmax(h, s_max[g][a]);
        }
        s_off[a] = __dmul_rn(0.5, __dadd_rn(l, h));
        s_scale[a] = __dmul_rn(0.5, __dsub_rn(h, l));
        F.offset[a] = s_off[a];
        F.scale[a] = s_scale[a];
        if (!(s_scale[a] > 0.0) && !s_status) {
          s_status = VDFCG_INVALID_ARGUMENT;
          s_axis = kMsgZeroSpread + a;
          F.err_value = l;
        }
      }
    }
    F.status = s_status;
    F.err_axis = s_axis;
    *frame = F;
  }
  __syncthreads();
  if (s_status) return;
  // z = (x - offset) / scale, its bounding box, and the data-space moments
  const bool need_temp = !cfg.has_temp && cfg.warm_m == 0;
  double zl[3], zh[3], sw = 0.0, sx[3] = {0, 0, 0}, sxx[3] = {0, 0, 0};
  for (int a = 0; a < 3; ++a) {
    zl[a] = dinf();
    zh[a] = -dinf();
  }
  for (int64_t p = threadIdx.x; p < n; p += blockDim.x) {
    const double wt = w[p];
    if (need_temp) sw += wt;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double v = x[a * n + p];
      const double zz = __dsub_rn(v, s_off[a]) / s_scale[a];
      z[a * n + p] = zz;
      zl[a] = fmin(zl[a], zz);
      zh[a] = fmax(zh[a], zz);
      if (need_temp) {
        const double xw = v * wt;
        sx[a] += xw;
        sxx[a] += xw * v;
      }
    }
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    zl[a] = warp_min(zl[a]);
    zh[a] = warp_max(zh[a]);
    if (lane == 0) {
      s_min[warp][a] = zl[a];
      s_max[warp][a] = zh[a];
    }
  }
  if (need_temp) {
    sw = warp_sum(sw);
#pragma unroll
    for (int a = 0; a < D; ++a) {
      sx[a] = warp_sum(sx[a]);
      sxx[a] = warp_sum(sxx[a]);
    }
    if (lane == 0) {
      s_sum[warp][0] = sw;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        s_sum[warp][1 + a] = sx[a];
        s_sum[warp][4 + a] = sxx[a];
      }
    }
  }
  __syncthreads();  // z is complete: distinct-point count in warp 0 (wgmm.cpp:124-132)
  if (warp == 0) {
    const int count = count_distinct_warp<D>(z, n, cfg.warm_m > 0 ? 0 : cfg.M, s_list);
    if (lane == 0) s_count = count;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Frame F = *frame;
    for (int a = 0; a < D; ++a) {
      double l = s_min[0][a], h = s_max[0][a];
      for (int g = 1; g < G; ++g) {
        l = fmin(l, s_min[g][a]);
        h = fmax(h, s_max[g][a]);
      }
      F.zlo[a] = l;
      F.zhi[a] = h;
    }
    if (cfg.has_temp) {
      for (int a = 0; a < D; ++a) F.temp[a] = cfg.temp[a];
    } else if (cfg.warm_m == 0) {
      double tsw = 0.0, tsx[3] = {0, 0, 0}, tsxx[3] = {0, 0, 0};
      for (int g = 0; g < G; ++g) {
        tsw += s_sum[g][0];
        for (int a = 0; a < D; ++a) {
          tsx[a] += s_sum[g][1 + a];
          tsxx[a] += s_sum[g][4 + a];
        }
      }
      for (int a = 0; a < D; ++a) {
        const double mean = tsx[a] / tsw;
        const double var = fmax(tsxx[a] / tsw - mean * mean, 0.0);
        F.temp[a] = var;
        if (!(var > 0.0) && !F.status) {
          F.status = VDFCG_INVALID_ARGUMENT;
          F.err_axis = kMsgTemperature;
        }
      }
    }
    F.m_init = cfg.warm_m > 0 ? cfg.warm_m : min(cfg.M, s_count);
    *frame = F;
  }
}

// mt19937_64 (the C++ standard's parameters), top 53 bits -> [0,1) (rng.hpp:22).
__global__ void mt_uniforms_kernel(uint64_t seed, int n, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  constexpr int NN = 312, MM = 156;
  constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  uint64_t mt[NN];
  mt[0] = seed;
  for (int i = 1; i < NN; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
  int idx = NN;
  for (int k = 0; k < n; ++k) {
    if (idx >= NN) {
      for (int i = 0; i < NN; ++i) {
        const uint64_t xx = (mt[i] & UM) | (mt[(i + 1) % NN] & LM);
        uint64_t xa = xx >> 1;
        if (xx & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        mt[i] = mt[(i + MM) % NN] ^ xa;
      }
      idx = 0;
    }
    uint64_t y = mt[idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    out[k] = static_cast<double>(y >> 11) * 0x1.0p-53;
  }
}

// Per-cell warm-start component counts from a previous results buffer: a cell restarts
// from its previous model when that fit succeeded, else from the seeded random init.
__global__ void warm_m_kernel(int n_cells, const int32_t* status, const int32_t* comps, int32_t* m) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += gridDim.x * blockDim.x)
    m[c] = (!status || status[c] == 0) ? comps[c] : 0;
}

void launch_warm_m(vdfcg_ctx* ctx, int n_cells, const int32_t* status, const int32_t* comps,
                   int32_t* m) {
  const int grid = std::max(1, std::min((n_cells + 255) / 256, ctx->sm_count * 8));
  VDFCG_LAUNCH(ctx, "warm_m", warm_m_kernel<<<grid, 256, 0, ctx->stream>>>(n_cells, status, comps, m));
}

void launch_mt_uniforms(vdfcg_ctx* ctx, uint64_t seed, int n, double* out) {
  VDFCG_LAUNCH(ctx, "mt19937_64", mt_uniforms_kernel<<<1, 1, 0, ctx->stream>>>(seed, n, out));
}

__global__ void canonicalize_kernel(int d, int m, const double* w, const double* mu,
                                    const double* cov, const double* scale, const double* offset,
                                    double* ow, double* omu, double* ocov) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  bool ident = true;
  if (scale && offset)
    for (int a = 0; a < d; ++a) ident = ident && scale[a] == 1.0 && offset[a] == 0.0;
  for (int i = 0; i < m; ++i) {
    ow[i] = w[i];
    for (int a = 0; a < d; ++a)
      omu[i * d + a] = ident ? mu[i * d + a] : __dadd_rn(__dmul_rn(mu[i * d + a], scale[a]), offset[a]);
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) {
        const double c = cov[(i * d + a) * d + b];
        ocov[(i * d + a) * d + b] = ident ? c : __dmul_rn(__dmul_rn(scale[a], c), scale[b]);
      }
    for (int a = 1; a < d; ++a)
      for (int b = 0; b < a; ++b) ocov[(i * d + a) * d + b] = ocov[(i * d + b) * d + a];
  }
}

void launch_canonicalize(vdfcg_ctx* ctx, int d, int m, const double* w, const double* mu,
                         const double* cov, const double* scale, const double* offset,
                         double* ow, double* omu, double* ocov) {
  VDFCG_LAUNCH(ctx, "canonicalize",
               canonicalize_kernel<<<1, 1, 0, ctx->stream>>>(d, m, w, mu, cov, scale, offset, ow,
                                                             omu, ocov));
}

// Warps per fit. Small fits (the cfg4 regime, <= ~4K non-empty bins) get one warp each:
// the per-iteration serial part (M-step, protocol) then stalls only its own warp while
// the other resident fits keep the FP64 pipe busy. Larger fits get up to 8 warps, and
// few fits are widened so the grid still fills every SM. Depends on the input shape only.
static int choose_warps(double pts_per_fit, int n_fits, int sm_count) {
  int G = 1;
  while (G < 8 && pts_per_fit / (32.0 * G) > 128.0) G *= 2;
  while (G < 8 && double(n_fits) * G < sm_count * 12.0 && pts_per_fit / (32.0 * G) > 8.0) G *= 2;
  return G;
}

void launch_em_cells(vdfcg_ctx* ctx, int d, const KeyCells& kc, const EmConfig& cfg,
                          const EmOut& out, double avg_particles, int shape_fits) {
  if (kc.n_cells == 0) return;
  const int K = std::max(std::max(cfg.M, cfg.warm_m), cfg.cell_warm_m ? cfg.cell_warm_K : 0);
  double bins = 1.0;
  for (int a = 0; a < d; ++a) bins *= kc.n_bins;
  const double est = std::min(bins, avg_particles);
  const int fits = shape_fits > 0 ? shape_fits : kc.n_cells;
  const int G = choose_warps(est, fits, ctx->sm_count);
  // Fewer cells than ~2 CTAs per SM, each with many bins: spread every cell over a
  // cluster of CTAs (~1K points each, <= 16) so the grid still fills the GPU; depends on
  // the input shape only (results are bitwise reproducible for a given shape)
  KeyCells k2 = kc;
  int cl = 1;
  if (fits < 2 * ctx->sm_count) {
    // est bounds the non-empty bins from above; ~half of them is the typical occupancy
    cl = static_cast<int>(std::min<double>(16.0, std::ceil(0.5 * est / (G * 32.0 * 4.0))));
    cl = std::min(cl, (2 * ctx->sm_count + fits - 1) / fits);
    if (cl <= 2) cl = 1;  // measured: 2-CTA clusters lose to one CTA (cfg3 2.55 vs 1.88 ms)
  }
  // VDFCG_EM_SHAPE="G,cl": force warps per CTA and CTAs per cell (measurements only)
  int Gs = G;
  if (const char* e = getenv("VDFCG_EM_SHAPE")) {
    int g2 = 0, c2 = 0;
    if (sscanf(e, "%d,%d", &g2, &c2) == 2 && g2 >= 1 && g2 <= 8 && c2 >= 1 && c2 <= 16) {
      Gs = g2;
      cl = c2;
    }
  }
  k2.cluster = cl;
  CoordArgs ca{};
  if (d == 2) launch_em_dim2(ctx, true, K, k2, ca, cfg, out, kc.n_cells, Gs, kc.n_bins);
  else launch_em_dim3(ctx, true, K, k2, ca, cfg, out, kc.n_cells, Gs, kc.n_bins);
}

void launch_fit_prologue(vdfcg_ctx* ctx, int d, const double* pts, const double* w, int64_t n,
                         double total_weight, const EmConfig& cfg, double* z, Frame* fr) {
  if (d == 2)
    VDFCG_LAUNCH(ctx, "fit_prologue",
                 fit_prologue_kernel<2><<<1, 1024, 0, ctx->stream>>>(pts, w, n, total_weight, cfg, z, fr));
  else
    VDFCG_LAUNCH(ctx, "fit_prologue",
                 fit_prologue_kernel<3><<<1, 1024, 0, ctx->stream>>>(pts, w, n, total_weight, cfg, z, fr));
}

void launch_em_points(vdfcg_ctx* ctx, int d, const double* pts, const double* w, int64_t n,
                      double total_weight, const EmConfig& cfg, const EmOut& out) {
  double* z = arena<double>(ctx, static_cast<size_t>(std::max<int64_t>(n, 1)) * d);
  Frame* fr = arena<Frame>(ctx, 1);
  launch_fit_prologue(ctx, d, pts, w, n, total_weight, cfg, z, fr);
  const int K = std::max(cfg.M, cfg.warm_m);
  // one fit: the widest CTA the register budget allows
  const int G = 8;
  CoordArgs ca{z, n, w, fr};
  KeyCells kc{};
  kc.n_cells = 1;
  if (d == 2) launch_em_dim2(ctx, false, K, kc, ca, cfg, out, 1, G, 0);
  else launch_em_dim3(ctx, false, K, kc, ca, cfg, out, 1, G, 0);
}

std::string prologue_message(int status, int id, double value, bool fit_prefix) {
  (void)status;
  char buf[256];
  if (id >= kMsgZeroSpread && id < kMsgZeroSpread + 3) {
    // std::ostream default formatting (6 significant digits) == %g
    std::snprintf(buf, sizeof(buf), "%sdegenerate data: axis %d has zero spread (all values %g)",
                  fit_prefix ? "fit: " : "", id - kMsgZeroSpread, value);
    return buf;
  }
  switch (id) {
    case kMsgEmpty: return std::string(fit_prefix ? "fit: " : "") + "weighted points: empty";
    case kMsgNegWeight:
      return std::string(fit_prefix ? "fit: " : "") + "weighted points: weights must be >= 0";
    case kMsgNoPosWeight:
      return std::string(fit_prefix ? "fit: " : "") +
             "weighted points: at least one weight must be > 0";
    case kMsgTemperature: return "temperature must be a positive per-axis variance";
    case kMsgDegenerateHist: return "degenerate histogram: no in-range weight";
    case kMsgAllDegenerate: return "all mixture components are degenerate";
    case kMsgInvalidMass: return "m_step: invalid responsibility mass";
    default: return "fit failed";
  }
}

}  // namespace vdfcg
