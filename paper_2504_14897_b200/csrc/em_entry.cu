// em_entry.cu — device kernels behind the fine-grained drop-in entry points
// (wgmm.hpp:74-120: init_model, e_step, m_step, prune_one, repair_covariance). They
// run the same per-component device logic as the fused fitter (em_dev.cuh).
#include <cub/block/block_reduce.cuh>

#include "em_dev.cuh"
#include "em_entry.cuh"

namespace vdfcg {

// model arrays in the ABI layout (d x d blocks) <-> 3x3 slots
template <int D>
VDFCG_DEV void cov_in(const double* c, int i, double* c9) {
#pragma unroll
  for (int e = 0; e < 9; ++e) c9[e] = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) c9[a * 3 + b] = c[(i * D + a) * D + b];
}
template <int D>
VDFCG_DEV void cov_out(const double* c9, int i, double* c) {
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) c[(i * D + a) * D + b] = c9[a * 3 + b];
}

// ------------------------------------------------------------------ init_model
template <int D>
__global__ void __launch_bounds__(1024) init_model_kernel(const double* __restrict__ z, int64_t n,
                                                          EmConfig cfg, Frame F, double* w_out,
                                                          double* mu_out, double* cov_out_p,
                                                          int* m_out) {
  __shared__ double s_min[32][3], s_max[32][3];
  __shared__ double s_list[kMaxK][3];
  __shared__ int s_count;
  __shared__ double alpha[kMaxK], mu[kMaxK * 3], cov[kMaxK * 9];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = blockDim.x >> 5;
  double lo[3] = {dinf(), dinf(), dinf()}, hi[3] = {-dinf(), -dinf(), -dinf()};
  for (int64_t p = threadIdx.x; p < n; p += blockDim.x)
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double v = z[a * n + p];
      lo[a] = fmin(lo[a], v);
      hi[a] = fmax(hi[a], v);
    }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lo[a] = warp_min(lo[a]);
    hi[a] = warp_max(hi[a]);
    if (lane == 0) {
      s_min[warp][a] = lo[a];
      s_max[warp][a] = hi[a];
    }
  }
  if (warp == 0) {
    const int cnt = count_distinct_warp<D>(z, n, cfg.warm_m > 0 ? 0 : cfg.M, s_list);
    if (lane == 0) s_count = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int a = 0; a < D; ++a) {
      double l = s_min[0][a], h = s_max[0][a];
      for (int g = 1; g < G; ++g) {
        l = fmin(l, s_min[g][a]);
        h = fmax(h, s_max[g][a]);
      }
      F.zlo[a] = l;
      F.zhi[a] = h;
    }
    F.m_init = min(cfg.M, s_count);
    const int m = init_model_dev<D>(F, cfg, alpha, mu, cov);
    for (int i = 0; i < m; ++i) {
      w_out[i] = alpha[i];
      for (int a = 0; a < D; ++a) mu_out[i * D + a] = mu[i * D + a];
      cov_out<D>(cov + i * 9, i, cov_out_p);
    }
    *m_out = m;
  }
}

void launch_init_model(vdfcg_ctx* ctx, int d, const double* z, int64_t n, const EmConfig& cfg,
                       const Frame& f, double* w, double* mu, double* cov, int* m_out) {
  if (d == 2)
    VDFCG_LAUNCH(ctx, "init_model", init_model_kernel<2><<<1, 1024, 0, ctx->stream>>>(z, n, cfg, f, w, mu, cov, m_out));
  else
    VDFCG_LAUNCH(ctx, "init_model", init_model_kernel<3><<<1, 1024, 0, ctx->stream>>>(z, n, cfg, f, w, mu, cov, m_out));
}

// ------------------------------------------------------------------ e_step
struct CompConst {
  double mu[3], Lo[3], rd[3], cst;
};

template <int D>
__global__ void estep_prep_kernel(int m, const double* alpha, const double* mu, double* cov,
                                  CompConst* cc, int* dead_list, int* n_dead) {
  const int lane = threadIdx.x;
  bool dead = false;
  if (lane < m) {
    double c9[9];
    cov_in<D>(cov, lane, c9);
    CompConst k{};
    dead = !prep_component<D>(c9, alpha[lane], k.Lo, k.rd, &k.cst);
    for (int a = 0; a < D; ++a) k.mu[a] = mu[lane * D + a];
    cc[lane] = k;
    cov_out<D>(c9, lane, cov);  // in-place repair is visible to the caller (wgmm.hpp:94-97)
  }
  const unsigned dm = __ballot_sync(0xffffffffu, dead);
  if (lane == 0) {
    int k = 0;
    for (int i = 0; i < m; ++i)
      if ((dm >> i) & 1) dead_list[k++] = i;
    *n_dead = k;
  }
}

template <int D>
__global__ void __launch_bounds__(256) estep_points_kernel(const double* __restrict__ x,
                                                           const double* __restrict__ w, int64_t n,
                                                           int m, const CompConst* __restrict__ cc,
                                                           double* __restrict__ resp,
                                                           double* partial) {
  __shared__ CompConst sc[kMaxK];
  __shared__ double red[8];
  if (threadIdx.x < m) sc[threadIdx.x] = cc[threadIdx.x];
  __syncthreads();
  Kahan ll;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double z[D];
#pragma unroll
    for (int a = 0; a < D; ++a) z[a] = x[a * n + p];
    double lp[kMaxK];
    double mx = -dinf();
    for (int i = 0; i < m; ++i) {
      lp[i] = comp_logp<D>(z, sc[i].mu, sc[i].Lo, sc[i].rd, sc[i].cst);
      mx = fmax(mx, lp[i]);
    }
    double s = 0.0;
    for (int i = 0; i < m; ++i) {
      lp[i] = exp(lp[i] - mx);
      s += lp[i];
    }
    for (int i = 0; i < m; ++i) resp[i + p * m] = lp[i] / s;
    ll.add(w[p] * (mx + log(s)));
  }
  const double v = warp_sum(ll.value());
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int g = 0; g < static_cast<int>(blockDim.x >> 5); ++g) t += red[g];
    partial[blockIdx.x] = t;
  }
}

__global__ void sum_partials_kernel(const double* partial, int n, double* out) {
  if (threadIdx.x == 0) {
    Kahan k;
    for (int i = 0; i < n; ++i) k.add(partial[i]);
    *out = k.value();
  }
}

void launch_e_step(vdfcg_ctx* ctx, int d, int m, const double* alpha, const double* mu,
                   double* cov, const double* x, const double* w, int64_t n, double* resp,
                   double* loglik, int* dead_list, int* n_dead) {
  CompConst* cc = arena<CompConst>(ctx, kMaxK);
  if (d == 2)
    VDFCG_LAUNCH(ctx, "e_step", estep_prep_kernel<2><<<1, 32, 0, ctx->stream>>>(m, alpha, mu, cov, cc, dead_list, n_dead));
  else
    VDFCG_LAUNCH(ctx, "e_step", estep_prep_kernel<3><<<1, 32, 0, ctx->stream>>>(m, alpha, mu, cov, cc, dead_list, n_dead));
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, ctx->sm_count * 4)));
  double* partial = arena<double>(ctx, grid);
  if (d == 2)
    VDFCG_LAUNCH(ctx, "e_step", estep_points_kernel<2><<<grid, 256, 0, ctx->stream>>>(x, w, n, m, cc, resp, partial));
  else
    VDFCG_LAUNCH(ctx, "e_step", estep_points_kernel<3><<<grid, 256, 0, ctx->stream>>>(x, w, n, m, cc, resp, partial));
  VDFCG_LAUNCH(ctx, "e_step", sum_partials_kernel<<<1, 32, 0, ctx->stream>>>(partial, grid, loglik));
}

// ------------------------------------------------------------------ m_step
// One block per component; the reference's two-pass formulas (wgmm.cpp:277-298) with
// fixed-order block reductions, then the collapse test + repair (wgmm.cpp:300-315).
template <int D>
__global__ void __launch_bounds__(1024) mstep_kernel(const double* __restrict__ x,
                                                     const double* __restrict__ w, int64_t n,
                                                     double total, const double* __restrict__ resp,
                                                     int m, const double* prev_mu,
                                                     const double* prev_cov, double* out_w,
                                                     double* out_mu, double* out_cov, int* degen,
                                                     int* bad) {
  using Reduce = cub::BlockReduce<double, 1024>;
  __shared__ typename Reduce::TempStorage rs;
  __shared__ double s_mass, s_mu[3];
  const int i = blockIdx.x;
  double part = 0.0;
  for (int64_t p = threadIdx.x; p < n; p += blockDim.x) part += resp[i + p * m] * w[p];
  const double mass = Reduce(rs).Sum(part);
  if (threadIdx.x == 0) s_mass = mass;
  __syncthreads();
  const double M = s_mass;
  if (!isfinite(M) || M < 0.0) {
    if (threadIdx.x == 0) atomicOr(bad, 1);
    return;
  }
  const bool starved = !(M > total * kMassFloorRel);
  if (threadIdx.x == 0) {
    out_w[i] = M / total;
    degen[i] = 0;
  }
  if (starved) {
    if (threadIdx.x == 0) {
      for (int a = 0; a < D; ++a) out_mu[i * D + a] = prev_mu[i * D + a];
      for (int e = 0; e < D * D; ++e) out_cov[i * D * D + e] = prev_cov[i * D * D + e];
    }
    return;
  }
  for (int a = 0; a < D; ++a) {
    double s = 0.0;
    for (int64_t p = threadIdx.x; p < n; p += blockDim.x) s += x[a * n + p] * (resp[i + p * m] * w[p]);
    __syncthreads();
    const double t = Reduce(rs).Sum(s);
    if (threadIdx.x == 0) s_mu[a] = t / M;
  }
  __syncthreads();
  double sg[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t p = threadIdx.x; p < n; p += blockDim.x) {
    const double wi = resp[i + p * m] * w[p];
    double c[3];
#pragma unroll
    for (int a = 0; a < D; ++a) c[a] = x[a * n + p] - s_mu[a];
    int k = 0;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = a; b < D; ++b) sg[k++] += (c[a] * wi) * c[b];
  }
  double tot[6];
  int k = 0;
  for (int a = 0; a < D; ++a)
    for (int b = a; b < D; ++b, ++k) {
      __syncthreads();
      tot[k] = Reduce(rs).Sum(sg[k]);
    }
  if (threadIdx.x == 0) {
    Sym3 sig;
    for (int e = 0; e < 9; ++e) sig.a[e] = 0.0;
    k = 0;
    for (int a = 0; a < D; ++a)
      for (int b = a; b < D; ++b, ++k) sig(a, b) = tot[k] / M;
    symmetrize_from_upper<D>(sig);
    for (int a = 0; a < D; ++a) out_mu[i * D + a] = s_mu[a];
    Sym3 acc;
    if (accept_covariance<D>(sig, acc)) {
      cov_out<D>(acc.a, i, out_cov);
    } else {
      for (int e = 0; e < D * D; ++e) out_cov[i * D * D + e] = prev_cov[i * D * D + e];
      degen[i] = 1;
    }
  }
}

void launch_m_step(vdfcg_ctx* ctx, int d, const double* x, const double* w, int64_t n,
                   double total, const double* resp, int m, const double* prev_mu,
                   const double* prev_cov, double* out_w, double* out_mu, double* out_cov,
                   int* degen, int* bad) {
  if (m == 0) return;
  if (d == 2)
    VDFCG_LAUNCH(ctx, "m_step", mstep_kernel<2><<<m, 1024, 0, ctx->stream>>>(x, w, n, total, resp, m, prev_mu, prev_cov, out_w, out_mu, out_cov, degen, bad));
  else
    VDFCG_LAUNCH(ctx, "m_step", mstep_kernel<3><<<m, 1024, 0, ctx->stream>>>(x, w, n, total, resp, m, prev_mu, prev_cov, out_w, out_mu, out_cov, degen, bad));
}

// ------------------------------------------------------------------ prune_one / repair
template <int D>
__global__ void prune_kernel(double* alpha, double* mu, double* cov, int* m_io, double thr,
                             int* pruned, int* idx, double* weight) {
  double c9[kMaxK * 9];
  int m = *m_io;
  for (int i = 0; i < m; ++i) cov_in<D>(cov, i, c9 + i * 9);
  int id = -1;
  double wt = 0.0;
  const bool p = prune_one_dev<D>(alpha, mu, c9, m, thr, &id, &wt);
  for (int i = 0; i < m; ++i) cov_out<D>(c9 + i * 9, i, cov);
  *m_io = m;
  *pruned = p ? 1 : 0;
  *idx = id;
  *weight = wt;
}

void launch_prune_one(vdfcg_ctx* ctx, int d, double* alpha, double* mu, double* cov, int* m_io,
                      double thr, int* pruned, int* idx, double* weight) {
  if (d == 2)
    VDFCG_LAUNCH(ctx, "prune_one", prune_kernel<2><<<1, 1, 0, ctx->stream>>>(alpha, mu, cov, m_io, thr, pruned, idx, weight));
  else
    VDFCG_LAUNCH(ctx, "prune_one", prune_kernel<3><<<1, 1, 0, ctx->stream>>>(alpha, mu, cov, m_io, thr, pruned, idx, weight));
}

template <int D>
__global__ void repair_kernel(const double* sigma, double* out, int* doublings, int* ok) {
  Sym3 s, r;
  for (int e = 0; e < 9; ++e) s.a[e] = 0.0;
  for (int a = 0; a < D; ++a)
    for (int b = 0; b < D; ++b) s(a, b) = sigma[a * D + b];
  int db = -1;
  const bool good = repair_covariance<D>(s, r, &db);
  *ok = good ? 1 : 0;
  *doublings = db;
  if (good)
    for (int a = 0; a < D; ++a)
      for (int b = 0; b < D; ++b) out[a * D + b] = r(a, b);
}

void launch_repair(vdfcg_ctx* ctx, int d, const double* sigma, double* out, int* doublings,
                   int* ok) {
  if (d == 1) {
    VDFCG_LAUNCH(ctx, "repair", repair_kernel<1><<<1, 1, 0, ctx->stream>>>(sigma, out, doublings, ok));
  } else if (d == 2) {
    VDFCG_LAUNCH(ctx, "repair", repair_kernel<2><<<1, 1, 0, ctx->stream>>>(sigma, out, doublings, ok));
  } else {
    VDFCG_LAUNCH(ctx, "repair", repair_kernel<3><<<1, 1, 0, ctx->stream>>>(sigma, out, doublings, ok));
  }
}

}  // namespace vdfcg
