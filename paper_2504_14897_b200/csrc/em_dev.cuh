// em_dev.cuh — per-component EM device logic shared by the fused batched fitter
// (em.cu) and the fine-grained drop-in entry points (em_entry.cu), so that
// vdfcg_e_step / vdfcg_m_step / vdfcg_prune_one / vdfcg_init_model exercise exactly
// the code the fused kernel runs.
#pragma once

#include "common.cuh"
#include "em.cuh"
#include "linalg.cuh"

namespace vdfcg {

// E-step component preparation (wgmm.cpp:197-229 + gaussian.hpp:9-42): Cholesky of the
// covariance (row-major 3x3 slot cov9), in-place repair when it fails. Returns false
// for a dead (unrepairable) component. Lo = {L10, L20, L21}, rd = 1/diag(L),
// cst = -0.5 (d log 2pi + log det) + log alpha.
template <int D>
VDFCG_DEV bool prep_component(double* cov9, double alpha, double* Lo, double* rd, double* cst) {
  Sym3 C, L;
#pragma unroll
  for (int e = 0; e < 9; ++e) C.a[e] = cov9[e];
  bool ok = cholesky<D>(C, L);
  if (!ok) {
    Sym3 R;
    int db;
    if (repair_covariance<D>(C, R, &db)) {
      symmetrize_from_upper<D>(R);
#pragma unroll
      for (int e = 0; e < 9; ++e) cov9[e] = R.a[e];
      ok = cholesky<D>(R, L);
    }
  }
  if (!ok) {
    *cst = -dinf();
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      rd[a] = 0.0;
      Lo[a] = 0.0;
    }
    return false;
  }
  double logdet_half = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    rd[a] = 1.0 / L(a, a);
    logdet_half += log(L(a, a));
  }
  Lo[0] = D >= 2 ? L(1, 0) : 0.0;
  Lo[1] = D >= 3 ? L(2, 0) : 0.0;
  Lo[2] = D >= 3 ? L(2, 1) : 0.0;
  const double la = alpha > 0.0 ? log(alpha) : -dinf();
  *cst = -0.5 * (D * kLog2Pi + 2.0 * logdet_half) + la;
  return true;
}

// log N(z | mu, L) + log alpha for one component (prepared by prep_component).
template <int D>
VDFCG_DEV double comp_logp(const double* z, const double* mu, const double* Lo, const double* rd,
                           double cst) {
  double y0, y1 = 0.0, y2 = 0.0;
  y0 = (z[0] - mu[0]) * rd[0];
  if (D >= 2) y1 = ((z[1] - mu[1]) - Lo[0] * y0) * rd[1];
  if (D >= 3) y2 = ((z[2] - mu[2]) - Lo[1] * y0 - Lo[2] * y1) * rd[2];
  double q = y0 * y0;
  if (D >= 2) q += y1 * y1;
  if (D >= 3) q += y2 * y2;
  return cst - 0.5 * q;
}

// Model arrays: alpha[K], mu[K*D], cov[K*9] (3x3 slots).
template <int D>
VDFCG_DEV void remove_component(double* alpha, double* mu, double* cov, int& m, int idx) {
  for (int j = idx; j + 1 < m; ++j) {
    alpha[j] = alpha[j + 1];
#pragma unroll
    for (int a = 0; a < D; ++a) mu[j * D + a] = mu[(j + 1) * D + a];
#pragma unroll
    for (int e = 0; e < 9; ++e) cov[j * 9 + e] = cov[(j + 1) * 9 + e];
  }
  --m;
}

// Rescale to unit sum by the sequential sum in component order (wgmm.cpp:331-332).
VDFCG_DEV void renormalize(double* alpha, int m) {
  double total = 0.0;
  for (int j = 0; j < m; ++j) total = __dadd_rn(total, alpha[j]);
  for (int j = 0; j < m; ++j) alpha[j] = alpha[j] / total;
}

// prune_one (wgmm.cpp:320-333): smallest weight (ties -> lowest index), strictly below
// the threshold, only while more than one component remains.
template <int D>
VDFCG_DEV bool prune_one_dev(double* alpha, double* mu, double* cov, int& m, double thr,
                             int* idx, double* weight) {
  if (m <= 1) return false;
  int sm = 0;
  for (int i = 1; i < m; ++i)
    if (alpha[i] < alpha[sm]) sm = i;
  if (!(alpha[sm] < thr)) return false;
  *idx = sm;
  *weight = alpha[sm];
  remove_component<D>(alpha, mu, cov, m, sm);
  renormalize(alpha, m);
  return true;
}

// init_model (wgmm.cpp:136-191) given the frame (normalization, bounding box of the
// normalized points, temperature, min(M, distinct)). Returns M.
template <int D>
VDFCG_DEV int init_model_dev(const Frame& F, const EmConfig& cfg, double* alpha, double* mu,
                             double* cov) {
  if (cfg.warm_m > 0) {  // warm start: re-express the canonical model in this frame
    double Dv[3];
#pragma unroll
    for (int a = 0; a < D; ++a) Dv[a] = 1.0 / F.scale[a];
    for (int i = 0; i < cfg.warm_m; ++i) {
      alpha[i] = cfg.warm_w[i];
#pragma unroll
      for (int a = 0; a < D; ++a)
        mu[i * D + a] = __dsub_rn(cfg.warm_mu[i * D + a], F.offset[a]) / F.scale[a];
      Sym3 cv;
#pragma unroll
      for (int e = 0; e < 9; ++e) cv.a[e] = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b)
          cv(a, b) = __dmul_rn(__dmul_rn(Dv[a], cfg.warm_cov[(i * D + a) * D + b]), Dv[b]);
      symmetrize_from_upper<D>(cv);
#pragma unroll
      for (int e = 0; e < 9; ++e) cov[i * 9 + e] = cv.a[e];
    }
    return cfg.warm_m;
  }
  const int m = F.m_init;
  for (int i = 0; i < m; ++i) {
    alpha[i] = 1.0 / m;
#pragma unroll
    for (int a = 0; a < D; ++a)
      mu[i * D + a] = __dadd_rn(F.zlo[a], __dmul_rn(__dsub_rn(F.zhi[a], F.zlo[a]), cfg.uniforms[i * D + a]));
#pragma unroll
    for (int e = 0; e < 9; ++e) cov[i * 9 + e] = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) cov[i * 9 + a * 3 + a] = F.temp[a] / __dmul_rn(F.scale[a], F.scale[a]);
  }
  return m;
}

// Number of distinct rows among the first points of z (SoA [D][n]), stopping at M
// (only "distinct < M" matters, wgmm.cpp:166-172). Executed by one full warp; list is
// a shared [16][3] scratch. Returns the count to every lane.
template <int D>
VDFCG_DEV int count_distinct_warp(const double* z, int64_t n, int M, double (*list)[3]) {
  const int lane = threadIdx.x & 31;
  int count = 0;
  for (int64_t b = 0; b < n && count < M; b += 32) {
    const int64_t p = b + lane;
    double zz[3] = {0, 0, 0};
    bool isnew = p < n;
    if (isnew) {
#pragma unroll
      for (int a = 0; a < D; ++a) zz[a] = z[a * n + p];
      for (int j = 0; j < count && isnew; ++j) {
        bool eq = true;
#pragma unroll
        for (int a = 0; a < D; ++a) eq = eq && (zz[a] == list[j][a]);
        if (eq) isnew = false;
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, isnew);
    while (mask && count < M) {
      const int l = __ffs(mask) - 1;
      double bz[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) bz[a] = __shfl_sync(0xffffffffu, zz[a], l);
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) list[count][a] = bz[a];
      }
      __syncwarp();
      ++count;
      if (lane > l && isnew) {
        bool eq = true;
#pragma unroll
        for (int a = 0; a < D; ++a) eq = eq && (zz[a] == bz[a]);
        if (eq) isnew = false;
      }
      if (lane == l) isnew = false;
      mask = __ballot_sync(0xffffffffu, isnew);
    }
  }
  return count;
}

}  // namespace vdfcg
