// em_kernel.cuh — the fused batched weighted-EM kernel (K5) as templates over the
// velocity dimension D and the component capacity K. Instantiated per D in em_d2.cu /
// em_d3.cu so the exact-K variants compile in parallel. See em.cu for the overview.
#pragma once

#include <cooperative_groups.h>
#include <cub/block/block_reduce.cuh>

#include <algorithm>

#include "common.cuh"
#include "em.cuh"
#include "em_dev.cuh"
#include "linalg.cuh"

namespace vdfcg {

template <int D>
struct NStat {
  static constexpr int value = 1 + D + D * (D + 1) / 2;
};

template <int D, int K>
struct EmState {
  static constexpr int NS = NStat<D>::value;
  static constexpr int KP = K;
  double alpha[K];
  double mu[K][D];
  double cov[K][9];
  double Lo[K][3];  // L(1,0), L(2,0), L(2,1)
  double rd[K][3];  // 1 / L(a,a)
  double cst[KP];   // -0.5 (d log 2pi + log det) + log alpha ; -inf when dead or padding
  double A[KP][6];  // L^-1 packed (affine form used by the point pass)
  double bv[KP][3]; // L^-1 mu
  double muc[KP][3];  // centre of the moment sums (mu_old, or mu_new in the exact pass)
  float Af[KP][6];    // FP32 E-step mode: the same affine form in single precision
  float bf[KP][3];
  float cstf[KP];
  double mu_new[K][D];
  double sig1[K][9];
  double st[K][NS];
  double st2[K][NS];
  double exp2tab[kExpTab];
  double logtab[256];
  double ll;
  double prev_ll;
  Frame fr;
  int m, status, err_id, converged, dead_mask, degen_mask, exact_mask, cert_mask, n_events,
      it_used, cell, stop;
  int minidx[3], maxidx[3];
};


template <int D>
struct KeySrc {
  // bin indices decoded once per fit (prologue) into packed fields: axis a at bit
  // a * SHIFT (10 bits for d=3, 16 for d=2), so the point pass only shifts and masks.
  static constexpr int SHIFT = D == 3 ? 10 : 16;
  static constexpr uint32_t MASK = (1u << SHIFT) - 1u;
  const uint32_t* keys;
  uint32_t* packed;
  const double* counts;
  int nb;
  const double* ztab;  // shared [D][nb]
  const float* ztabf;  // shared [D][nb], FP32 E-step mode
  VDFCG_DEV void load(int p, double (&z)[D], double& w) const {
    const uint32_t k = packed[p];
#pragma unroll
    for (int a = 0; a < D; ++a) z[a] = ztab[a * nb + ((k >> (SHIFT * a)) & MASK)];
    w = __ldg(counts + p);
  }
  VDFCG_DEV void load2(int p, double (&z)[D], float (&zf)[D], double& w) const {
    const uint32_t k = packed[p];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int t = a * nb + ((k >> (SHIFT * a)) & MASK);
      z[a] = ztab[t];
      zf[a] = ztabf[t];
    }
    w = __ldg(counts + p);
  }
};

template <int D>
struct CoordSrc {
  const double* z;
  int64_t n;
  const double* w;
  VDFCG_DEV void load(int p, double (&zz)[D], double& ww) const {
#pragma unroll
    for (int a = 0; a < D; ++a) zz[a] = __ldg(z + a * n + p);
    ww = __ldg(w + p);
  }
};

template <int D>
VDFCG_DEV constexpr int uidx(int a, int b) {  // packed upper index, a <= b
  return D == 2 ? (a == 0 ? b : 2) : (a == 0 ? b : (a == 1 ? 2 + b : 5));
}

// Thread-block cluster (single large fits): CL=true spreads one fit's points over the CTAs
// of a cluster; every CTA runs the (identical, deterministic) protocol and the partial
// sufficient statistics are combined through distributed shared memory.
template <bool CL>
VDFCG_DEV int cluster_rank() {
  if constexpr (CL) return static_cast<int>(cooperative_groups::this_cluster().block_rank());
  else return 0;
}
template <bool CL>
VDFCG_DEV int cluster_size() {
  if constexpr (CL) return static_cast<int>(cooperative_groups::this_cluster().num_blocks());
  else return 1;
}

// ---------------------------------------------------------------- the point pass
// EXACT=false: pass 1, statistics centred on mu_old (+ loglik). EXACT=true: the
// covariance sums centred on mu_new for the components flagged in exact_mask.
template <int D, int K, bool EXACT, bool CL, class Src>
VDFCG_DEV void em_pass(const Src& src, int n, EmState<D, K>& S, double* red) {
  constexpr int NS = NStat<D>::value;
  const int m = S.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = blockDim.x >> 5;
  constexpr int GPW = 32;  // points per warp per iteration (one per lane)
  double acc[K][NS];
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int t = 0; t < NS; ++t) acc[j][t] = 0.0;
  // Per-lane plain sum + the fixed-order tree below: the reference's Kahan sum
  // (gaussian.hpp:55-68) guards one sequential sum over all points; the error here stays
  // ~1e-15 relative either way.
  double ll = 0.0;
  // One point per lane, all K component slots. The loop is warp-uniform (a missing point
  // gets weight 0 and adds nothing). Slots >= m carry cst = -inf, A = b = 0, so they add
  // exactly nothing and are never read.
  const int crank = cluster_rank<CL>(), cn = cluster_size<CL>();
  for (int b0 = (crank * G + warp) * GPW; b0 < n; b0 += cn * G * GPW) {
    const int p = b0 + lane;
    const bool valid = p < n;
    double z[D], w;
    src.load(valid ? p : b0, z, w);
    if (!valid) w = 0.0;
    double lp[K];
#pragma unroll
    for (int j = 0; j < K; ++j) lp[j] = comp_logp2_affine<D>(z, S.A[j], S.bv[j], S.cst[j]);
    double mx = lp[0];  // slot 0 is always active (m >= 1)
#pragma unroll
    for (int j = 1; j < K; ++j) mx = lp[j] > mx ? lp[j] : mx;
#pragma unroll
    for (int j = 0; j < K; ++j) lp[j] = exp2_nonpos(lp[j] - mx, S.exp2tab);
    double sum = lp[0];
#pragma unroll
    for (int j = 1; j < K; ++j) sum += lp[j];
    if (!EXACT) ll += w * fma(mx, 0.6931471805599453, log_ge1(sum, S.logtab));
    const double ws = w * rcp_newton(sum);
    if (!EXACT) {
      // Pass 1 accumulates about the frame origin (z is the normalised coordinate,
      // |z| <= 1): the D(D+1)/2 products are shared by every component. The M-step
      // turns the raw sums into Eq. 9 (Sigma = S/m - mu mu^T with mu = t/m, the
      // reference's own mean) and runs the exact pass where the cancellation could cost
      // more than ~1e-12 of the smallest eigenvalue.
      double zz[D * (D + 1) / 2];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b2 = a; b2 < D; ++b2) zz[uidx<D>(a, b2)] = z[a] * z[b2];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const double g = lp[j] * ws;
        acc[j][0] += g;
#pragma unroll
        for (int a = 0; a < D; ++a) acc[j][1 + a] = fma(g, z[a], acc[j][1 + a]);
#pragma unroll
        for (int u = 0; u < D * (D + 1) / 2; ++u) acc[j][1 + D + u] = fma(g, zz[u], acc[j][1 + D + u]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (!((S.exact_mask >> j) & 1)) continue;
        const double g = lp[j] * ws;
        double dl[D];
#pragma unroll
        for (int a = 0; a < D; ++a) dl[a] = z[a] - S.muc[j][a];
        acc[j][0] += g;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const double gd = g * dl[a];
          acc[j][1 + a] += gd;
#pragma unroll
          for (int b2 = a; b2 < D; ++b2) acc[j][1 + D + uidx<D>(a, b2)] += gd * dl[b2];
        }
      }
    }
  }
  // fixed-order reduction: lanes (reduce-scatter) -> warps -> cluster CTAs (ascending)
  constexpr int W = K * NS + 1;
  {  // reduce-scatter: each lane ends with ~2 of the K*NS+1 warp totals
    double v[K * NS + 1];
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
      for (int t = 0; t < NS; ++t) v[j * NS + t] = acc[j][t];
    v[K * NS] = EXACT ? 0.0 : ll;
    int start, count;
    warp_scatter_sum(v, lane, start, count);
#pragma unroll
    for (int j = 0; j < WarpScatter<K * NS + 1>::HOUT; ++j) {
      const int gi = start + j;
      if (j < count && (gi == K * NS ? !EXACT : gi / NS < m)) red[warp * W + gi] = v[j];
    }
  }
  if constexpr (CL) cooperative_groups::this_cluster().sync();  // every CTA's partials visible
  else __syncthreads();
  for (int t = threadIdx.x; t < W; t += blockDim.x) {
    if (t >= K * NS ? EXACT : t / NS >= m) continue;
    double sum = 0.0;
    for (int r = 0; r < cn; ++r) {  // CTAs in rank order, then warps: fixed summation order
      const double* rr = red;
      if constexpr (CL) rr = cooperative_groups::this_cluster().map_shared_rank(red, r);
      for (int g = 0; g < G; ++g) sum += rr[g * W + t];
    }
    if (t >= K * NS) S.ll = sum;
    else if (EXACT) S.st2[t / NS][t % NS] = sum;
    else S.st[t / NS][t % NS] = sum;
  }
  if constexpr (CL) cooperative_groups::this_cluster().sync();  // remote reads done
  else __syncthreads();
}

// FP32 E-step mode (FitConfig.estep_fp32, tolerance 1e-4): log-densities, the
// log-sum-exp (MUFU ex2/lg2/rcp) and the responsibilities in single precision; the
// weighted sufficient statistics and the log-likelihood are still accumulated in FP64
// about the frame origin, and the M-step / exact pass / protocol are unchanged FP64.
VDFCG_DEV float ex2f_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
VDFCG_DEV float lg2f_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int D, int K, class Src>
VDFCG_DEV void em_pass_f32(const Src& src, int n, EmState<D, K>& S, double* red) {
  constexpr int NS = NStat<D>::value;
  constexpr int KP = EmState<D, K>::KP;
  const int m = S.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = blockDim.x >> 5;
  double acc[KP][NS];
#pragma unroll
  for (int j = 0; j < KP; ++j)
#pragma unroll
    for (int t = 0; t < NS; ++t) acc[j][t] = 0.0;
  double ll = 0.0;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    double z[D], w;
    float zf[D];
    src.load2(p, z, zf, w);
    float u[KP];
    float mx = -__int_as_float(0x7f800000);
#pragma unroll
    for (int i = 0; i < KP; ++i) {
      const float y0 = fmaf(S.Af[i][0], zf[0], -S.bf[i][0]);
      float q = y0 * y0;
      if (D >= 2) {
        const float y1 = fmaf(S.Af[i][2], zf[1], fmaf(S.Af[i][1], zf[0], -S.bf[i][1]));
        q = fmaf(y1, y1, q);
      }
      if (D >= 3) {
        const float y2 = fmaf(S.Af[i][5], zf[2], fmaf(S.Af[i][4], zf[1], fmaf(S.Af[i][3], zf[0], -S.bf[i][2])));
        q = fmaf(y2, y2, q);
      }
      u[i] = S.cstf[i] - q;  // log2 domain (pre-scaled affine form)
      mx = u[i] > mx ? u[i] : mx;
    }
    float sum = 0.0f;
#pragma unroll
    for (int i = 0; i < KP; ++i) {
      u[i] = ex2f_approx(u[i] - mx);
      sum += u[i];
    }
    ll += w * (0.6931471805599453 * (static_cast<double>(mx) + static_cast<double>(lg2f_approx(sum))));
    const float inv = __frcp_rn(sum);
    double zz[D * (D + 1) / 2];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b2 = a; b2 < D; ++b2) zz[uidx<D>(a, b2)] = z[a] * z[b2];
#pragma unroll
    for (int i = 0; i < KP; ++i) {
      const double g = static_cast<double>(u[i] * inv) * w;
      acc[i][0] += g;
#pragma unroll
      for (int a = 0; a < D; ++a) acc[i][1 + a] = fma(g, z[a], acc[i][1 + a]);
#pragma unroll
      for (int t = 0; t < D * (D + 1) / 2; ++t) acc[i][1 + D + t] = fma(g, zz[t], acc[i][1 + D + t]);
    }
  }
  constexpr int W = K * NS + 1;
  {  // reduce-scatter (as in em_pass)
    double v[K * NS + 1];
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
      for (int t = 0; t < NS; ++t) v[j * NS + t] = acc[j][t];
    v[K * NS] = ll;
    int start, count;
    warp_scatter_sum(v, lane, start, count);
#pragma unroll
    for (int j = 0; j < WarpScatter<K * NS + 1>::HOUT; ++j) {
      const int gi = start + j;
      if (j < count && (gi == K * NS || gi / NS < m)) red[warp * W + gi] = v[j];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < W; t += blockDim.x) {
    if (t < K * NS) {
      const int i = t / NS;
      if (i >= m) continue;
      double sum = 0.0;
      for (int g = 0; g < G; ++g) sum += red[g * W + t];
      S.st[i][t % NS] = sum;
    } else {
      double sum = 0.0;
      for (int g = 0; g < G; ++g) sum += red[g * W + t];
      S.ll = sum;
    }
  }
  __syncthreads();
}

template <int D>
VDFCG_DEV void load_cov(const double* c9, Sym3& s) {
#pragma unroll
  for (int e = 0; e < 9; ++e) s.a[e] = c9[e];
}

// The init configuration of cell c: its own warm model when the per-cell warm buffers say
// so (time series), else the shared config (shared warm model or seeded random init).
template <int D>
VDFCG_DEV EmConfig cell_config(const EmConfig& cfg, int c) {
  EmConfig e = cfg;
  if (cfg.cell_warm_m && cfg.cell_warm_m[c] > 0) {
    const int64_t base = static_cast<int64_t>(c) * cfg.cell_warm_K;
    e.warm_m = cfg.cell_warm_m[c];
    e.warm_w = cfg.cell_warm_w + base;
    e.warm_mu = cfg.cell_warm_mu + base * D;
    e.warm_cov = cfg.cell_warm_cov + base * D * D;
  }
  return e;
}

// ---------------------------------------------------------------- the fit
template <int D, int K, bool F32, bool CL, class Src>
VDFCG_DEV void run_fit(const Src& src, int n, EmState<D, K>& S, double* red, const EmConfig& cfg,
                       const EmOut& out, int c) {
  const bool writer = cluster_rank<CL>() == 0;  // one CTA of a cluster writes the results
  constexpr int NS = NStat<D>::value;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ---- init (wgmm.cpp:136-191)
  if (threadIdx.x == 0) {
    S.n_events = 0;
    S.converged = 0;
    S.stop = 0;
    S.it_used = 0;
    S.prev_ll = dnan();
    if (!S.status) {
      const EmConfig ec = cell_config<D>(cfg, c);
      S.m = init_model_dev<D>(S.fr, ec, S.alpha, &S.mu[0][0], &S.cov[0][0]);
    }
  }
  __syncthreads();

  for (int it = 1; it <= cfg.max_it && !S.status; ++it) {
    // ---- E-step preparation: one lane per component (wgmm.cpp:197-229)
    if (warp == 0) {
      bool dead = false;
      if (lane < S.m) {
        dead = !prep_component<D>(S.cov[lane], S.alpha[lane], S.Lo[lane], S.rd[lane], &S.cst[lane]);
        affine_from_chol<D>(S.mu[lane], S.Lo[lane], S.rd[lane], S.A[lane], S.bv[lane]);
#pragma unroll
        for (int e = 0; e < 6; ++e) S.A[lane][e] *= kSqrtHalfLog2E;
#pragma unroll
        for (int a = 0; a < 3; ++a) S.bv[lane][a] *= kSqrtHalfLog2E;
        S.cst[lane] *= kLog2E;
#pragma unroll
        for (int a = 0; a < D; ++a) S.muc[lane][a] = S.mu[lane][a];
        if constexpr (F32) {  // single-precision copy for the FP32 E-step only
#pragma unroll
          for (int e = 0; e < 6; ++e) S.Af[lane][e] = static_cast<float>(S.A[lane][e]);
#pragma unroll
          for (int a = 0; a < 3; ++a) S.bf[lane][a] = static_cast<float>(S.bv[lane][a]);
          S.cstf[lane] = static_cast<float>(S.cst[lane]);
        }
      } else if (lane < EmState<D, K>::KP) {  // inactive / padding slot: contributes zero
        if constexpr (F32) {
#pragma unroll
          for (int e = 0; e < 6; ++e) S.Af[lane][e] = 0.0f;
#pragma unroll
          for (int a = 0; a < 3; ++a) S.bf[lane][a] = 0.0f;
          S.cstf[lane] = -__int_as_float(0x7f800000);
        }
        S.cst[lane] = -dinf();
#pragma unroll
        for (int e = 0; e < 6; ++e) S.A[lane][e] = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          S.bv[lane][a] = 0.0;
          S.muc[lane][a] = 0.0;
        }
      }
      const unsigned dm = __ballot_sync(0xffffffffu, dead);
      if (lane == 0) {
        S.dead_mask = static_cast<int>(dm);
        if (S.m > 0 && __popc(dm) == S.m) {
          S.status = VDFCG_RUNTIME_ERROR;
          S.err_id = kMsgAllDegenerate;
        }
      }
    }
    __syncthreads();
    if (S.status) break;

    // ---- E-step + sufficient statistics (one pass over the points)
    if constexpr (F32) em_pass_f32<D, K>(src, n, S, red);
    else em_pass<D, K, false, CL>(src, n, S, red);

    // ---- M-step part 1 (wgmm.cpp:269-298)
    if (warp == 0) {
      bool bad = false, need = false, cert = false;
      if (lane < S.m) {
        const int i = lane;
        const double mass = S.st[i][0];
        bad = !isfinite(mass) || mass < 0.0;
        const bool starved = !(mass > S.fr.total * kMassFloorRel);
        if (!bad && !starved) {
          const double inv = 1.0 / mass;
          double mn[D];
          double dd = 0.0;  // squared distance of the new mean from the accumulation origin
#pragma unroll
          for (int a = 0; a < D; ++a) {
            mn[a] = S.st[i][1 + a] * inv;
            S.mu_new[i][a] = mn[a];
            dd += mn[a] * mn[a];
          }
          Sym3 s1;
#pragma unroll
          for (int e = 0; e < 9; ++e) s1.a[e] = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = a; b < D; ++b)
              s1(a, b) = S.st[i][1 + D + uidx<D>(a, b)] * inv - mn[a] * mn[b];
          symmetrize_from_upper<D>(s1);
#pragma unroll
          for (int e = 0; e < 9; ++e) S.sig1[i][e] = s1.a[e];
          // Raw moments lose ~eps*|mu|^2 absolute; recompute Eq. 9 around the new mean
          // whenever that could exceed ~1e-12 of the smallest eigenvalue (lmin >= lb) or
          // the LLT fails, so the collapse test and the parameters see reference numerics.
          const double lb = lmin_lower_bound<D>(s1);
          need = !(lb > 0.0) || dd > 1e4 * lb;
          cert = lb > 1e-14 * trace3<D>(s1);
        }
      }
      const unsigned bm = __ballot_sync(0xffffffffu, bad);
      const unsigned nm = __ballot_sync(0xffffffffu, need);
      const unsigned cm = __ballot_sync(0xffffffffu, cert);
      if (lane == 0) {
        S.exact_mask = static_cast<int>(nm);
        S.cert_mask = static_cast<int>(cm);
        if (bm) {
          S.status = VDFCG_RUNTIME_ERROR;
          S.err_id = kMsgInvalidMass;
        }
      }
    }
    __syncthreads();
    if (S.status) break;
    if (S.exact_mask) {
      if (threadIdx.x == 0 && writer && cfg.exact_counter) atomicAdd(cfg.exact_counter, 1ull);
      if (warp == 0 && lane < S.m && ((S.exact_mask >> lane) & 1)) {
#pragma unroll
        for (int a = 0; a < D; ++a) S.muc[lane][a] = S.mu_new[lane][a];
      }
      __syncthreads();
      em_pass<D, K, true, CL>(src, n, S, red);
    }

    // ---- M-step part 2: covariances, collapse test, repair (wgmm.cpp:299-316)
    if (warp == 0) {
      bool degen = false;
      if (lane < S.m) {
        const int i = lane;
        const double mass = S.st[i][0];
        S.alpha[i] = mass / S.fr.total;
        const bool starved = !(mass > S.fr.total * kMassFloorRel);
        if (!starved) {
          Sym3 sg;
          bool certified;
          if ((S.exact_mask >> i) & 1) {
#pragma unroll
            for (int e = 0; e < 9; ++e) sg.a[e] = 0.0;
            const double inv = 1.0 / mass;
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
              for (int b = a; b < D; ++b) sg(a, b) = S.st2[i][1 + D + uidx<D>(a, b)] * inv;
            symmetrize_from_upper<D>(sg);
            certified = lmin_lower_bound<D>(sg) > 1e-14 * trace3<D>(sg);
          } else {
            load_cov<D>(S.sig1[i], sg);
            certified = (S.cert_mask >> i) & 1;
          }
#pragma unroll
          for (int a = 0; a < D; ++a) S.mu[i][a] = S.mu_new[i][a];
          Sym3 acc;
          if (certified) {
#pragma unroll
            for (int e = 0; e < 9; ++e) S.cov[i][e] = sg.a[e];
          } else if (accept_covariance<D>(sg, acc)) {
#pragma unroll
            for (int e = 0; e < 9; ++e) S.cov[i][e] = acc.a[e];
          } else {
            degen = true;
          }
        }
      }
      const unsigned gm = __ballot_sync(0xffffffffu, degen);
      if (lane == 0) S.degen_mask = static_cast<int>(gm);
    }
    __syncthreads();

    // ---- protocol: removal, pruning, convergence (wgmm.cpp:383-417), thread 0
    if (threadIdx.x == 0) {
      const double ll = S.ll;
      if (writer && out.trace && it - 1 < out.trace_cap)
        out.trace[static_cast<int64_t>(c) * out.trace_cap + (it - 1)] = ll;
      const int mask = S.dead_mask | S.degen_mask;
      bool pruned = false;
      for (int i = S.m - 1; i >= 0; --i) {
        if (!((mask >> i) & 1)) continue;
        if (S.m <= 1) break;
        if (writer && out.ev_it && S.n_events < out.K) {
          const int64_t e = static_cast<int64_t>(c) * out.K + S.n_events;
          out.ev_it[e] = it;
          out.ev_comp[e] = i;
          out.ev_w[e] = S.alpha[i];
        }
        ++S.n_events;
        remove_component<D>(S.alpha, &S.mu[0][0], &S.cov[0][0], S.m, i);
        pruned = true;
      }
      if (pruned) renormalize(S.alpha, S.m);
      if (it % cfg.interval == 0) {  // prune_one, wgmm.cpp:320-333
        int idx = -1;
        double wgt = 0.0;
        if (prune_one_dev<D>(S.alpha, &S.mu[0][0], &S.cov[0][0], S.m, cfg.prune_thr, &idx, &wgt)) {
          if (writer && out.ev_it && S.n_events < out.K) {
            const int64_t e = static_cast<int64_t>(c) * out.K + S.n_events;
            out.ev_it[e] = it;
            out.ev_comp[e] = idx;
            out.ev_w[e] = wgt;
          }
          ++S.n_events;
          pruned = true;
        }
      }
      S.it_used = it;
      if (!pruned && isfinite(S.prev_ll) && fabs(ll - S.prev_ll) < cfg.tol * fabs(S.prev_ll)) {
        S.converged = 1;
        S.stop = 1;
      }
      S.prev_ll = pruned ? dnan() : ll;
    }
    __syncthreads();
    if (S.stop) break;
  }

  // ---- epilogue: denormalize (wgmm.cpp:102-120) and write
  if (!writer) return;
  const int K_out = out.K;
  const int64_t base = static_cast<int64_t>(c) * K_out;
  if (S.status == 0) {
    bool ident = true;
#pragma unroll
    for (int a = 0; a < D; ++a) ident = ident && S.fr.scale[a] == 1.0 && S.fr.offset[a] == 0.0;
    for (int i = threadIdx.x; i < S.m; i += blockDim.x) {
      out.w[base + i] = S.alpha[i];
      Sym3 cv;
      load_cov<D>(S.cov[i], cv);
      if (!ident) {
        Sym3 t;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b < D; ++b)
            t(a, b) = __dmul_rn(__dmul_rn(S.fr.scale[a], cv(a, b)), S.fr.scale[b]);
        symmetrize_from_upper<D>(t);
        cv = t;
      }
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double v = ident ? S.mu[i][a] : __dadd_rn(__dmul_rn(S.mu[i][a], S.fr.scale[a]), S.fr.offset[a]);
        out.mu[(base + i) * D + a] = v;
#pragma unroll
        for (int b = 0; b < D; ++b) out.cov[((base + i) * D + a) * D + b] = cv(a, b);
      }
    }
  }
  // slots past the fitted components (and every slot of a failed cell) are zeroed, so
  // result buffers are fully defined and bitwise reproducible
  for (int i = (S.status == 0 ? S.m : 0) + threadIdx.x; i < K_out; i += blockDim.x) {
    out.w[base + i] = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      out.mu[(base + i) * D + a] = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) out.cov[((base + i) * D + a) * D + b] = 0.0;
    }
  }
  if (threadIdx.x == 0) {
    out.status[c] = S.status;
    out.comps[c] = S.status ? 0 : S.m;
    out.iters[c] = S.status ? 0 : min(S.it_used, cfg.max_it);
    out.conv[c] = S.status ? 0 : S.converged;
    out.final_ll[c] = S.status ? dnan() : S.ll;
    if (out.n_events) out.n_events[c] = S.status ? 0 : min(S.n_events, K_out);
    if (out.err_axis) out.err_axis[c] = S.status ? S.err_id : -1;
    if (out.err_value) out.err_value[c] = S.fr.err_value;
  }
  (void)NS;
}

// ---------------------------------------------------------------- prologues
// Histogram-derived cell: normalize over the occupied bins, z tables, temperature.
template <int D, int K>
VDFCG_DEV int key_prologue(const KeyCells& kc, int c, const EmConfig& cfg, EmState<D, K>& S,
                           double* ztab, double* red, KeySrc<D>& src) {
  const int nb = kc.n_bins;
  const int64_t base = kc.offsets[c];
  const int n = kc.nnz[c];
  src.keys = kc.keys + base;
  src.counts = kc.counts + base;
  src.nb = nb;
  src.packed = kc.packed + base;
  src.ztab = ztab;
  src.ztabf = reinterpret_cast<const float*>(ztab + D * nb);
  if (threadIdx.x == 0) {
    S.status = 0;
    S.err_id = -1;
    S.fr.err_value = 0.0;
    for (int a = 0; a < 3; ++a) {
      S.minidx[a] = nb;
      S.maxidx[a] = -1;
    }
  }
  __syncthreads();
  const bool cell_warm = cfg.warm_m > 0 || (cfg.cell_warm_m && cfg.cell_warm_m[c] > 0);
  const bool need_temp = !cfg.has_temp && !cell_warm;
  double sw = 0.0, sx[3] = {0, 0, 0}, sxx[3] = {0, 0, 0};
  int mn[3] = {nb, nb, nb}, mxi[3] = {-1, -1, -1};
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    uint32_t k = __ldg(src.keys + p);
    int idx[3];
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const uint32_t q = k / static_cast<uint32_t>(nb);
      idx[a] = static_cast<int>(k - q * static_cast<uint32_t>(nb));
      k = q;
    }
    {
      uint32_t pk = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) pk |= static_cast<uint32_t>(idx[a]) << (KeySrc<D>::SHIFT * a);
      src.packed[p] = pk;
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
      mn[a] = min(mn[a], idx[a]);
      mxi[a] = max(mxi[a], idx[a]);
    }
    if (need_temp) {
      const double w = __ldg(src.counts + p);
      sw += w;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double x = bin_center(kc.lo[a], kc.hi[a], nb, idx[a]);
        const double xw = x * w;
        sx[a] += xw;
        sxx[a] += xw * x;
      }
    }
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    mn[a] = warp_min(mn[a]);
    mxi[a] = warp_max(mxi[a]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = blockDim.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      atomicMin(&S.minidx[a], mn[a]);
      atomicMax(&S.maxidx[a], mxi[a]);
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
      red[warp * 8 + 0] = sw;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        red[warp * 8 + 1 + a] = sx[a];
        red[warp * 8 + 4 + a] = sxx[a];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Frame& F = S.fr;
    const double total = kc.in_range[c];
    F.total = total;
    F.status = 0;
    if (n <= 0 || !(total > 0.0)) {
      S.status = VDFCG_INVALID_ARGUMENT;
      S.err_id = kMsgDegenerateHist;
    } else {
      for (int a = 0; a < D; ++a) {
        const double lo = bin_center(kc.lo[a], kc.hi[a], nb, S.minidx[a]);
        const double hi = bin_center(kc.lo[a], kc.hi[a], nb, S.maxidx[a]);
        F.offset[a] = __dmul_rn(0.5, __dadd_rn(lo, hi));
        F.scale[a] = __dmul_rn(0.5, __dsub_rn(hi, lo));
      }
      for (int a = 0; a < D; ++a) {
        if (!(F.scale[a] > 0.0)) {
          S.status = VDFCG_INVALID_ARGUMENT;
          S.err_id = kMsgZeroSpread + a;
          F.err_value = bin_center(kc.lo[a], kc.hi[a], nb, S.minidx[a]);
          break;
        }
      }
      if (!S.status) {
        if (cfg.has_temp) {
          for (int a = 0; a < D; ++a) F.temp[a] = cfg.temp[a];
        } else if (!cell_warm) {
          double tsw = 0.0, tsx[3] = {0, 0, 0}, tsxx[3] = {0, 0, 0};
          for (int g = 0; g < G; ++g) {
            tsw += red[g * 8];
            for (int a = 0; a < D; ++a) {
              tsx[a] += red[g * 8 + 1 + a];
              tsxx[a] += red[g * 8 + 4 + a];
            }
          }
          for (int a = 0; a < D; ++a) {
            const double mean = tsx[a] / tsw;
            const double var = fmax(tsxx[a] / tsw - mean * mean, 0.0);
            F.temp[a] = var;
            if (!(var > 0.0)) {
              S.status = VDFCG_INVALID_ARGUMENT;
              S.err_id = kMsgTemperature;
            }
          }
        }
        F.m_init = min(cfg.M, n);  // bin centres are distinct points (wgmm.cpp:166-172)
      }
    }
  }
  __syncthreads();
  if (S.status) return n;
  for (int t = threadIdx.x; t < D * nb; t += blockDim.x) {
    const int a = t / nb, i = t - a * nb;
    ztab[t] = __dsub_rn(bin_center(kc.lo[a], kc.hi[a], nb, i), S.fr.offset[a]) / S.fr.scale[a];
    reinterpret_cast<float*>(ztab + D * nb)[t] = static_cast<float>(ztab[t]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int a = 0; a < D; ++a) {
      S.fr.zlo[a] = ztab[a * nb + S.minidx[a]];
      S.fr.zhi[a] = ztab[a * nb + S.maxidx[a]];
    }
  }
  __syncthreads();
  return n;
}

template <int D, int K, bool KEYS, bool F32 = false, bool CLU = false>
// Register caps measured on 48^3 cells: K = 4 at 128 (112: 578 ms, 120: 555, 128: 538,
// 136: 637, 152: 547 per cfg4 species); K = 3 at 128 (104: 224, 112: 218, 128: 201 ms per
// 131072 cells); K <= 2 at 80 (K=2: 72: 63.6, 80: 59.9, 88: 62.0, 128: 63.5 ms); K >= 5 at
// 255 (K=8: 200: 337, 224: 326, 255: 240 ms per 65536 cells).
#ifndef VDFCG_EM_MAXREG_K1
#define VDFCG_EM_MAXREG_K1 80
#endif
#ifndef VDFCG_EM_MAXREG_K2
#define VDFCG_EM_MAXREG_K2 80
#endif
#ifndef VDFCG_EM_MAXREG_K3
#define VDFCG_EM_MAXREG_K3 128
#endif
#ifndef VDFCG_EM_MAXREG_K4
#define VDFCG_EM_MAXREG_K4 128
#endif
__global__ void __launch_bounds__(256) __maxnreg__(K == 1 ? VDFCG_EM_MAXREG_K1 : K == 2 ? VDFCG_EM_MAXREG_K2 : K == 3 ? VDFCG_EM_MAXREG_K3 : (K <= 4 ? VDFCG_EM_MAXREG_K4 : 255)) em_kernel(KeyCells kc, CoordArgs ca, EmConfig cfg,
                                                 EmOut out, int* counter, int red_stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EmState<D, K>& S = *reinterpret_cast<EmState<D, K>*>(smem_raw);
  constexpr size_t st_bytes = (sizeof(EmState<D, K>) + 15) & ~size_t(15);
  double* red = reinterpret_cast<double*>(smem_raw + st_bytes);
  double* ztab = red + (blockDim.x >> 5) * red_stride;
  const int n_cells = KEYS ? kc.n_cells : 1;
  for (int j = threadIdx.x; j < kExpTab; j += blockDim.x) S.exp2tab[j] = kExp2Tab[j];
  for (int j = threadIdx.x; j < 256; j += blockDim.x) S.logtab[j] = kLogTab[j];
  for (int pass = 0;; ++pass) {
    // cells: persistent CTAs pull fits from a queue; a single fit (!KEYS) is processed once
    // by every CTA of the cluster
    // (cells on clusters: one cell per cluster, one pass)
    if (KEYS && !CLU && threadIdx.x == 0) S.cell = atomicAdd(counter, 1);
    __syncthreads();
    const int c = KEYS ? (CLU ? (pass == 0 ? static_cast<int>(blockIdx.x) / cluster_size<CLU>() : n_cells) : S.cell)
                       : pass;
    if (c >= n_cells) break;
    if (KEYS) {
      KeySrc<D> src;
      const int n = key_prologue<D, K>(kc, c, cfg, S, ztab, red, src);
      run_fit<D, K, F32, CLU>(src, n, S, red, cfg, out, c);
    } else {
      if (threadIdx.x == 0) {
        S.fr = *ca.frame;
        S.status = S.fr.status;
        S.err_id = S.fr.err_axis;
      }
      __syncthreads();
      CoordSrc<D> src{ca.z, ca.n, ca.w};
      if (S.status) {
        if (threadIdx.x == 0 && cluster_rank<CLU>() == 0) {
          out.status[c] = S.status;
          out.comps[c] = 0;
          out.iters[c] = 0;
          out.conv[c] = 0;
          out.final_ll[c] = dnan();
          if (out.n_events) out.n_events[c] = 0;
          if (out.err_axis) out.err_axis[c] = S.err_id;
          if (out.err_value) out.err_value[c] = S.fr.err_value;
        }
      } else {
        run_fit<D, K, false, CLU>(src, static_cast<int>(ca.n), S, red, cfg, out, c);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- host launch
template <int D, int K, bool KEYS, bool F32>
void launch_em_tf(vdfcg_ctx* ctx, const KeyCells& kc, const CoordArgs& ca,
                  const EmConfig& cfg, const EmOut& out, int n_cells, int G, int n_bins) {
  constexpr int NS = NStat<D>::value;
  const int red_stride = std::max(K * NS + 1, 8);
  const size_t st = (sizeof(EmState<D, K>) + 15) & ~size_t(15);
  // z tables: FP64 [D][nb] + FP32 [D][nb]
  const size_t smem = st + size_t(G) * red_stride * 8 + (KEYS ? size_t(D) * n_bins * 12 : 0);
  auto k = em_kernel<D, K, KEYS, F32>;
  VDFCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int occ = 0;
  VDFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, G * 32, smem));
  if (occ < 1) throw CudaError("EM kernel cannot be resident (registers/shared memory)");
  int* counter = arena<int>(ctx, 1);
  VDFCG_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), ctx->stream));
  if constexpr (!KEYS) {
    // one fit: a cluster of CTAs, ~4 points per lane each, at most 16 (non-portable size);
    // up to ~8 points per lane a single CTA without cluster barriers is faster (measured:
    // 1684 points 0.47 ms alone vs 0.49 ms on two CTAs; 12.7K points 1.59 ms on 13 CTAs)
    const int64_t per_cta = int64_t(G) * 32 * 4;
    int cl = static_cast<int>(std::min<int64_t>(16, std::max<int64_t>(1, (ca.n + per_cta - 1) / per_cta)));
    if (cl <= 2) cl = 1;
    if (cl == 1) {
      VDFCG_LAUNCH(ctx, "em_fit", k<<<1, G * 32, smem, ctx->stream>>>(kc, ca, cfg, out, counter, red_stride));
      return;
    }
    auto kc2 = em_kernel<D, K, KEYS, F32, true>;
    VDFCG_CUDA(cudaFuncSetAttribute(kc2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (cl > 8) VDFCG_CUDA(cudaFuncSetAttribute(kc2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cl);
    lc.blockDim = dim3(G * 32);
    lc.dynamicSmemBytes = smem;
    lc.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    VDFCG_LAUNCH(ctx, "em_fit", cudaLaunchKernelEx(&lc, kc2, kc, ca, cfg, out, counter, red_stride));
  } else {
    const int cl = F32 ? 1 : std::min(16, std::max(1, kc.cluster));
    if (cl > 1) {  // few, large cells: one cell per cluster of `cl` CTAs
      auto kc2 = em_kernel<D, K, KEYS, F32, true>;
      VDFCG_CUDA(cudaFuncSetAttribute(kc2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      if (cl > 8) VDFCG_CUDA(cudaFuncSetAttribute(kc2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(n_cells * cl);
      lc.blockDim = dim3(G * 32);
      lc.dynamicSmemBytes = smem;
      lc.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      VDFCG_LAUNCH(ctx, "em_fit", cudaLaunchKernelEx(&lc, kc2, kc, ca, cfg, out, counter, red_stride));
      return;
    }
    const int grid = std::max(1, std::min(n_cells, ctx->sm_count * occ));
    VDFCG_LAUNCH(ctx, "em_fit",
                 k<<<grid, G * 32, smem, ctx->stream>>>(kc, ca, cfg, out, counter, red_stride));
  }
}

template <int D, int K, bool KEYS>
void launch_em_t(vdfcg_ctx* ctx, const KeyCells& kc, const CoordArgs& ca,
                 const EmConfig& cfg, const EmOut& out, int n_cells, int G, int n_bins) {
  if constexpr (KEYS) {
    if (cfg.f32) {
      launch_em_tf<D, K, true, true>(ctx, kc, ca, cfg, out, n_cells, G, n_bins);
      return;
    }
  }
  launch_em_tf<D, K, KEYS, false>(ctx, kc, ca, cfg, out, n_cells, G, n_bins);
}

template <int D, bool KEYS>
void launch_em_k(vdfcg_ctx* ctx, int K, const KeyCells& kc, const CoordArgs& ca,
                 const EmConfig& cfg, const EmOut& out, int n_cells, int G, int n_bins) {
  switch (K) {  // exact capacities for the common sizes, next larger otherwise
    case 1: launch_em_t<D, 1, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins); break;
    case 2: launch_em_t<D, 2, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins); break;
    case 3: launch_em_t<D, 3, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins); break;
    case 4: launch_em_t<D, 4, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins); break;
    case 5: launch_em_t<D, 5, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins); break;
    case 6: launch_em_t<D, 6, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins); break;
    case 7:
    case 8: launch_em_t<D, 8, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins); break;
    case 9: case 10: case 11:
    case 12: launch_em_t<D, 12, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins); break;
    default: launch_em_t<D, 16, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins); break;
  }
}

// Warps per fit: enough lanes that each holds ~16 points per pass, and enough CTAs in
// flight to fill every SM; deterministic in the input shape only.

}  // namespace vdfcg
