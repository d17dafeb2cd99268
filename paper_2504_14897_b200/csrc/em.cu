// em.cu — K5: the batched weighted-EM fitter (sm_100a, FP64 CUDA cores).
//
// One CTA of G warps owns one fit (a spatial cell, or the single point set of
// vdfcg_fit) at a time and pulls the next one from an atomic queue (persistent grid).
// Per fit, entirely on-device (wgmm.cpp:364-423):
//   prologue   normalize over the non-empty bins (wgmm.cpp:78-100), temperature
//              (wgmm.cpp:22-25), seeded init or warm start (wgmm.cpp:136-191)
//   iteration  lanes of warp 0 factor every component (LLT + in-place repair,
//              wgmm.cpp:197-229); all threads stream the points once: log-density via
//              the Cholesky factor, per-point log-sum-exp, responsibilities and the
//              weighted sufficient statistics (mass, sum g(x-mu_old), sum g(x-mu_old)^2)
//              in registers; fixed-order warp-shuffle + cross-warp reduction (bitwise
//              reproducible); M-step per component lane (Eq. 9 with the NEW mean via the
//              shifted sums; an exact second pass centred on the new mean when the shift
//              would cost precision, see need_exact below), collapse test + repair
//              (wgmm.cpp:300-315); thread 0 runs degenerate removal, scheduled pruning
//              and the convergence test (wgmm.cpp:386-417) on the E-step log-likelihood
//   epilogue   denormalize (wgmm.cpp:102-120) and write parameters + diagnostics.
// Points never leave L1/L2 between iterations of a fit; parameters live in shared memory.
#include <cub/block/block_reduce.cuh>

#include <algorithm>
#include <cstdio>
#include <string>

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
  double alpha[K];
  double mu[K][D];
  double cov[K][9];
  double Lo[K][3];  // L(1,0), L(2,0), L(2,1)
  double rd[K][3];  // 1 / L(a,a)
  double cst[K];    // -0.5 (d log 2pi + log det) + log alpha ; -inf when dead
  double A[K][6];   // L^-1 packed (affine form used by the point pass)
  double bv[K][3];  // L^-1 mu
  double mu_new[K][D];
  double sig1[K][9];
  double st[K][NS];
  double st2[K][NS];
  double exp2tab[64];
  double ll;
  double prev_ll;
  Frame fr;
  int m, status, err_id, converged, dead_mask, degen_mask, exact_mask, cert_mask, n_events,
      it_used, cell, stop;
  int minidx[3], maxidx[3];
};

struct CoordArgs {
  const double* z;  // SoA normalized points [D][n]
  int64_t n;
  const double* w;
  const Frame* frame;
};

template <int D>
struct KeySrc {
  const uint32_t* keys;
  const double* counts;
  int nb;
  uint32_t magic;      // ceil(2^32 / nb): exact quotient for keys < 2^32 / nb (nb <= 255)
  const double* ztab;  // shared [D][nb]
  VDFCG_DEV void load(int p, double (&z)[D], double& w) const {
    uint32_t k = __ldg(keys + p);
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const uint32_t q = magic ? __umulhi(k, magic) : k / static_cast<uint32_t>(nb);
      const uint32_t idx = k - q * static_cast<uint32_t>(nb);
      z[a] = ztab[a * nb + idx];
      k = q;
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

// ---------------------------------------------------------------- the point pass
// EXACT=false: pass 1, statistics centred on mu_old (+ loglik). EXACT=true: the
// covariance sums centred on mu_new for the components flagged in exact_mask.
template <int D, int K, bool EXACT, class Src>
VDFCG_DEV void em_pass(const Src& src, int n, EmState<D, K>& S, double* red) {
  constexpr int NS = NStat<D>::value;
  const int m = S.m;
  double acc[K][NS];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < NS; ++j) acc[i][j] = 0.0;
  Kahan ll;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    double z[D], w;
    src.load(p, z, w);
    double lp[K];
    double mx = -dinf();
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i < m) {
        lp[i] = comp_logp_affine<D>(z, S.A[i], S.bv[i], S.cst[i]);
        mx = fmax(mx, lp[i]);
      }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i < m) {
        lp[i] = exp_nonpos(lp[i] - mx, S.exp2tab);
        s += lp[i];
      }
    }
    if (!EXACT) ll.add(w * (mx + log(s)));
    const double ws = w * rcp_newton(s);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i < m) {
        if (EXACT && !((S.exact_mask >> i) & 1)) continue;
        const double g = lp[i] * ws;
        double dl[D];
#pragma unroll
        for (int a = 0; a < D; ++a) dl[a] = z[a] - (EXACT ? S.mu_new[i][a] : S.mu[i][a]);
        acc[i][0] += g;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const double gd = g * dl[a];
          acc[i][1 + a] += gd;
#pragma unroll
          for (int b = a; b < D; ++b) acc[i][1 + D + uidx<D>(a, b)] += gd * dl[b];
        }
      }
    }
  }
  // fixed-order reduction: lanes (xor tree) -> warps (ascending)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, G = blockDim.x >> 5;
  constexpr int W = K * NS + 1;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    if (i < m) {
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const double v = warp_sum(acc[i][j]);
        if (lane == 0) red[warp * W + i * NS + j] = v;
      }
    }
  }
  if (!EXACT) {
    const double v = warp_sum(ll.value());
    if (lane == 0) red[warp * W + K * NS] = v;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < W; t += blockDim.x) {
    if (t < K * NS) {
      const int i = t / NS;
      if (i >= m) continue;
      double sum = 0.0;
      for (int g = 0; g < G; ++g) sum += red[g * W + t];
      if (EXACT) S.st2[i][t % NS] = sum; else S.st[i][t % NS] = sum;
    } else if (!EXACT) {
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

// ---------------------------------------------------------------- the fit
template <int D, int K, class Src>
VDFCG_DEV void run_fit(const Src& src, int n, EmState<D, K>& S, double* red, const EmConfig& cfg,
                       const EmOut& out, int c) {
  constexpr int NS = NStat<D>::value;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ---- init (wgmm.cpp:136-191)
  if (threadIdx.x == 0) {
    S.n_events = 0;
    S.converged = 0;
    S.stop = 0;
    S.it_used = 0;
    S.prev_ll = dnan();
    if (!S.status) S.m = init_model_dev<D>(S.fr, cfg, S.alpha, &S.mu[0][0], &S.cov[0][0]);
  }
  __syncthreads();

  for (int it = 1; it <= cfg.max_it && !S.status; ++it) {
    // ---- E-step preparation: one lane per component (wgmm.cpp:197-229)
    if (warp == 0) {
      bool dead = false;
      if (lane < S.m) {
        dead = !prep_component<D>(S.cov[lane], S.alpha[lane], S.Lo[lane], S.rd[lane], &S.cst[lane]);
        affine_from_chol<D>(S.mu[lane], S.Lo[lane], S.rd[lane], S.A[lane], S.bv[lane]);
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
    em_pass<D, K, false>(src, n, S, red);

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
          double db[D];
          double dd = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            db[a] = S.st[i][1 + a] * inv;
            S.mu_new[i][a] = S.mu[i][a] + db[a];
            dd += db[a] * db[a];
          }
          Sym3 s1;
#pragma unroll
          for (int e = 0; e < 9; ++e) s1.a[e] = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = a; b < D; ++b)
              s1(a, b) = S.st[i][1 + D + uidx<D>(a, b)] * inv - db[a] * db[b];
          symmetrize_from_upper<D>(s1);
#pragma unroll
          for (int e = 0; e < 9; ++e) S.sig1[i][e] = s1.a[e];
          // The shifted form loses ~eps*|d|^2 absolute; recompute Eq. 9 around the new
          // mean whenever that could reach 1e-12 of the smallest eigenvalue (or the LLT
          // fails), so the collapse test sees reference-grade numerics. lmin >= lb.
          const double lb = lmin_lower_bound<D>(s1);
          need = !(lb > 0.0) || dd > 1e3 * lb;
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
    if (S.exact_mask) em_pass<D, K, true>(src, n, S, red);

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
      if (out.trace && it - 1 < out.trace_cap)
        out.trace[static_cast<int64_t>(c) * out.trace_cap + (it - 1)] = ll;
      const int mask = S.dead_mask | S.degen_mask;
      bool pruned = false;
      for (int i = S.m - 1; i >= 0; --i) {
        if (!((mask >> i) & 1)) continue;
        if (S.m <= 1) break;
        if (out.ev_it && S.n_events < out.K) {
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
          if (out.ev_it && S.n_events < out.K) {
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
  // n^d * (magic*n - 2^32) < 2^32 keeps umulhi exact for every key (holds for n <= 255)
  src.magic = (D == 3 ? nb <= 255 : nb <= 1625) ? static_cast<uint32_t>((0x100000000ULL + nb - 1) / nb) : 0u;
  src.ztab = ztab;
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
  const bool need_temp = !cfg.has_temp && cfg.warm_m == 0;
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
        } else if (cfg.warm_m == 0) {
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

template <int D, int K, bool KEYS>
__global__ void __launch_bounds__(256, (K <= 4 ? 2 : 1)) em_kernel(KeyCells kc, CoordArgs ca, EmConfig cfg,
                                                 EmOut out, int* counter, int red_stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EmState<D, K>& S = *reinterpret_cast<EmState<D, K>*>(smem_raw);
  constexpr size_t st_bytes = (sizeof(EmState<D, K>) + 15) & ~size_t(15);
  double* red = reinterpret_cast<double*>(smem_raw + st_bytes);
  double* ztab = red + (blockDim.x >> 5) * red_stride;
  const int n_cells = KEYS ? kc.n_cells : 1;
  for (int j = threadIdx.x; j < 64; j += blockDim.x) S.exp2tab[j] = kExp2Tab[j];
  for (;;) {
    if (threadIdx.x == 0) S.cell = atomicAdd(counter, 1);
    __syncthreads();
    const int c = S.cell;
    if (c >= n_cells) break;
    if (KEYS) {
      KeySrc<D> src;
      const int n = key_prologue<D, K>(kc, c, cfg, S, ztab, red, src);
      run_fit<D, K>(src, n, S, red, cfg, out, c);
    } else {
      if (threadIdx.x == 0) {
        S.fr = *ca.frame;
        S.status = S.fr.status;
        S.err_id = S.fr.err_axis;
      }
      __syncthreads();
      CoordSrc<D> src{ca.z, ca.n, ca.w};
      if (S.status) {
        if (threadIdx.x == 0) {
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
        run_fit<D, K>(src, static_cast<int>(ca.n), S, red, cfg, out, c);
      }
    }
    __syncthreads();
  }
}

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

// ---------------------------------------------------------------- host launchers
template <int D, int K, bool KEYS>
static void launch_em_t(vdfcg_ctx* ctx, const KeyCells& kc, const CoordArgs& ca,
                        const EmConfig& cfg, const EmOut& out, int n_cells, int G, int n_bins) {
  constexpr int NS = NStat<D>::value;
  const int red_stride = std::max(K * NS + 1, 8);
  const size_t st = (sizeof(EmState<D, K>) + 15) & ~size_t(15);
  const size_t smem = st + size_t(G) * red_stride * 8 + (KEYS ? size_t(D) * n_bins * 8 : 0);
  auto k = em_kernel<D, K, KEYS>;
  VDFCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int occ = 0;
  VDFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, G * 32, smem));
  if (occ < 1) throw CudaError("EM kernel cannot be resident (registers/shared memory)");
  const int grid = std::max(1, std::min(n_cells, ctx->sm_count * occ));
  int* counter = arena<int>(ctx, 1);
  VDFCG_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), ctx->stream));
  VDFCG_LAUNCH(ctx, "em_fit",
               k<<<grid, G * 32, smem, ctx->stream>>>(kc, ca, cfg, out, counter, red_stride));
}

template <int D, bool KEYS>
static void launch_em_k(vdfcg_ctx* ctx, int K, const KeyCells& kc, const CoordArgs& ca,
                        const EmConfig& cfg, const EmOut& out, int n_cells, int G, int n_bins) {
  if (K <= 2) launch_em_t<D, 2, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins);
  else if (K <= 4) launch_em_t<D, 4, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins);
  else if (K <= 8) launch_em_t<D, 8, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins);
  else launch_em_t<D, 16, KEYS>(ctx, kc, ca, cfg, out, n_cells, G, n_bins);
}

// Warps per fit: enough lanes that each holds ~16 points per pass, and enough CTAs in
// flight to fill every SM; deterministic in the input shape only.
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
                          const EmOut& out, double avg_particles) {
  if (kc.n_cells == 0) return;
  const int K = std::max(cfg.M, cfg.warm_m);
  double bins = 1.0;
  for (int a = 0; a < d; ++a) bins *= kc.n_bins;
  const double est = std::min(bins, avg_particles);
  const int G = choose_warps(est, kc.n_cells, ctx->sm_count);
  CoordArgs ca{};
  if (d == 2) launch_em_k<2, true>(ctx, K, kc, ca, cfg, out, kc.n_cells, G, kc.n_bins);
  else launch_em_k<3, true>(ctx, K, kc, ca, cfg, out, kc.n_cells, G, kc.n_bins);
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
  if (d == 2) launch_em_k<2, false>(ctx, K, kc, ca, cfg, out, 1, G, 0);
  else launch_em_k<3, false>(ctx, K, kc, ca, cfg, out, 1, G, 0);
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
