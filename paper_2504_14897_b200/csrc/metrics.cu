// metrics.cu — fit quality on the device.
//
// cell_metrics_kernel: one CTA per cell (grid-stride over cells) computes the
// reference's MetricsReport (pipeline.cpp:106-128) from the cell's compacted histogram
// and fitted model:
//   * model pdf on the full bins^d grid (evaluate_pdf, wgmm.cpp:425-453), reduced to
//     sum q (an exp-free recurrence along each innermost-axis row, see below) and
//     #(q > 0) (exact underflow intervals per row);
//   * a pass over the non-empty bins for kl_pq / kl_qp / jsd (metrics.cpp:12-46; bins
//     with p = 0 contribute  0.5 qn ln 2  to the JSD and make kl_qp divergent, so they
//     need only the full-grid sums), weighted_loglik (wgmm.cpp:257-267), the data
//     moments (wgmm.cpp:473-480) and, on thread 0, the mixture moments, bic and the
//     compression ratios (metrics.cpp:48-83).
// Reductions are fixed-order (warp xor trees, then warps in order): bitwise
// reproducible run to run.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "linalg.cuh"
#include "metrics.cuh"

namespace vdfcg {
namespace {

constexpr double kLn2 = 0.6931471805599453;
constexpr int kMB = 256;  // threads per metrics CTA

struct PrepComp {
  double w, logw, cst;  // cst = d ln 2pi + 2 sum ln L_kk (log_component_densities)
  double mu[3];
  double L[6];          // L10 L20 L21 (strict lower) then 1/L00 1/L11 1/L22
};

// Cholesky of one component; false when the LLT fails (llt_ok).
template <int D>
VDFCG_DEV bool prep_comp(double w, const double* mu, const double* cov, PrepComp& p) {
  Sym3 a, L;
#pragma unroll
  for (int i = 0; i < 9; ++i) a.a[i] = 0.0;
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int s = 0; s < D; ++s) a(r, s) = cov[r * D + s];
  if (!cholesky<D>(a, L)) return false;
  double ld = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) ld += log(L(k, k));
  p.w = w;
  p.logw = w > 0.0 ? log(w) : -dinf();
  p.cst = D * kLog2Pi + 2.0 * ld;
#pragma unroll
  for (int r = 0; r < 3; ++r) p.mu[r] = r < D ? mu[r] : 0.0;
  p.L[0] = L(1, 0);
  p.L[1] = D > 2 ? L(2, 0) : 0.0;
  p.L[2] = D > 2 ? L(2, 1) : 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) p.L[3 + k] = k < D ? 1.0 / L(k, k) : 0.0;
  return true;
}

// -0.5 (cst + |L^-1 (x - mu)|^2)  (gaussian.hpp:22-28 / log_component_densities)
template <int D>
VDFCG_DEV double log_gauss(const PrepComp& p, const double* x) {
  const double y0 = (x[0] - p.mu[0]) * p.L[3];
  const double y1 = (x[1] - p.mu[1] - p.L[0] * y0) * p.L[4];
  double q = y0 * y0 + y1 * y1;
  if (D > 2) {
    const double y2 = (x[2] - p.mu[2] - p.L[1] * y0 - p.L[2] * y1) * p.L[5];
    q += y2 * y2;
  }
  return -0.5 * (p.cst + q);
}

// x < this => exp(x) rounds to 0 (half the smallest subnormal, 2^-1075)
constexpr double kExpUnderflow = -745.1332191019411;

// Bin centres of the leading (d-1) axes of innermost-axis row `row`.
template <int D>
VDFCG_DEV void lead_coords(int64_t row, int nb, const double* lo, const double* dx, double* x) {
#pragma unroll
  for (int a = D - 2; a >= 0; --a) {
    const int i = static_cast<int>(row % nb);
    row /= nb;
    x[a] = __dadd_rn(lo[a], __dmul_rn(static_cast<double>(i) + 0.5, dx[a]));
  }
}

// Row-invariant part of the triangular solve: y_last = (x_last + base) * lin and the
// squared leading terms q0.
template <int D>
VDFCG_DEV void row_terms(const PrepComp& p, const double* x, double& base, double& lin, double& q0) {
  const double y0 = (x[0] - p.mu[0]) * p.L[3];
  if (D == 2) {
    base = -p.mu[1] - p.L[0] * y0;
    lin = p.L[4];
    q0 = y0 * y0;
  } else {
    const double y1 = (x[1] - p.mu[1] - p.L[0] * y0) * p.L[4];
    base = -p.mu[2] - p.L[1] * y0 - p.L[2] * y1;
    lin = p.L[5];
    q0 = y0 * y0 + y1 * y1;
  }
}

// Fixed-order block reduction of NV sums; every thread gets the totals in `v`.
template <int NV>
VDFCG_DEV void block_sum(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) red[warp * NV + i] = v[i];
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w * NV + threadIdx.x];
    red[32 * NV + threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = red[32 * NV + i];
  __syncthreads();
}

template <int D>
__global__ void __launch_bounds__(kMB) cell_metrics_kernel(CellsDev c, CellBinsDev b, CellModels r,
                                                           MetricsOut o) {
  __shared__ PrepComp comp[kMaxK];
  __shared__ double red[33 * 17];
  __shared__ double s_delta[kMaxK], s_rdelta[kMaxK], s_hh[kMaxK];
  __shared__ int s_ok;
  const int nb = c.n_bins;
  double dx[D], lo[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lo[a] = c.lo[a];
    dx[a] = (c.hi[a] - c.lo[a]) / static_cast<double>(nb);
  }
  double area = 1.0;
  int64_t total_bins = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    area *= dx[a];
    total_bins *= nb;
  }
  const int64_t rows = total_bins / nb;
  for (int cell = blockIdx.x; cell < c.n_cells; cell += gridDim.x) {
    const int M = r.comps[cell];
    const double in_range = b.in_range[cell];
    bool ok = r.status[cell] == 0 && M > 0 && M <= kMaxK && in_range > 0.0;
    if (threadIdx.x == 0) {  // GmmModel::validate (wgmm.cpp:46-63)
      double tot = 0.0;
      for (int i = 0; ok && i < M; ++i) {
        const double w = r.w[size_t(cell) * r.K + i];
        ok = w > 0.0;
        const double* cv = r.cov + (size_t(cell) * r.K + i) * D * D;
        for (int a = 0; a < D; ++a)
          for (int e = a + 1; e < D; ++e) ok = ok && cv[a * D + e] == cv[e * D + a];
        tot += w;
      }
      s_ok = ok && fabs(tot - 1.0) <= 1e-12;
    }
    __syncthreads();
    ok = s_ok;
    __syncthreads();
    if (ok && threadIdx.x < M) {
      const size_t ci = size_t(cell) * r.K + threadIdx.x;
      PrepComp& pc = comp[threadIdx.x];
      if (!prep_comp<D>(r.w[ci], r.mu + ci * D, r.cov + ci * D * D, pc)) {
        s_ok = 0;  // evaluate_pdf: "model component covariance is not SPD"
      } else {  // innermost-axis step of y and its recurrence factor, per component
        const double delta = dx[D - 1] * pc.L[3 + D - 1];
        s_delta[threadIdx.x] = delta;
        s_rdelta[threadIdx.x] = 1.0 / delta;
        s_hh[threadIdx.x] = exp(-delta * delta);
      }
    }
    __syncthreads();
    ok = s_ok;
    if (!ok) {
      if (threadIdx.x < kMetricFields && o.f[threadIdx.x]) o.f[threadIdx.x][cell] = dnan();
      __syncthreads();
      continue;
    }
    // ---- full grid: sum q and #(q > 0)
    double g[2] = {0.0, 0.0};
    const double dxl = dx[D - 1], lol = lo[D - 1];
    // (a) sum q over (row, component) items. Along the innermost axis the exponent is
    // quadratic in j, so exp(E(j+1)) = exp(E(j)) * g_j with g_{j+1} = g_j * h and
    // h = exp(-delta^2), delta = dx / L_dd: two multiplies per bin instead of an exp.
    // Each row walks out from the component's peak in both directions (values fall
    // monotonically, so nothing overflows), re-anchoring with a direct exp every 32
    // bins (relative error ~32^2 eps); a direction stops once its anchor underflows.
    for (int64_t item = threadIdx.x; item < rows * M; item += kMB) {
      // component-major items: the lanes of a warp walk consecutive rows of one component,
      // whose walk lengths (distance from the component's centre) are similar
      const int k = static_cast<int>(item / rows);
      const int64_t row = item - k * rows;
      double x[3];
      lead_coords<D>(row, nb, lo, dx, x);
      double base, lin, q0;
      row_terms<D>(comp[k], x, base, lin, q0);
      const double w = comp[k].w, c0 = comp[k].cst + q0;
      const double delta = s_delta[k], hh = s_hh[k], half = 0.5 * delta * delta;
      const double yfirst = (__dadd_rn(lol, __dmul_rn(0.5, dxl)) + base) * lin;
      const int js = static_cast<int>(fmin(fmax(rint(-yfirst * s_rdelta[k]), 0.0), double(nb - 1)));
      double sq = 0.0;
      // forward from the peak; the first anchor also seeds the backward walk:
      // exp(E(js-1) - E(js)) = exp(-delta^2) / g(js)
      double vb = 0.0, bb = 0.0;
      for (int j = js; j < nb; j += 32) {
        const double y = (__dadd_rn(lol, __dmul_rn(static_cast<double>(j) + 0.5, dxl)) + base) * lin;
        double v = w * exp(-0.5 * (c0 + y * y));
        if (!(v > 0.0)) break;
        double gg = exp(-(y * delta + half));
        if (j == js) {
          bb = hh / gg;
          vb = v * bb;
          bb *= hh;
        }
        const int e = min(nb, j + 32);
        for (int t = j; t < e; ++t) {
          sq += v;
          v *= gg;
          gg *= hh;
        }
      }
      for (int j = js - 1; j >= 0; j -= 32) {
        double v, b2;
        if (j == js - 1) {
          v = vb;
          b2 = bb;
        } else {
          const double y = (__dadd_rn(lol, __dmul_rn(static_cast<double>(j) + 0.5, dxl)) + base) * lin;
          v = w * exp(-0.5 * (c0 + y * y));
          b2 = exp(y * delta - half);
        }
        if (!(v > 0.0)) break;
        const int e = max(-1, j - 32);
        for (int t = j; t > e; --t) {
          sq += v;
          v *= b2;
          b2 *= hh;
        }
      }
      g[0] += sq;
    }
    // (b) #(q > 0): bin j of a row has q > 0 iff some component's log term
    // log w - (c0 + y_j^2)/2 is above the exp underflow limit — the union over the
    // components of one interval of j each.
    for (int64_t row = threadIdx.x; row < rows; row += kMB) {
      double x[3];
      lead_coords<D>(row, nb, lo, dx, x);
      int ia[kMaxK], ib[kMaxK];
      int ni = 0;
      for (int k = 0; k < M; ++k) {
        double base, lin, q0;
        row_terms<D>(comp[k], x, base, lin, q0);
        const double R = 2.0 * (comp[k].logw - kExpUnderflow) - comp[k].cst - q0;
        if (!(R > 0.0)) continue;
        const double rt = sqrt(R), rdelta = s_rdelta[k];
        const double yfirst = (__dadd_rn(lol, __dmul_rn(0.5, dxl)) + base) * lin;
        const double a = fmax(ceil((-rt - yfirst) * rdelta), 0.0);
        const double b2 = fmin(floor((rt - yfirst) * rdelta), double(nb - 1));
        if (!(a <= b2)) continue;
        int p = ni++;
        while (p > 0 && ia[p - 1] > static_cast<int>(a)) {  // insertion sort by start
          ia[p] = ia[p - 1];
          ib[p] = ib[p - 1];
          --p;
        }
        ia[p] = static_cast<int>(a);
        ib[p] = static_cast<int>(b2);
      }
      int cnt = 0, cur_a = -1, cur_b = -2;
      for (int t = 0; t < ni; ++t) {
        if (ia[t] > cur_b + 1) {
          cnt += cur_b - cur_a + 1;
          cur_a = ia[t];
          cur_b = ib[t];
        } else {
          cur_b = max(cur_b, ib[t]);
        }
      }
      cnt += cur_b - cur_a + 1;
      g[1] += static_cast<double>(cnt);
    }
    block_sum<2>(g, red);
    const double sum_q = g[0], n_qpos = g[1];
    const double zq = sum_q * area, zp = in_range * area;
    if (!(zq > 0.0) || !isfinite(zq)) {  // PdfGrid::normalized: degenerate model grid
      if (threadIdx.x < kMetricFields && o.f[threadIdx.x]) o.f[threadIdx.x][cell] = dnan();
      __syncthreads();
      continue;
    }
    // ---- non-empty bins
    // acc: 0 kl_pq, 1 kl_qp, 2 jsd, 3 sum q (p>0), 4 #(q>0, p>0), 5 #(q==0, p>0), 6 loglik,
    //      7 sum c, 8..10 sum c x, 11..16 sum c x x^T (upper, row-major)
    double acc[17];
#pragma unroll
    for (int i = 0; i < 17; ++i) acc[i] = 0.0;
    const int64_t off = c.offsets[cell];
    const int nnz = b.nnz[cell];
    for (int e = threadIdx.x; e < nnz; e += kMB) {
      uint32_t key = b.keys[off + e];
      const double cnt = b.counts[off + e];
      double x[3];
#pragma unroll
      for (int a = D - 1; a >= 0; --a) {
        const int i = static_cast<int>(key % static_cast<uint32_t>(nb));
        key /= static_cast<uint32_t>(nb);
        x[a] = __dadd_rn(lo[a], __dmul_rn(static_cast<double>(i) + 0.5, dx[a]));
      }
      double lg[kMaxK];
      double q = 0.0;
      for (int k = 0; k < M; ++k) {
        lg[k] = log_gauss<D>(comp[k], x);
        q += comp[k].w * exp(lg[k]);
      }
      // log sum_k w_k N_k = log q while q is a normal number (the reference's max-shifted
      // log-sum-exp, wgmm.cpp:262-264, equals it to rounding); the shifted form only
      // where q underflows
      double lse;
      if (q > 1e-290) {
        lse = log(q);
      } else {
        double mx = -dinf();
        for (int k = 0; k < M; ++k) mx = fmax(mx, lg[k] + comp[k].logw);
        double s = 0.0;
        for (int k = 0; k < M; ++k) s += exp(lg[k] + comp[k].logw - mx);
        lse = mx + log(s);
      }
      acc[6] += cnt * lse;
      const double pn = (cnt / zp) * area;
      const double qn = (q / zq) * area;
      if (qn > 0.0) {
        acc[0] += pn * log(pn / qn);
        acc[1] += qn * log(qn / pn);
        acc[4] += 1.0;
      } else {
        acc[5] += 1.0;
      }
      const double mn = 0.5 * (pn + qn);
      acc[2] += 0.5 * pn * log(pn / mn) + (qn > 0.0 ? 0.5 * qn * log(qn / mn) : 0.0);
      acc[3] += q;
      acc[7] += cnt;
      int u = 11;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        acc[8 + a] += x[a] * cnt;
#pragma unroll
        for (int e2 = a; e2 < D; ++e2) acc[u++] += (x[a] * cnt) * x[e2];
      }
    }
    block_sum<17>(acc, red);
    if (threadIdx.x == 0) {
      double v[kMetricFields];
      // jsd: + 0.5 qn ln 2 over the bins with p = 0
      double jsd = acc[2] + 0.5 * kLn2 * ((sum_q - acc[3]) / zq * area);
      v[0] = (jsd < -1e-9 || jsd > kLn2 + 1e-9) ? dnan() : fmin(fmax(jsd, 0.0), kLn2);
      v[1] = acc[5] > 0.0 ? dinf() : acc[0];
      v[2] = n_qpos > acc[4] ? dinf() : acc[1];
      const double ll = acc[6];
      const double kpar = static_cast<double>(M * (1 + D * (D + 3) / 2));
      v[3] = ll;
      v[4] = -2.0 * ll + kpar * log(in_range);
      v[5] = -2.0 * ll + kpar * log(static_cast<double>(total_bins));
      // moment errors (metrics.cpp:58-65): mixture vs weighted data moments
      double mm[3] = {0, 0, 0}, m2[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int k = 0; k < M; ++k) {
        const size_t ci = size_t(cell) * r.K + k;
        const double w = r.w[ci];
        const double* mu = r.mu + ci * D;
        const double* cv = r.cov + ci * D * D;
        for (int a = 0; a < D; ++a) mm[a] += w * mu[a];
        for (int a = 0; a < D; ++a)
          for (int e2 = 0; e2 < D; ++e2) m2[a * D + e2] += w * (cv[a * D + e2] + mu[a] * mu[e2]);
      }
      const double tw = acc[7];
      double tr = 0.0, num = 0.0, n2 = 0.0, dn = 0.0;
      int u = 11;
      double dm2[9];
      for (int a = 0; a < D; ++a)
        for (int e2 = a; e2 < D; ++e2) {
          dm2[a * D + e2] = acc[u] / tw;
          dm2[e2 * D + a] = acc[u] / tw;
          ++u;
        }
      for (int a = 0; a < D; ++a) {
        const double dmean = acc[8 + a] / tw;
        num += (mm[a] - dmean) * (mm[a] - dmean);
        tr += dm2[a * D + a];
      }
      for (int e2 = 0; e2 < D * D; ++e2) {
        n2 += (m2[e2] - dm2[e2]) * (m2[e2] - dm2[e2]);
        dn += dm2[e2] * dm2[e2];
      }
      v[6] = sqrt(num) / sqrt(tr);
      v[7] = sqrt(n2) / sqrt(dn);
      const double payload = static_cast<double>(M) * (1 + D + D * (D + 1) / 2) * 8.0;
      v[8] = static_cast<double>(total_bins) * 8.0 / payload;
      v[9] = static_cast<double>(c.offsets[cell + 1] - off) * D * 8.0 / payload;
      for (int f = 0; f < kMetricFields; ++f)
        if (o.f[f]) o.f[f][cell] = v[f];
    }
    __syncthreads();
  }
}

// ---- single-fit entry points -------------------------------------------------------
// Per-block model preparation; err (optional) is set when a covariance is not SPD.
template <int D>
VDFCG_DEV bool load_model_block(const ModelDev& m, PrepComp* comp, bool repair, int* err) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  if (threadIdx.x < m.m) {
    const int i = threadIdx.x;
    double mu[3], cov[9];
    const bool map = repair && m.scale && m.offset;
    for (int a = 0; a < D; ++a)
      mu[a] = map ? __dadd_rn(__dmul_rn(m.mu[i * D + a], m.scale[a]), m.offset[a]) : m.mu[i * D + a];
    for (int a = 0; a < D; ++a)
      for (int e = 0; e < D; ++e) {
        const double v = m.cov[(i * D + a) * D + e];
        cov[a * D + e] = map ? __dmul_rn(__dmul_rn(m.scale[a], v), m.scale[e]) : v;
      }
    if (map)
      for (int a = 1; a < D; ++a)
        for (int e = 0; e < a; ++e) cov[a * D + e] = cov[e * D + a];
    PrepComp p;
    bool good = prep_comp<D>(m.w[i], mu, cov, p);
    if (!good && repair) {  // log_component_densities repair-on-copy (wgmm.cpp:204-215)
      Sym3 s, fixed;
      for (int t = 0; t < 9; ++t) s.a[t] = 0.0;
      for (int a = 0; a < D; ++a)
        for (int e = 0; e < D; ++e) s(a, e) = cov[a * D + e];
      int dbl = 0;
      if (repair_covariance<D>(s, fixed, &dbl)) {
        symmetrize_from_upper<D>(fixed);
        double c2[9];
        for (int a = 0; a < D; ++a)
          for (int e = 0; e < D; ++e) c2[a * D + e] = fixed(a, e);
        good = prep_comp<D>(m.w[i], mu, c2, p);
      }
      if (!good) {  // unrepairable: its log-density row is -inf
        p.w = 0.0;
        p.logw = -dinf();
        p.cst = 0.0;
        for (int t = 0; t < 3; ++t) p.mu[t] = 0.0;
        for (int t = 0; t < 6; ++t) p.L[t] = t < 3 ? 0.0 : 1.0;
        good = true;
      }
    }
    if (!good) {
      bad = 1;
      if (err) atomicExch(err, 1);
    }
    comp[i] = p;
  }
  __syncthreads();
  return bad == 0;
}

__global__ void evaluate_pdf_kernel(ModelDev m, int nb, double xlo, double dxx, double ylo,
                                    double dyy, double* out, int* err) {
  __shared__ PrepComp comp[kMaxK];
  if (!load_model_block<2>(m, comp, false, err)) return;
  double vol = 1.0;
  if (m.scale && m.offset) vol = m.scale[0] * m.scale[1];
  const double inv_vol = 1.0 / vol;
  const int64_t n2 = int64_t(nb) * nb;
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < n2;
       o += int64_t(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(o % nb), j = static_cast<int>(o / nb);
    double x[2] = {__dadd_rn(xlo, __dmul_rn(static_cast<double>(i) + 0.5, dxx)),
                   __dadd_rn(ylo, __dmul_rn(static_cast<double>(j) + 0.5, dyy))};
    if (m.scale && m.offset)
      for (int a = 0; a < 2; ++a) x[a] = (x[a] - m.offset[a]) / m.scale[a];
    double p = 0.0;
    for (int k = 0; k < m.m; ++k) p += comp[k].w * exp(log_gauss<2>(comp[k], x));
    out[o] = p * inv_vol;
  }
}

template <int D>
__global__ void __launch_bounds__(256) loglik_kernel(ModelDev m, const double* pts,
                                                     const double* wts, int64_t n,
                                                     double* partial) {
  __shared__ PrepComp comp[kMaxK];
  __shared__ double red[33 * 2];
  load_model_block<D>(m, comp, true, nullptr);
  Kahan ll;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    double x[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = pts[a * n + r];
    double lg[kMaxK], mx = -dinf();
    for (int k = 0; k < m.m; ++k) {
      lg[k] = comp[k].logw == -dinf() ? -dinf() : log_gauss<D>(comp[k], x) + comp[k].logw;
      mx = fmax(mx, lg[k]);
    }
    double s = 0.0;
    for (int k = 0; k < m.m; ++k) s += exp(lg[k] - mx);
    ll.add(wts[r] * (mx + log(s)));
  }
  double v[2] = {ll.s, -ll.c};
  block_sum<2>(v, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = v[0] + v[1];
}

__global__ void sum_partials_kernel(const double* partial, int n, double* out, int stride, int nv) {
  if (threadIdx.x < nv) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += partial[i * stride + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

__global__ void __launch_bounds__(256) divergence_kernel(const double* p, const double* q, int64_t n,
                                                         double area, double* partial) {
  __shared__ double red[33 * 5];
  double acc[5] = {0, 0, 0, 0, 0};  // kl_pq, kl_qp, jsd, #inf pq, #inf qp
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double pn = p[i] * area, qn = q[i] * area;
    if (pn > 0.0) {
      if (qn > 0.0) acc[0] += pn * log(pn / qn);
      else acc[3] += 1.0;
    }
    if (qn > 0.0) {
      if (pn > 0.0) acc[1] += qn * log(qn / pn);
      else acc[4] += 1.0;
    }
    const double mn = 0.5 * (pn + qn);
    if (pn > 0.0) acc[2] += 0.5 * pn * log(pn / mn);
    if (qn > 0.0) acc[2] += 0.5 * qn * log(qn / mn);
  }
  block_sum<5>(acc, red);
  if (threadIdx.x < 5) partial[blockIdx.x * 5 + threadIdx.x] = acc[threadIdx.x];
}

__global__ void divergence_final_kernel(const double* sums, double* out) {
  out[0] = sums[2];
  out[1] = sums[3] > 0.0 ? dinf() : sums[0];
  out[2] = sums[4] > 0.0 ? dinf() : sums[1];
}

}  // namespace

void launch_cell_metrics(vdfcg_ctx* ctx, const CellsDev& c, const CellBinsDev& b,
                         const CellModels& r, const MetricsOut& o) {
  if (c.n_cells <= 0) return;
  const int grid = std::min(c.n_cells, ctx->sm_count * 8);
  if (c.d == 2)
    VDFCG_LAUNCH(ctx, "cell_metrics", cell_metrics_kernel<2><<<grid, kMB, 0, ctx->stream>>>(c, b, r, o));
  else
    VDFCG_LAUNCH(ctx, "cell_metrics", cell_metrics_kernel<3><<<grid, kMB, 0, ctx->stream>>>(c, b, r, o));
}

void launch_evaluate_pdf(vdfcg_ctx* ctx, const ModelDev& m, int nb, const double* lo,
                         const double* hi, double* out, int* err) {
  const int64_t n2 = int64_t(nb) * nb;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n2 + 255) / 256, ctx->sm_count * 8)));
  VDFCG_LAUNCH(ctx, "evaluate_pdf",
               evaluate_pdf_kernel<<<grid, 256, 0, ctx->stream>>>(m, nb, lo[0], (hi[0] - lo[0]) / nb, lo[1],
                                                                  (hi[1] - lo[1]) / nb, out, err));
}

void launch_weighted_loglik(vdfcg_ctx* ctx, const ModelDev& m, const double* pts,
                            const double* wts, int64_t n, double* out) {
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, ctx->sm_count * 4)));
  double* partial = arena<double>(ctx, grid);
  if (m.d == 2)
    VDFCG_LAUNCH(ctx, "weighted_loglik", loglik_kernel<2><<<grid, 256, 0, ctx->stream>>>(m, pts, wts, n, partial));
  else
    VDFCG_LAUNCH(ctx, "weighted_loglik", loglik_kernel<3><<<grid, 256, 0, ctx->stream>>>(m, pts, wts, n, partial));
  VDFCG_LAUNCH(ctx, "reduce", sum_partials_kernel<<<1, 32, 0, ctx->stream>>>(partial, grid, out, 1, 1));
}

void launch_pdf_divergences(vdfcg_ctx* ctx, const double* p, const double* q, int64_t n,
                            double area, double* out) {
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, ctx->sm_count * 4)));
  double* partial = arena<double>(ctx, size_t(grid) * 5);
  double* sums = arena<double>(ctx, 5);
  VDFCG_LAUNCH(ctx, "pdf_divergences",
               divergence_kernel<<<grid, 256, 0, ctx->stream>>>(p, q, n, area, partial));
  VDFCG_LAUNCH(ctx, "reduce", sum_partials_kernel<<<1, 32, 0, ctx->stream>>>(partial, grid, sums, 5, 5));
  VDFCG_LAUNCH(ctx, "reduce", divergence_final_kernel<<<1, 1, 0, ctx->stream>>>(sums, out));
}

}  // namespace vdfcg
