// vdfc_oracle.cpp — CPU restatement of the reference (proj/) hot path. TEST
// INFRASTRUCTURE: the checker for the CUDA product and the timed CPU baseline, never
// the product itself. Every function cites the reference file:line it restates.
// Eigen's LLT / triangular solve / SelfAdjointEigenSolver are replaced by explicit
// d <= 3 loops in the same operation order; build with -ffp-contract=off because the
// reference builds Release without -march (CMakeLists.txt:7-9), i.e. no FMA.
#include "vdfc_oracle.h"

#include <zlib.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

struct RepairError : std::runtime_error {  // types.hpp:99-101 CovarianceRepairError
  using std::runtime_error::runtime_error;
};
struct CodecErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return VDFCG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return VDFCG_INVALID_ARGUMENT;
  } catch (const RepairError& e) {
    g_err = e.what();
    return VDFCG_REPAIR_FAILED;
  } catch (const CodecErr& e) {
    g_err = e.what();
    return VDFCG_CODEC_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VDFCG_RUNTIME_ERROR;
  }
}

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();
constexpr double kMassFloorRel = 1e-250;  // wgmm.cpp:20

// ---------------------------------------------------------------------------
// rng.hpp:17-48
struct Rng {
  std::mt19937_64 eng;
  double spare = 0.0;
  bool has_spare = false;
  explicit Rng(std::uint64_t seed) : eng(seed) {}
  double uniform() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }  // rng.hpp:22
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }  // :25
  double normal() {                                                           // :28-40
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * M_PI * u2;
    spare = r * std::sin(a);
    has_spare = true;
    return r * std::cos(a);
  }
};

// ---------------------------------------------------------------------------
// Small dense linear algebra, d <= 3 (replaces Eigen).
using Mat3 = std::array<std::array<double, 3>, 3>;

// Eigen llt_inplace<Lower>::unblocked order; llt_ok (gaussian.hpp:15-19): every pivot
// strictly positive and finite.
bool cholesky(const Mat3& a, int d, Mat3& L) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) L[i][j] = 0.0;
  for (int k = 0; k < d; ++k) {
    double x = a[k][k];
    if (k > 0) {
      double sq = 0.0;
      for (int j = 0; j < k; ++j) sq += L[k][j] * L[k][j];
      x -= sq;
    }
    if (!(x > 0.0)) return false;  // Eigen: if (x <= 0) fail; NaN -> sqrt(NaN) -> not finite
    const double s = std::sqrt(x);
    if (!std::isfinite(s)) return false;
    L[k][k] = s;
    for (int i = k + 1; i < d; ++i) {
      double v = a[i][k];
      for (int j = 0; j < k; ++j) v -= L[i][j] * L[k][j];
      L[i][k] = v / s;
    }
  }
  for (int k = 0; k < d; ++k)
    if (!(L[k][k] > 0.0) || !std::isfinite(L[k][k])) return false;
  return true;
}

// gaussian.hpp:46-49
void symmetrize_from_upper(Mat3& m, int d) {
  for (int i = 1; i < d; ++i)
    for (int j = 0; j < i; ++j) m[i][j] = m[j][i];
}

// Symmetric eigenvalues by cyclic Jacobi (relative accuracy for the collapse test of
// wgmm.cpp:305-306; replaces Eigen::SelfAdjointEigenSolver).
void sym_eigenvalues(const Mat3& in, int d, double* ev) {
  double a[3][3];
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) a[i][j] = in[i][j];
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) off += std::fabs(a[p][q]);
    if (off == 0.0 || !std::isfinite(off)) break;
    for (int p = 0; p < d; ++p) {
      for (int q = p + 1; q < d; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0);
        const double s = t * c;
        a[p][p] -= t * apq;
        a[q][q] += t * apq;
        a[p][q] = a[q][p] = 0.0;
        for (int r = 0; r < d; ++r) {
          if (r == p || r == q) continue;
          const double arp = a[r][p], arq = a[r][q];
          a[r][p] = a[p][r] = c * arp - s * arq;
          a[r][q] = a[q][r] = s * arp + c * arq;
        }
      }
    }
  }
  for (int i = 0; i < d; ++i) ev[i] = a[i][i];
}

// ---------------------------------------------------------------------------
struct Comp {
  double w = 0.0;
  double mu[3] = {0, 0, 0};
  Mat3 cov{};
};
struct Model {
  int d = 0;
  std::vector<Comp> c;
  bool has_map = false;
  double scale[3] = {1, 1, 1};
  double offset[3] = {0, 0, 0};
  bool identity() const {  // types.hpp:71-73
    if (!has_map) return true;
    for (int a = 0; a < d; ++a)
      if (!(scale[a] == 1.0) || !(offset[a] == 0.0)) return false;
    return true;
  }
};

Model from_view(const vdfcg_model* v) {
  if (!v) throw std::invalid_argument("null model");
  Model m;
  m.d = v->dimension;
  if (m.d < 1 || m.d > 3) throw std::invalid_argument("model dimension must be 1..3");
  m.c.resize(v->components);
  for (int i = 0; i < v->components; ++i) {
    m.c[i].w = v->weights[i];
    for (int a = 0; a < m.d; ++a) m.c[i].mu[a] = v->means[i * m.d + a];
    for (int a = 0; a < m.d; ++a)
      for (int b = 0; b < m.d; ++b) m.c[i].cov[a][b] = v->covariances[(i * m.d + a) * m.d + b];
  }
  if (v->scale && v->offset) {
    m.has_map = true;
    for (int a = 0; a < m.d; ++a) {
      m.scale[a] = v->scale[a];
      m.offset[a] = v->offset[a];
    }
  }
  return m;
}

void to_view(const Model& m, vdfcg_model* v) {
  v->dimension = m.d;
  v->components = static_cast<int32_t>(m.c.size());
  for (size_t i = 0; i < m.c.size(); ++i) {
    v->weights[i] = m.c[i].w;
    for (int a = 0; a < m.d; ++a) v->means[i * m.d + a] = m.c[i].mu[a];
    for (int a = 0; a < m.d; ++a)
      for (int b = 0; b < m.d; ++b) v->covariances[(i * m.d + a) * m.d + b] = m.c[i].cov[a][b];
  }
  if (v->scale && v->offset) {
    for (int a = 0; a < m.d; ++a) {
      v->scale[a] = m.has_map ? m.scale[a] : 1.0;
      v->offset[a] = m.has_map ? m.offset[a] : 0.0;
    }
  }
}

// Points: N x d column-major + weights (histogram.hpp:33-43).
struct Points {
  int64_t n = 0;
  int d = 0;
  std::vector<double> x;  // column-major
  std::vector<double> w;
  double total = 0.0;
  double at(int64_t r, int a) const { return x[a * n + r]; }
};

// histogram.cpp:20-26 WeightedPoints::validate
void validate_points(const double* w, int64_t n) {
  if (n == 0) throw std::invalid_argument("weighted points: empty");
  bool any = false;
  for (int64_t i = 0; i < n; ++i) {
    if (!(w[i] >= 0.0)) throw std::invalid_argument("weighted points: weights must be >= 0");
    if (w[i] > 0.0) any = true;
  }
  if (!any) throw std::invalid_argument("weighted points: at least one weight must be > 0");
}

// wgmm.cpp:65-76 FitConfig::validate
void validate_config(const vdfcg_fit_config* cfg, int d) {
  if (!cfg) throw std::invalid_argument("null fit config");
  if (cfg->initial_components < 1) throw std::invalid_argument("initial_components must be >= 1");
  if (cfg->max_em_iterations < 1) throw std::invalid_argument("max_em_iterations must be >= 1");
  if (!(cfg->prune_threshold > 0.0)) throw std::invalid_argument("prune_threshold must be > 0");
  if (cfg->prune_threshold >= 1.0 / cfg->initial_components)
    throw std::invalid_argument("prune_threshold must be < 1/initial_components");
  if (cfg->prune_check_interval < 1)
    throw std::invalid_argument("prune_check_interval must be >= 1");
  if (!(cfg->loglik_rel_tolerance > 0.0))
    throw std::invalid_argument("loglik_rel_tolerance must be > 0");
  if (cfg->has_temperature) {
    for (int a = 0; a < d; ++a)
      if (!(cfg->temperature[a] > 0.0))
        throw std::invalid_argument("temperature must be > 0 on every axis");
  }
}

// wgmm.cpp:78-100
void normalize_impl(const Points& p, Points& out, double* scale, double* offset) {
  validate_points(p.w.data(), p.n);
  const int d = p.d;
  double lo[3], hi[3];
  for (int a = 0; a < d; ++a) {
    lo[a] = p.at(0, a);
    hi[a] = p.at(0, a);
    for (int64_t r = 1; r < p.n; ++r) {  // Eigen colwise().minCoeff(): comparisons only
      const double v = p.at(r, a);
      if (v < lo[a]) lo[a] = v;
      if (v > hi[a]) hi[a] = v;
    }
  }
  for (int a = 0; a < d; ++a) {
    offset[a] = 0.5 * (lo[a] + hi[a]);
    scale[a] = 0.5 * (hi[a] - lo[a]);
  }
  for (int a = 0; a < d; ++a) {
    if (!(scale[a] > 0.0)) {
      // std::ostream default formatting of a double == %g (6 significant digits)
      char msg[160];
      std::snprintf(msg, sizeof(msg), "degenerate data: axis %d has zero spread (all values %g)", a,
                    lo[a]);
      throw std::invalid_argument(msg);
    }
  }
  out = p;
  for (int a = 0; a < d; ++a)
    for (int64_t r = 0; r < p.n; ++r) out.x[a * p.n + r] = (p.at(r, a) - offset[a]) / scale[a];
}

// wgmm.cpp:102-120
Model denormalize_impl(const Model& m) {
  Model out;
  out.d = m.d;
  out.has_map = false;
  if (m.identity()) {
    out.c = m.c;
    return out;
  }
  for (const Comp& c : m.c) {
    Comp t;
    t.w = c.w;
    for (int a = 0; a < m.d; ++a) t.mu[a] = c.mu[a] * m.scale[a] + m.offset[a];  // types.hpp:76
    for (int a = 0; a < m.d; ++a)
      for (int b = 0; b < m.d; ++b) t.cov[a][b] = (m.scale[a] * c.cov[a][b]) * m.scale[b];
    symmetrize_from_upper(t.cov, m.d);
    out.c.push_back(t);
  }
  return out;
}

// wgmm.cpp:124-132 (std::set of rows)
int64_t count_distinct(const Points& p, int64_t stop_at) {
  std::set<std::vector<double>> seen;
  std::vector<double> row(p.d);
  for (int64_t r = 0; r < p.n; ++r) {
    for (int a = 0; a < p.d; ++a) row[a] = p.at(r, a);
    seen.insert(row);
    if (static_cast<int64_t>(seen.size()) >= stop_at) break;
  }
  return static_cast<int64_t>(seen.size());
}

// wgmm.cpp:136-191
Model init_impl(const Points& np, const vdfcg_fit_config* cfg, const double* temperature,
                const double* scale, const double* offset) {
  validate_config(cfg, np.d);
  const int d = np.d;
  Model out;
  out.d = d;
  out.has_map = true;
  for (int a = 0; a < d; ++a) {
    out.scale[a] = scale[a];
    out.offset[a] = offset[a];
  }
  if (cfg->warm_start) {  // :142-161
    Model warm = from_view(cfg->warm_start);
    if (warm.d != d)
      throw std::invalid_argument("warm-start model dimension does not match the data");
    const Model canonical = warm.identity() ? warm : denormalize_impl(warm);
    double D[3];
    for (int a = 0; a < d; ++a) D[a] = 1.0 / scale[a];  // cwiseInverse
    for (const Comp& c : canonical.c) {
      Comp t;
      t.w = c.w;
      for (int a = 0; a < d; ++a) t.mu[a] = (c.mu[a] - offset[a]) / scale[a];  // forward
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) t.cov[a][b] = (D[a] * c.cov[a][b]) * D[b];
      symmetrize_from_upper(t.cov, d);
      out.c.push_back(t);
    }
    return out;
  }
  for (int a = 0; a < d; ++a)
    if (!(temperature[a] > 0.0))
      throw std::invalid_argument("temperature must be a positive per-axis variance");

  int m = cfg->initial_components;
  const int64_t distinct = count_distinct(np, m);  // only "distinct < m" matters
  if (distinct < m) m = static_cast<int>(distinct);

  double lo[3], hi[3];
  for (int a = 0; a < d; ++a) {
    lo[a] = np.at(0, a);
    hi[a] = np.at(0, a);
    for (int64_t r = 1; r < np.n; ++r) {
      const double v = np.at(r, a);
      if (v < lo[a]) lo[a] = v;
      if (v > hi[a]) hi[a] = v;
    }
  }
  Mat3 base{};
  for (int a = 0; a < d; ++a) base[a][a] = temperature[a] / (scale[a] * scale[a]);

  Rng rng(cfg->seed);
  out.c.resize(m);
  for (int i = 0; i < m; ++i) {
    out.c[i].w = 1.0 / m;
    for (int a = 0; a < d; ++a) out.c[i].mu[a] = rng.uniform(lo[a], hi[a]);
    out.c[i].cov = base;
  }
  return out;
}

// wgmm.cpp:340-362
Mat3 repair_impl(const Mat3& sigma, int d, int* doublings) {
  Mat3 sym{};
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) sym[a][b] = 0.5 * (sigma[a][b] + sigma[b][a]);
  symmetrize_from_upper(sym, d);
  if (doublings) *doublings = -1;
  Mat3 L;
  if (cholesky(sym, d, L)) return sym;
  double tr = 0.0;
  for (int a = 0; a < d; ++a) tr += sym[a][a];
  const double lambda0 = 1e-8 * tr / static_cast<double>(d);
  double lambda = lambda0;
  for (int k = 0; k <= 60; ++k, lambda *= 2.0) {
    Mat3 loaded = sym;
    for (int a = 0; a < d; ++a) loaded[a][a] += lambda;
    if (cholesky(loaded, d, L)) {
      if (doublings) *doublings = k;
      return loaded;
    }
  }
  throw RepairError("covariance repair failed after 60 doublings");
}

// wgmm.cpp:197-229 log_component_densities + gaussian.hpp:33-42.
// logp is M x N column-major.
void log_component_densities(Model& m, const Points& p, std::vector<double>& logp,
                             std::vector<int>* unrepairable) {
  const int M = static_cast<int>(m.c.size());
  const int d = m.d;
  logp.resize(static_cast<size_t>(M) * p.n);  // every entry is written below
  const double log2pi = std::log(2.0 * M_PI);
  for (int i = 0; i < M; ++i) {
    Comp& c = m.c[i];
    Mat3 L;
    bool ok = cholesky(c.cov, d, L);
    if (!ok) {
      bool dead = false;
      try {
        c.cov = repair_impl(c.cov, d, nullptr);
        symmetrize_from_upper(c.cov, d);
        dead = !cholesky(c.cov, d, L);
      } catch (const RepairError&) {
        dead = true;
      }
      if (dead) {
        if (unrepairable) unrepairable->push_back(i);
        for (int64_t n = 0; n < p.n; ++n) logp[i + n * M] = -kInf;
        continue;
      }
    }
    const double log_alpha = c.w > 0.0 ? std::log(c.w) : -kInf;
    double logdet_half = 0.0;
    for (int k = 0; k < d; ++k) logdet_half += std::log(L[k][k]);
    const double cst = d * log2pi + 2.0 * logdet_half;
    // forward substitution L y = (x - mu), per axis in Eigen's order; d is unrolled
    // (same operations, same order) so the port is a fair CPU baseline
    const double* x0 = p.x.data();
    const double* x1 = x0 + p.n;
    const double* x2 = x1 + p.n;
    double* out = logp.data() + i;
    if (d == 2) {
      for (int64_t n = 0; n < p.n; ++n) {
        const double y0 = (x0[n] - c.mu[0]) / L[0][0];
        const double y1 = ((x1[n] - c.mu[1]) - L[1][0] * y0) / L[1][1];
        const double q = y0 * y0 + y1 * y1;
        out[n * M] = -0.5 * (q + cst) + log_alpha;
      }
    } else if (d == 3) {
      for (int64_t n = 0; n < p.n; ++n) {
        const double y0 = (x0[n] - c.mu[0]) / L[0][0];
        const double y1 = ((x1[n] - c.mu[1]) - L[1][0] * y0) / L[1][1];
        const double y2 = (((x2[n] - c.mu[2]) - L[2][0] * y0) - L[2][1] * y1) / L[2][2];
        const double q = (y0 * y0 + y1 * y1) + y2 * y2;
        out[n * M] = -0.5 * (q + cst) + log_alpha;
      }
    } else {
      for (int64_t n = 0; n < p.n; ++n) {
        double y[3];
        for (int a = 0; a < d; ++a) {
          double v = p.at(n, a) - c.mu[a];
          for (int b = 0; b < a; ++b) v -= L[a][b] * y[b];
          y[a] = v / L[a][a];
        }
        double q = 0.0;
        for (int a = 0; a < d; ++a) q += y[a] * y[a];
        out[n * M] = -0.5 * (q + cst) + log_alpha;
      }
    }
  }
}

struct Kahan {  // gaussian.hpp:55-68
  double s = 0.0, c = 0.0;
  void add(double x) {
    const double y = x - c;
    const double t = s + y;
    c = (t - s) - y;
    s = t;
  }
};

// wgmm.cpp:233-255
double e_step_impl(Model& m, const Points& p, std::vector<double>& resp,
                   std::vector<int>& unrepairable) {
  const int M = static_cast<int>(m.c.size());
  thread_local std::vector<double> logp;  // reused across iterations (capacity kept)
  log_component_densities(m, p, logp, &unrepairable);
  if (static_cast<int>(unrepairable.size()) == M)
    throw std::runtime_error("all mixture components are degenerate");
  resp.resize(static_cast<size_t>(M) * p.n);  // every entry is written below
  Kahan ll;
  thread_local std::vector<double> u;
  u.resize(M);
  for (int64_t n = 0; n < p.n; ++n) {
    const double* col = &logp[n * M];
    double mx = col[0];
    for (int i = 1; i < M; ++i)
      if (col[i] > mx) mx = col[i];
    double s = 0.0;
    for (int i = 0; i < M; ++i) {
      u[i] = std::exp(col[i] - mx);
      s += u[i];
    }
    for (int i = 0; i < M; ++i) resp[i + n * M] = u[i] / s;
    ll.add(p.w[n] * (mx + std::log(s)));
  }
  return ll.s;
}

// wgmm.cpp:269-318
Model m_step_impl(const Points& p, double total, const std::vector<double>& resp,
                  const Model& prev, std::vector<int>* degenerate) {
  const int M = static_cast<int>(prev.c.size());
  const int d = p.d;
  if (!(total > 0.0)) throw std::runtime_error("m_step: zero total weight");
  // one pass per component for the mass and the first moments (each sum keeps the
  // sequential order over n; the mass check below still precedes any use)
  std::vector<double> mass(M, 0.0);
  thread_local std::vector<double> wi, sms;
  wi.resize(static_cast<size_t>(M) * p.n);
  sms.assign(static_cast<size_t>(M) * 3, 0.0);
  for (int i = 0; i < M; ++i) {
    double* wr = &wi[static_cast<size_t>(i) * p.n];
    double s = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0;
    const double* x0 = p.x.data();
    const double* x1 = x0 + p.n;
    const double* x2 = x1 + p.n;
    const double* r = resp.data() + i;
    if (d == 3) {
      for (int64_t n = 0; n < p.n; ++n) {
        const double v = r[n * M] * p.w[n];
        wr[n] = v;
        s += v;
        s0 += x0[n] * v;
        s1 += x1[n] * v;
        s2 += x2[n] * v;
      }
    } else {
      for (int64_t n = 0; n < p.n; ++n) {
        const double v = r[n * M] * p.w[n];
        wr[n] = v;
        s += v;
        s0 += x0[n] * v;
        if (d > 1) s1 += x1[n] * v;
      }
    }
    mass[i] = s;
    sms[i * 3 + 0] = s0;
    sms[i * 3 + 1] = s1;
    sms[i * 3 + 2] = s2;
  }
  for (int i = 0; i < M; ++i)
    if (!std::isfinite(mass[i]) || mass[i] < 0.0)
      throw std::runtime_error("m_step: invalid responsibility mass");

  Model out;
  out.d = prev.d;
  out.has_map = prev.has_map;
  std::memcpy(out.scale, prev.scale, sizeof(out.scale));
  std::memcpy(out.offset, prev.offset, sizeof(out.offset));
  out.c.resize(M);
  for (int i = 0; i < M; ++i) {
    Comp& c = out.c[i];
    c.w = mass[i] / total;
    if (!(mass[i] > total * kMassFloorRel)) {  // starved: freeze
      std::memcpy(c.mu, prev.c[i].mu, sizeof(c.mu));
      c.cov = prev.c[i].cov;
      continue;
    }
    const double* wr = &wi[static_cast<size_t>(i) * p.n];
    const double* sm = &sms[i * 3];
    for (int a = 0; a < d; ++a) c.mu[a] = sm[a] / mass[i];
    Mat3 sigma{};
    double ss[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    if (d == 3) {
      const double* x0 = p.x.data();
      const double* x1 = x0 + p.n;
      const double* x2 = x1 + p.n;
      const double m0 = c.mu[0], m1 = c.mu[1], m2 = c.mu[2];
      double s00 = 0.0, s01 = 0.0, s02 = 0.0, s11 = 0.0, s12 = 0.0, s22 = 0.0;
      for (int64_t n = 0; n < p.n; ++n) {
        const double c0 = x0[n] - m0, c1 = x1[n] - m1, c2 = x2[n] - m2;
        const double a0 = c0 * wr[n], a1 = c1 * wr[n], a2 = c2 * wr[n];
        s00 += a0 * c0;
        s01 += a0 * c1;
        s02 += a0 * c2;
        s11 += a1 * c1;
        s12 += a1 * c2;
        s22 += a2 * c2;
      }
      ss[0][0] = s00; ss[0][1] = s01; ss[0][2] = s02;
      ss[1][1] = s11; ss[1][2] = s12; ss[2][2] = s22;
    } else {
      for (int64_t n = 0; n < p.n; ++n) {
        double cen[3] = {0.0, 0.0, 0.0};
        for (int a = 0; a < d; ++a) cen[a] = p.at(n, a) - c.mu[a];
        for (int a = 0; a < d; ++a)
          for (int b = a; b < d; ++b) ss[a][b] += (cen[a] * wr[n]) * cen[b];
      }
    }
    for (int a = 0; a < d; ++a)
      for (int b = a; b < d; ++b) sigma[a][b] = ss[a][b] / mass[i];
    symmetrize_from_upper(sigma, d);
    bool collapsed = false;
    bool finite = true;
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) finite = finite && std::isfinite(sigma[a][b]);
    if (finite) {
      double ev[3] = {0.0, 0.0, 0.0};
      sym_eigenvalues(sigma, d, ev);
      double mn = ev[0], mx = ev[0];
      for (int a = 1; a < d; ++a) {
        mn = std::min(mn, ev[a]);
        mx = std::max(mx, ev[a]);
      }
      if (mn <= 1e-14 * mx) collapsed = true;
    }
    if (!collapsed) {
      try {
        int doublings = -1;
        Mat3 rep = repair_impl(sigma, d, &doublings);
        if (doublings > 2) {
          collapsed = true;
        } else {
          symmetrize_from_upper(rep, d);
          c.cov = rep;
        }
      } catch (const RepairError&) {
        collapsed = true;
      }
    }
    if (collapsed) {
      c.cov = prev.c[i].cov;
      if (degenerate) degenerate->push_back(i);
    }
  }
  return out;
}

// wgmm.cpp:320-333
bool prune_one_impl(Model& m, double threshold, int* idx, double* weight) {
  if (m.c.size() <= 1) return false;
  int smallest = 0;
  for (int i = 1; i < static_cast<int>(m.c.size()); ++i)
    if (m.c[i].w < m.c[smallest].w) smallest = i;
  if (!(m.c[smallest].w < threshold)) return false;
  *idx = smallest;
  *weight = m.c[smallest].w;
  m.c.erase(m.c.begin() + smallest);
  double total = 0.0;
  for (const Comp& c : m.c) total += c.w;
  for (Comp& c : m.c) c.w /= total;
  return true;
}

// wgmm.cpp:473-480 weighted_data_moments
void data_moments(const Points& p, double* mean, double* m2) {
  double total = 0.0;
  for (int64_t n = 0; n < p.n; ++n) total += p.w[n];
  if (!(total > 0.0)) throw std::invalid_argument("weighted moments: zero total weight");
  const int d = p.d;
  for (int a = 0; a < d; ++a) {
    double s = 0.0;
    for (int64_t n = 0; n < p.n; ++n) s += p.at(n, a) * p.w[n];
    mean[a] = s / total;
  }
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double s = 0.0;
      for (int64_t n = 0; n < p.n; ++n) s += (p.at(n, a) * p.w[n]) * p.at(n, b);
      m2[a * d + b] = s / total;
    }
}

struct FitOut {
  Model model;
  std::vector<double> trace;
  int iterations = 0;
  bool converged = false;
  std::vector<std::array<double, 3>> events;  // it, idx, weight
};

// wgmm.cpp:364-423
FitOut fit_impl(const Points& pts, const vdfcg_fit_config* cfg) {
  validate_config(cfg, pts.d);
  Points np;
  double scale[3], offset[3];
  try {
    normalize_impl(pts, np, scale, offset);
  } catch (const std::invalid_argument& e) {
    throw std::invalid_argument(std::string("fit: ") + e.what());
  }
  double temperature[3];
  if (cfg->has_temperature) {
    for (int a = 0; a < pts.d; ++a) temperature[a] = cfg->temperature[a];
  } else {  // wgmm.cpp:22-25 weighted_axis_variance
    double mean[3], m2[9];
    data_moments(pts, mean, m2);
    for (int a = 0; a < pts.d; ++a)
      temperature[a] = std::max(m2[a * pts.d + a] - mean[a] * mean[a], 0.0);
  }
  Model model = init_impl(np, cfg, temperature, scale, offset);

  FitOut r;
  double prev_ll = kNaN;
  int it = 0;
  std::vector<double> resp;
  std::vector<int> unrep;
  for (it = 1; it <= cfg->max_em_iterations; ++it) {
    unrep.clear();
    const double ll = e_step_impl(model, np, resp, unrep);
    std::vector<int> degenerate = unrep;
    model = m_step_impl(np, np.total, resp, model, &degenerate);
    r.trace.push_back(ll);

    bool pruned = false;
    std::sort(degenerate.begin(), degenerate.end(), std::greater<int>());
    degenerate.erase(std::unique(degenerate.begin(), degenerate.end()), degenerate.end());
    for (int idx : degenerate) {
      if (model.c.size() <= 1) break;
      r.events.push_back({static_cast<double>(it), static_cast<double>(idx), model.c[idx].w});
      model.c.erase(model.c.begin() + idx);
      pruned = true;
    }
    if (pruned) {
      double total = 0.0;
      for (const Comp& c : model.c) total += c.w;
      for (Comp& c : model.c) c.w /= total;
    }
    if (it % cfg->prune_check_interval == 0) {
      int idx = 0;
      double w = 0.0;
      if (prune_one_impl(model, cfg->prune_threshold, &idx, &w)) {
        r.events.push_back({static_cast<double>(it), static_cast<double>(idx), w});
        pruned = true;
      }
    }
    if (!pruned && std::isfinite(prev_ll) &&
        std::fabs(ll - prev_ll) < cfg->loglik_rel_tolerance * std::fabs(prev_ll)) {
      r.converged = true;
      break;
    }
    prev_ll = pruned ? kNaN : ll;
  }
  r.iterations = std::min(it, cfg->max_em_iterations);
  r.model = denormalize_impl(model);
  return r;
}

Points make_points(const double* points, const double* weights, int64_t n, int d,
                   double total_weight) {
  Points p;
  p.n = n;
  p.d = d;
  p.x.assign(points, points + n * d);
  p.w.assign(weights, weights + n);
  p.total = total_weight;
  return p;
}

void write_fit_result(const FitOut& f, vdfcg_fit_result* res) {
  const int M = static_cast<int>(f.model.c.size());
  if (M > res->capacity_components) throw std::invalid_argument("result capacity too small");
  if (static_cast<int>(f.trace.size()) > res->capacity_trace)
    throw std::invalid_argument("trace capacity too small");
  to_view(f.model, &res->model);
  for (size_t t = 0; t < f.trace.size(); ++t) res->loglik_trace[t] = f.trace[t];
  res->trace_len = static_cast<int32_t>(f.trace.size());
  res->iterations_used = f.iterations;
  res->converged = f.converged ? 1 : 0;
  res->n_events = static_cast<int32_t>(f.events.size());
  for (size_t e = 0; e < f.events.size() && static_cast<int>(e) < res->capacity_components; ++e) {
    if (res->event_iteration) res->event_iteration[e] = static_cast<int32_t>(f.events[e][0]);
    if (res->event_component) res->event_component[e] = static_cast<int32_t>(f.events[e][1]);
    if (res->event_weight) res->event_weight[e] = f.events[e][2];
  }
}

// ---------------------------------------------------------------------------
// Histogram, histogram.cpp:36-41: NaN goes out of range (x86: floor(NaN) cast is
// INT_MIN, which fails the in-range test at :70).
inline int bin_index(double v, double lo, double hi, int n, double inv) {
  if (v < lo || v > hi) return -1;
  if (!(v == v)) return -1;
  int i = static_cast<int>(std::floor((v - lo) * inv));
  if (i >= n) i = n - 1;
  return i;
}

inline double center(double lo, double hi, int n, int i) {  // types.hpp:48,51
  const double dx = (hi - lo) / n;
  return lo + (i + 0.5) * dx;
}

void plane_axes(int plane, int* ax, int* ay) {  // types.hpp:20-27
  switch (plane) {
    case 0: *ax = 0; *ay = 1; return;
    case 1: *ax = 1; *ay = 2; return;
    case 2: *ax = 0; *ay = 2; return;
    default: throw std::invalid_argument("unknown plane");
  }
}

const char* plane_name(int p) { return p == 0 ? "uv" : p == 1 ? "vw" : "uw"; }

void validate_particles(int d, const double* w, int64_t n) {  // synthdata.cpp:18-31
  if (d != 2 && d != 3) throw std::invalid_argument("particle dimension must be 2 or 3");
  if (w)
    for (int64_t i = 0; i < n; ++i)
      if (!(w[i] > 0.0)) throw std::invalid_argument("particle weights must all be > 0");
}

void bin2d(const double* vel, int64_t n, int d, const double* w, int plane, int nb, double xlo,
           double xhi, double ylo, double yhi, double* counts, double* oor) {
  validate_particles(d, w, n);
  if (nb < 2) throw std::invalid_argument("n_bins must be >= 2");
  if (!(std::isfinite(xlo) && std::isfinite(xhi) && xlo < xhi && std::isfinite(ylo) &&
        std::isfinite(yhi) && ylo < yhi))
    throw std::invalid_argument("axis range must satisfy min < max");
  int ax, ay;
  plane_axes(plane, &ax, &ay);
  if (ay >= d)
    throw std::invalid_argument(std::string("plane ") + plane_name(plane) +
                                " requires the w axis, but particles are " + std::to_string(d) +
                                "-dimensional");
  std::fill(counts, counts + static_cast<int64_t>(nb) * nb, 0.0);
  double o = 0.0;
  const double inv_dx = nb / (xhi - xlo);
  const double inv_dy = nb / (yhi - ylo);
  for (int64_t r = 0; r < n; ++r) {
    const double wt = w ? w[r] : 1.0;
    const int i = bin_index(vel[ax * n + r], xlo, xhi, nb, inv_dx);
    const int j = bin_index(vel[ay * n + r], ylo, yhi, nb, inv_dy);
    if (i < 0 || j < 0)
      o += wt;
    else
      counts[i + static_cast<int64_t>(j) * nb] += wt;
  }
  *oor = o;
}

// Per-cell bin + compaction (Appendix A generalisation). Writes compacted keys/counts.
void bin_one_cell(const vdfcg_cells* cells, int c, std::vector<double>& dense, uint32_t* keys,
                  double* counts, int32_t* nnz, double* oor, double* in_range) {
  const int d = cells->dimension;
  const int nb = cells->n_bins;
  int64_t nbins_total = 1;
  for (int a = 0; a < d; ++a) nbins_total *= nb;
  dense.assign(nbins_total, 0.0);
  const int64_t b = cells->cell_offsets[c], e = cells->cell_offsets[c + 1];
  double inv[3];
  for (int a = 0; a < d; ++a) inv[a] = nb / (cells->hi[a] - cells->lo[a]);
  double o = 0.0;
  for (int64_t r = b; r < e; ++r) {
    const double wt = cells->weights ? cells->weights[r] : 1.0;
    int64_t key = 0;
    bool out = false;
    for (int a = 0; a < d; ++a) {
      const int i = bin_index(cells->velocity[a][r], cells->lo[a], cells->hi[a], nb, inv[a]);
      if (i < 0) out = true;
      key = key * nb + i;
    }
    if (out)
      o += wt;
    else
      dense[key] += wt;
  }
  int64_t k = 0;
  double tot = 0.0;
  for (int64_t f = 0; f < nbins_total; ++f) {
    tot += dense[f];
    if (dense[f] > 0.0) {
      keys[b + k] = static_cast<uint32_t>(f);
      counts[b + k] = dense[f];
      ++k;
    }
  }
  *nnz = static_cast<int32_t>(k);
  *oor = o;
  *in_range = tot;
}

// Points of one cell in data space (bin centres), N x d column-major.
Points cell_points(const vdfcg_cells* cells, int c, const uint32_t* keys, const double* counts,
                   int32_t nnz, double in_range) {
  const int d = cells->dimension;
  const int nb = cells->n_bins;
  const int64_t b = cells->cell_offsets[c];
  Points p;
  p.n = nnz;
  p.d = d;
  p.x.resize(static_cast<size_t>(nnz) * d);
  p.w.resize(nnz);
  for (int64_t r = 0; r < nnz; ++r) {
    uint32_t key = keys[b + r];
    int idx[3];
    for (int a = d - 1; a >= 0; --a) {
      idx[a] = static_cast<int>(key % nb);
      key /= nb;
    }
    for (int a = 0; a < d; ++a) p.x[a * nnz + r] = center(cells->lo[a], cells->hi[a], nb, idx[a]);
    p.w[r] = counts[b + r];
  }
  p.total = in_range;
  return p;
}

uint32_t crc32_bytes(const uint8_t* p, size_t n) {
  return static_cast<uint32_t>(::crc32(0L, reinterpret_cast<const Bytef*>(p), static_cast<uInt>(n)));
}

void put_u8(std::vector<uint8_t>& b, uint8_t v) { b.push_back(v); }
void put_u16(std::vector<uint8_t>& b, uint16_t v) {
  b.push_back(static_cast<uint8_t>(v & 0xff));
  b.push_back(static_cast<uint8_t>(v >> 8));
}
void put_u32(std::vector<uint8_t>& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put_u64(std::vector<uint8_t>& b, uint64_t v) {
  for (int i = 0; i < 8; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put_f64(std::vector<uint8_t>& b, double v) {
  uint64_t u;
  std::memcpy(&u, &v, 8);
  put_u64(b, u);
}

// wgmm.cpp:46-63 GmmModel::validate (canonical models only)
void validate_model(const Model& m) {
  if (m.d < 1) throw std::invalid_argument("model dimension must be positive");
  if (m.c.empty()) throw std::invalid_argument("model has no components");
  double total = 0.0;
  for (const Comp& c : m.c) {
    if (!(c.w > 0.0)) throw std::invalid_argument("component weight must be > 0");
    for (int a = 0; a < m.d; ++a)
      for (int b = 0; b < m.d; ++b)
        if (!(c.cov[a][b] == c.cov[b][a]))
          throw std::invalid_argument("component covariance is not symmetric");
    total += c.w;
  }
  if (std::fabs(total - 1.0) > 1e-12) throw std::invalid_argument("component weights must sum to 1");
}

// codec.cpp:103-136
std::vector<uint8_t> encode_impl(const Model& model, const vdfcg_model_meta* meta,
                                 bool validate = true) {
  if (validate) validate_model(model);
  const Model canonical = model.identity() ? model : denormalize_impl(model);
  const int d = canonical.d;
  if (meta->label_len > 0xffff) throw std::invalid_argument("species label too long");
  std::vector<uint8_t> out = {'G', 'M', 'M', 'C'};
  put_u8(out, 1);
  put_u8(out, static_cast<uint8_t>(d));
  put_u8(out, meta->plane >= 0 && meta->plane <= 2 ? static_cast<uint8_t>(meta->plane) : 255);
  put_u8(out, 0);
  put_u32(out, static_cast<uint32_t>(canonical.c.size()));
  put_u64(out, static_cast<uint64_t>(meta->cycle));
  for (int a = 0; a < d; ++a) {
    put_f64(out, meta->range_lo[a]);
    put_f64(out, meta->range_hi[a]);
  }
  put_u16(out, static_cast<uint16_t>(meta->label_len));
  for (int i = 0; i < meta->label_len; ++i) out.push_back(static_cast<uint8_t>(meta->species_label[i]));
  put_u32(out, crc32_bytes(out.data(), out.size()));
  for (const Comp& c : canonical.c) {
    put_f64(out, c.w);
    for (int a = 0; a < d; ++a) put_f64(out, c.mu[a]);
    for (int i = 0; i < d; ++i)
      for (int j = i; j < d; ++j) put_f64(out, c.cov[i][j]);
  }
  return out;
}

// ---- fit quality ----------------------------------------------------------
// gaussian.hpp:22-28 log_gaussian through the Eigen-order Cholesky factor.
double log_gaussian(const double* z, const double* mu, const Mat3& L, int d) {
  double y[3];
  for (int a = 0; a < d; ++a) {
    double v = z[a] - mu[a];
    for (int b = 0; b < a; ++b) v -= L[a][b] * y[b];
    y[a] = v / L[a][a];
  }
  double ld = 0.0;
  for (int k = 0; k < d; ++k) ld += std::log(L[k][k]);
  double sq = 0.0;
  for (int a = 0; a < d; ++a) sq += y[a] * y[a];
  return -0.5 * (d * std::log(2.0 * M_PI) + 2.0 * ld + sq);
}

// wgmm.cpp:425-453 evaluate_pdf over the bins^d grid in flat key order (i*n+j)*n+k.
void evaluate_grid(const Model& m, int nb, const double* lo, const double* hi,
                   std::vector<double>& out) {
  validate_model(m);
  const int d = m.d;
  std::vector<Mat3> L(m.c.size());
  for (size_t k = 0; k < m.c.size(); ++k)
    if (!cholesky(m.c[k].cov, d, L[k])) throw std::runtime_error("model component covariance is not SPD");
  double vol = 1.0;
  if (m.has_map)
    for (int a = 0; a < d; ++a) vol *= m.scale[a];
  const double inv_vol = 1.0 / vol;
  int64_t total = 1;
  for (int a = 0; a < d; ++a) total *= nb;
  out.assign(total, 0.0);
  for (int64_t key = 0; key < total; ++key) {
    int64_t r = key;
    double z[3];
    for (int a = d - 1; a >= 0; --a) {
      const int i = static_cast<int>(r % nb);
      r /= nb;
      const double x = center(lo[a], hi[a], nb, i);
      z[a] = m.has_map ? (x - m.offset[a]) / m.scale[a] : x;
    }
    double p = 0.0;
    for (size_t k = 0; k < m.c.size(); ++k) p += m.c[k].w * std::exp(log_gaussian(z, m.c[k].mu, L[k], d));
    out[key] = p * inv_vol;
  }
}

// pdf_grid.cpp:5-19 PdfGrid::normalized
void normalize_grid(std::vector<double>& v, double area) {
  double s = 0.0;
  for (double x : v) {
    if (x < 0.0) throw std::invalid_argument("pdf grid values must be non-negative");
    s += x;
  }
  const double total = s * area;
  if (!(total > 0.0) || !std::isfinite(total))
    throw std::invalid_argument("degenerate pdf grid: total mass is zero or non-finite");
  for (double& x : v) x /= total;
}

// metrics.cpp:12-26 kl_divergence
double kl_impl(const double* p, const double* q, int64_t n, double area) {
  double sum = 0.0;
  for (int64_t b = 0; b < n; ++b) {
    const double pn = p[b] * area;
    if (!(pn > 0.0)) continue;
    const double qn = q[b] * area;
    if (!(qn > 0.0)) return kInf;
    sum += pn * std::log(pn / qn);
  }
  return sum;
}

// metrics.cpp:28-46 jsd (out of [0, ln 2] beyond 1e-9 -> the reference throws logic_error)
double jsd_impl(const double* p, const double* q, int64_t n, double area) {
  double sum = 0.0;
  for (int64_t b = 0; b < n; ++b) {
    const double pn = p[b] * area;
    const double qn = q[b] * area;
    const double mn = 0.5 * (pn + qn);
    if (pn > 0.0) sum += 0.5 * pn * std::log(pn / mn);
    if (qn > 0.0) sum += 0.5 * qn * std::log(qn / mn);
  }
  constexpr double ln2 = 0.6931471805599453;
  if (sum < -1e-9 || sum > ln2 + 1e-9)
    throw std::logic_error("jsd outside [0, ln 2] beyond numerical slack");
  return std::clamp(sum, 0.0, ln2);
}

// wgmm.cpp:257-267 weighted_loglik
double weighted_loglik_impl(const Model& model, const Points& p) {
  Model scratch = model.identity() ? model : denormalize_impl(model);
  std::vector<double> logp;
  log_component_densities(scratch, p, logp, nullptr);
  const int M = static_cast<int>(scratch.c.size());
  Kahan ll;
  for (int64_t n = 0; n < p.n; ++n) {
    double mx = -kInf;
    for (int i = 0; i < M; ++i) mx = std::max(mx, logp[i + n * M]);
    double s = 0.0;
    for (int i = 0; i < M; ++i) s += std::exp(logp[i + n * M] - mx);
    ll.add(p.w[n] * (mx + std::log(s)));
  }
  return ll.s;
}

// wgmm.cpp:455-471 mixture_moments (identity or mapped model)
void mixture_moments_impl(const Model& m, double* mean, double* m2) {
  const int d = m.d;
  double mu[3] = {0, 0, 0}, s2[9] = {0};
  for (const Comp& c : m.c) {
    for (int a = 0; a < d; ++a) mu[a] += c.w * c.mu[a];
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) s2[a * d + b] += c.w * (c.cov[a][b] + c.mu[a] * c.mu[b]);
  }
  if (m.identity()) {
    std::copy(mu, mu + d, mean);
    std::copy(s2, s2 + d * d, m2);
    return;
  }
  for (int a = 0; a < d; ++a) mean[a] = mu[a] * m.scale[a] + m.offset[a];
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b)
      m2[a * d + b] = m.scale[a] * s2[a * d + b] * m.scale[b] + m.scale[a] * mu[a] * m.offset[b] +
                      m.offset[a] * (m.scale[b] * mu[b]) + m.offset[a] * m.offset[b];
}

// metrics.cpp:58-65 moment_errors
void moment_errors_impl(const Model& m, const Points& p, double* mean_err, double* m2_err) {
  const int d = m.d;
  double mm[3], m2[9], dm[3], d2[9];
  mixture_moments_impl(m, mm, m2);
  data_moments(p, dm, d2);
  double tr = 0.0, num = 0.0, n2 = 0.0, dn = 0.0;
  for (int a = 0; a < d; ++a) tr += d2[a * d + a];
  for (int a = 0; a < d; ++a) num += (mm[a] - dm[a]) * (mm[a] - dm[a]);
  for (int e = 0; e < d * d; ++e) {
    n2 += (m2[e] - d2[e]) * (m2[e] - d2[e]);
    dn += d2[e] * d2[e];
  }
  *mean_err = std::sqrt(num) / std::sqrt(tr);
  *m2_err = std::sqrt(n2) / std::sqrt(dn);
}

int64_t payload_bytes(int M, int d) { return static_cast<int64_t>(M) * (1 + d + d * (d + 1) / 2) * 8; }

}  // namespace

// ===========================================================================
extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

void oracle_uniforms(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
}

int oracle_generate(int32_t d, int32_t m, const double* fractions, const double* means,
                    const double* covs, int64_t n, uint64_t seed, double* vel, double* temp) {
  return guarded([&] {
    if (d != 2 && d != 3) throw std::invalid_argument("scenario dimension must be 2 or 3");
    if (n < 1) throw std::invalid_argument("particle_count must be >= 1");
    if (m < 1) throw std::invalid_argument("scenario needs at least one component");
    double total = 0.0;
    std::vector<Mat3> chol(m);
    std::vector<double> cdf(m);
    double acc = 0.0;
    for (int k = 0; k < m; ++k) {
      Mat3 c{};
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) c[a][b] = covs[(k * d + a) * d + b];
      if (!cholesky(c, d, chol[k]))
        throw std::invalid_argument("component " + std::to_string(k) +
                                    ": covariance is not symmetric positive definite");
      total += fractions[k];
      acc += fractions[k];
      cdf[k] = acc;
    }
    if (std::fabs(total - 1.0) > 1e-12)
      throw std::invalid_argument("fractions must sum to 1 (got " + std::to_string(total) + ")");
    cdf[m - 1] = 1.0;
    for (int a = 0; a < d; ++a) temp[a] = 0.0;
    for (int k = 0; k < m; ++k)
      for (int a = 0; a < d; ++a) temp[a] += fractions[k] * covs[(k * d + a) * d + a];
    Rng rng(seed);
    double z[3];
    for (int64_t r = 0; r < n; ++r) {
      const double u = rng.uniform();
      int k = 0;
      while (k + 1 < m && u >= cdf[k]) ++k;
      for (int a = 0; a < d; ++a) z[a] = rng.normal();
      for (int a = 0; a < d; ++a) {
        double s = 0.0;
        for (int b = 0; b < d; ++b) s += chol[k][a][b] * z[b];
        vel[a * n + r] = means[k * d + a] + s;
      }
    }
  });
}

int oracle_bin_particles(const double* vel, int64_t n, int32_t d, const double* w, int32_t plane,
                         int32_t nb, double xlo, double xhi, double ylo, double yhi,
                         double* counts, double* oor) {
  return guarded([&] { bin2d(vel, n, d, w, plane, nb, xlo, xhi, ylo, yhi, counts, oor); });
}

int oracle_all_planes(const double* vel, int64_t n, int32_t d, const double* w, int32_t nb,
                      double lo, double hi, double* counts3, double* oor3) {
  return guarded([&] {
    if (d != 3)
      throw std::invalid_argument("all_planes requires d=3 particles; use bin_particles for d=2");
    const int64_t stride = static_cast<int64_t>(nb) * nb;
    for (int p = 0; p < 3; ++p)
      bin2d(vel, n, d, w, p, nb, lo, hi, lo, hi, counts3 + p * stride, oor3 + p);
  });
}

int oracle_to_weighted_points(const double* counts, int32_t nb, double xlo, double xhi,
                              double ylo, double yhi, int32_t drop_empty, int64_t capacity,
                              double* points, double* weights, int64_t* count,
                              double* total_weight) {
  return guarded([&] {
    const int64_t nn = static_cast<int64_t>(nb) * nb;
    double tot = 0.0;
    for (int64_t f = 0; f < nn; ++f) tot += counts[f];  // Histogram2D::in_range_count
    if (!(tot > 0.0)) throw std::invalid_argument("degenerate histogram: no in-range weight");
    int64_t kept = 0;
    if (drop_empty) {
      for (int64_t f = 0; f < nn; ++f)
        if (counts[f] > 0.0) ++kept;
    } else {
      kept = nn;
    }
    if (kept > capacity) throw std::invalid_argument("to_weighted_points: capacity too small");
    int64_t r = 0;
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < nb; ++j) {
        const double w = counts[i + static_cast<int64_t>(j) * nb];
        if (drop_empty && !(w > 0.0)) continue;
        points[r] = center(xlo, xhi, nb, i);
        points[kept + r] = center(ylo, yhi, nb, j);
        weights[r] = w;
        ++r;
      }
    *count = kept;
    *total_weight = tot;
  });
}

int oracle_validate_fit_config(const vdfcg_fit_config* cfg, int32_t d) {
  return guarded([&] { validate_config(cfg, d); });
}

int oracle_normalize(const double* points, const double* weights, int64_t n, int32_t d,
                     double* out_points, double* scale, double* offset) {
  return guarded([&] {
    Points p = make_points(points, weights, n, d, 0.0);
    Points o;
    normalize_impl(p, o, scale, offset);
    std::copy(o.x.begin(), o.x.end(), out_points);
  });
}

int oracle_denormalize_model(const vdfcg_model* in, vdfcg_model* out) {
  return guarded([&] { to_view(denormalize_impl(from_view(in)), out); });
}

int oracle_init_model(const double* np, int64_t n, int32_t d, const vdfcg_fit_config* cfg,
                      const double* temperature, const double* scale, const double* offset,
                      vdfcg_model* out) {
  return guarded([&] {
    std::vector<double> w(n, 1.0);
    Points p = make_points(np, w.data(), n, d, 0.0);
    to_view(init_impl(p, cfg, temperature, scale, offset), out);
  });
}

int oracle_e_step(vdfcg_model* model, const double* points, const double* weights, int64_t n,
                  double* resp, double* loglik, int32_t* unrep, int32_t* n_unrep) {
  return guarded([&] {
    Model m = from_view(model);
    Points p = make_points(points, weights, n, m.d, 0.0);
    std::vector<double> r;
    std::vector<int> u;
    *loglik = e_step_impl(m, p, r, u);
    std::copy(r.begin(), r.end(), resp);
    for (size_t i = 0; i < u.size(); ++i) unrep[i] = u[i];
    *n_unrep = static_cast<int32_t>(u.size());
    to_view(m, model);  // in-place covariance repair is visible to the caller
  });
}

int oracle_m_step(const double* points, const double* weights, int64_t n, double total,
                  const double* resp, const vdfcg_model* prev, vdfcg_model* out, int32_t* degen,
                  int32_t* n_degen) {
  return guarded([&] {
    Model pm = from_view(prev);
    Points p = make_points(points, weights, n, pm.d, total);
    const size_t M = pm.c.size();
    std::vector<double> r(resp, resp + M * n);
    std::vector<int> dg;
    Model o = m_step_impl(p, total, r, pm, &dg);
    to_view(o, out);
    if (degen)
      for (size_t i = 0; i < dg.size(); ++i) degen[i] = dg[i];
    if (n_degen) *n_degen = static_cast<int32_t>(dg.size());
  });
}

int oracle_prune_one(vdfcg_model* model, double threshold, int32_t iteration, int32_t* pruned,
                     int32_t* ev_comp, double* ev_w) {
  (void)iteration;
  return guarded([&] {
    Model m = from_view(model);
    int idx = -1;
    double w = 0.0;
    const bool p = prune_one_impl(m, threshold, &idx, &w);
    *pruned = p ? 1 : 0;
    if (p) {
      *ev_comp = idx;
      *ev_w = w;
    }
    to_view(m, model);
  });
}

int oracle_repair_covariance(const double* sigma, int32_t d, double* out, int32_t* doublings) {
  return guarded([&] {
    Mat3 s{};
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) s[a][b] = sigma[a * d + b];
    int db = -1;
    Mat3 r = repair_impl(s, d, &db);
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) out[a * d + b] = r[a][b];
    if (doublings) *doublings = db;
  });
}

int oracle_fit(const double* points, const double* weights, int64_t n, int32_t d,
               double total_weight, const vdfcg_fit_config* cfg, vdfcg_fit_result* res) {
  return guarded([&] {
    Points p = make_points(points, weights, n, d, total_weight);
    FitOut f = fit_impl(p, cfg);
    write_fit_result(f, res);
  });
}

int oracle_mixture_moments(const vdfcg_model* model, double* mean, double* m2) {
  return guarded([&] {
    Model m = from_view(model);
    const int d = m.d;
    for (int a = 0; a < d; ++a) mean[a] = 0.0;
    for (int a = 0; a < d * d; ++a) m2[a] = 0.0;
    for (const Comp& c : m.c) {
      for (int a = 0; a < d; ++a) mean[a] += c.w * c.mu[a];
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) m2[a * d + b] += c.w * (c.cov[a][b] + c.mu[a] * c.mu[b]);
    }
    if (m.identity()) return;
    // wgmm.cpp:463-469: pull back to data space.
    double mx[3], m2x[9];
    for (int a = 0; a < d; ++a) mx[a] = mean[a] * m.scale[a] + m.offset[a];
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) {
        const double sa = m.scale[a], sb = m.scale[b];
        m2x[a * d + b] = sa * m2[a * d + b] * sb + sa * mean[a] * m.offset[b] +
                         m.offset[a] * (sb * mean[b]) + m.offset[a] * m.offset[b];
      }
    std::copy(mx, mx + d, mean);
    std::copy(m2x, m2x + d * d, m2);
  });
}

int oracle_weighted_data_moments(const double* points, const double* weights, int64_t n, int32_t d,
                                 double* mean, double* m2) {
  return guarded([&] {
    Points p = make_points(points, weights, n, d, 0.0);
    data_moments(p, mean, m2);
  });
}

int64_t oracle_model_payload_bytes(int32_t m, int32_t d) {
  return static_cast<int64_t>(m) * (1 + d + d * (d + 1) / 2) * 8;
}

int oracle_encode_model(const vdfcg_model* model, const vdfcg_model_meta* meta, uint8_t* out,
                        int64_t capacity, int64_t* length) {
  return guarded([&] {
    std::vector<uint8_t> b = encode_impl(from_view(model), meta);
    if (static_cast<int64_t>(b.size()) > capacity)
      throw std::invalid_argument("encode_model: capacity too small");
    std::copy(b.begin(), b.end(), out);
    *length = static_cast<int64_t>(b.size());
  });
}

int oracle_bin_cells(const vdfcg_cells* cells, vdfcg_cell_bins* out) {
  return guarded([&] {
    std::vector<double> dense;
    for (int c = 0; c < cells->n_cells; ++c)
      bin_one_cell(cells, c, dense, out->keys, out->counts, &out->nnz[c], &out->out_of_range[c],
                   &out->in_range[c]);
  });
}

// Per-particle cell ids (vdfcg_particles): a stable counting sort by cell id keeps every
// cell's particles in input order (the sequential order the reference would sum a part's
// weights in, histogram.cpp:66-74), then each cell is binned as above. offsets: [n_cells+1].
int oracle_bin_cells_indexed(const vdfcg_particles* p, int64_t* offsets, vdfcg_cell_bins* out) {
  return guarded([&] {
    const int64_t n = p->n_particles;
    const int nc = p->n_cells;
    std::vector<int64_t> cnt(size_t(nc) + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
      const int32_t c = p->cell[i];
      if (c < 0 || c >= nc) throw std::invalid_argument("cell index out of range");
      ++cnt[size_t(c) + 1];
    }
    for (int c = 0; c < nc; ++c) cnt[size_t(c) + 1] += cnt[size_t(c)];
    for (int c = 0; c <= nc; ++c) offsets[c] = cnt[size_t(c)];
    const int d = p->dimension;
    std::vector<double> vel(size_t(d) * size_t(n)), w(p->weights ? size_t(n) : 0);
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t r = pos[size_t(p->cell[i])]++;
      for (int a = 0; a < d; ++a) vel[size_t(a) * n + r] = p->velocity[a][i];
      if (p->weights) w[size_t(r)] = p->weights[i];
    }
    vdfcg_cells cells{};
    cells.dimension = d;
    cells.n_particles = n;
    for (int a = 0; a < d; ++a) cells.velocity[a] = vel.data() + size_t(a) * n;
    cells.weights = p->weights ? w.data() : nullptr;
    cells.n_cells = nc;
    cells.cell_offsets = offsets;
    cells.n_bins = p->n_bins;
    for (int a = 0; a < 3; ++a) {
      cells.lo[a] = p->lo[a];
      cells.hi[a] = p->hi[a];
    }
    std::vector<double> dense;
    for (int c = 0; c < nc; ++c)
      bin_one_cell(&cells, c, dense, out->keys, out->counts, &out->nnz[c], &out->out_of_range[c],
                   &out->in_range[c]);
  });
}

int oracle_compress_cells(const vdfcg_cells* cells, const vdfcg_fit_config* cfg,
                          int32_t cell_begin, int32_t cell_end, int32_t threads,
                          vdfcg_cell_bins* bins, vdfcg_cell_results* out) {
  return guarded([&] {
    validate_config(cfg, cells->dimension);
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    std::atomic<int> next{cell_begin};
    const int d = cells->dimension;
    const int K = out->capacity_components;
    auto worker = [&] {
      std::vector<double> dense;
      for (;;) {
        const int c = next.fetch_add(1);
        if (c >= cell_end) break;
        bin_one_cell(cells, c, dense, bins->keys, bins->counts, &bins->nnz[c],
                     &bins->out_of_range[c], &bins->in_range[c]);
        int status = VDFCG_OK;
        FitOut f;
        try {
          if (!(bins->in_range[c] > 0.0))
            throw std::invalid_argument("degenerate histogram: no in-range weight");
          Points p = cell_points(cells, c, bins->keys, bins->counts, bins->nnz[c], bins->in_range[c]);
          f = fit_impl(p, cfg);
        } catch (const std::invalid_argument&) {
          status = VDFCG_INVALID_ARGUMENT;
        } catch (const RepairError&) {
          status = VDFCG_REPAIR_FAILED;
        } catch (const std::exception&) {
          status = VDFCG_RUNTIME_ERROR;
        }
        out->status[c] = status;
        const int M = status == VDFCG_OK ? static_cast<int>(f.model.c.size()) : 0;
        out->components[c] = M;
        out->iterations[c] = status == VDFCG_OK ? f.iterations : 0;
        out->converged[c] = status == VDFCG_OK && f.converged ? 1 : 0;
        for (int i = 0; i < M; ++i) {
          out->weights[c * K + i] = f.model.c[i].w;
          for (int a = 0; a < d; ++a) out->means[(c * K + i) * d + a] = f.model.c[i].mu[a];
          for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b)
              out->covariances[((c * K + i) * d + a) * d + b] = f.model.c[i].cov[a][b];
        }
        out->final_loglik[c] = (status == VDFCG_OK && !f.trace.empty()) ? f.trace.back() : kNaN;
        if (out->loglik_trace && out->capacity_trace > 0)
          for (int t = 0; t < out->capacity_trace; ++t)
            out->loglik_trace[static_cast<int64_t>(c) * out->capacity_trace + t] =
                t < static_cast<int>(f.trace.size()) ? f.trace[t] : kNaN;
        if (out->n_events) {
          const int ne = std::min<int>(static_cast<int>(f.events.size()), K);
          out->n_events[c] = ne;
          for (int e = 0; e < ne; ++e) {
            if (out->event_iteration) out->event_iteration[c * K + e] = static_cast<int32_t>(f.events[e][0]);
            if (out->event_component) out->event_component[c * K + e] = static_cast<int32_t>(f.events[e][1]);
            if (out->event_weight) out->event_weight[c * K + e] = f.events[e][2];
          }
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
  });
}

int oracle_pack_cells(int32_t n_cells, int32_t d, const vdfcg_cell_results* res,
                      const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                      int64_t* offsets) {
  return guarded([&] {
    const int K = res->capacity_components;
    int64_t pos = 0;
    offsets[0] = 0;
    for (int c = 0; c < n_cells; ++c) {
      if (res->status[c] == VDFCG_OK && res->components[c] > 0) {
        Model m;
        m.d = d;
        m.c.resize(res->components[c]);
        for (int i = 0; i < res->components[c]; ++i) {
          m.c[i].w = res->weights[c * K + i];
          for (int a = 0; a < d; ++a) m.c[i].mu[a] = res->means[(c * K + i) * d + a];
          for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b)
              m.c[i].cov[a][b] = res->covariances[((c * K + i) * d + a) * d + b];
        }
        // The batched writer packs the fit output without re-validating it.
        const std::vector<uint8_t> hdr_and_payload = encode_impl(m, meta, false);
        if (pos + static_cast<int64_t>(hdr_and_payload.size()) > capacity)
          throw std::invalid_argument("pack_cells: capacity too small");
        std::copy(hdr_and_payload.begin(), hdr_and_payload.end(), records + pos);
        pos += static_cast<int64_t>(hdr_and_payload.size());
      }
      offsets[c + 1] = pos;
    }
  });
}

int oracle_evaluate_pdf(const vdfcg_model* model, int32_t nb, double xlo, double xhi, double ylo,
                        double yhi, double* out) {
  return guarded([&] {
    const Model m = from_view(model);
    if (m.d != 2) throw std::invalid_argument("evaluate_pdf expects a 2-dimensional model");
    if (!(nb >= 1) || !(xlo < xhi) || !(ylo < yhi) || !std::isfinite(xlo) || !std::isfinite(xhi) ||
        !std::isfinite(ylo) || !std::isfinite(yhi))
      throw std::invalid_argument("invalid grid spec");
    const double lo[2] = {xlo, ylo}, hi[2] = {xhi, yhi};
    std::vector<double> g;
    evaluate_grid(m, nb, lo, hi, g);
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < nb; ++j) out[i + static_cast<int64_t>(j) * nb] = g[static_cast<int64_t>(i) * nb + j];
  });
}

int oracle_weighted_loglik(const vdfcg_model* model, const double* points, const double* weights,
                           int64_t n, double* out) {
  return guarded([&] {
    const Model m = from_view(model);
    Points p = make_points(points, weights, n, m.d, 0.0);
    *out = weighted_loglik_impl(m, p);
  });
}

int oracle_pdf_divergences(const double* p, const double* q, int64_t n, double area, double* jsd,
                           double* kl_pq, double* kl_qp) {
  return guarded([&] {
    if (kl_pq) *kl_pq = kl_impl(p, q, n, area);
    if (kl_qp) *kl_qp = kl_impl(q, p, n, area);
    if (jsd) *jsd = jsd_impl(p, q, n, area);
  });
}

int oracle_cell_metrics(const vdfcg_cells* cells, const vdfcg_cell_bins* bins,
                        const vdfcg_cell_results* res, int32_t cell_begin, int32_t cell_end,
                        int32_t threads, vdfcg_cell_metrics* out) {
  return guarded([&] {
    const int d = cells->dimension;
    const int nb = cells->n_bins;
    const int K = res->capacity_components;
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    std::atomic<int> next{cell_begin};
    auto put = [](double* a, int c, double v) {
      if (a) a[c] = v;
    };
    auto worker = [&] {
      std::vector<double> hist, model;
      for (;;) {
        const int c = next.fetch_add(1);
        if (c >= cell_end) break;
        double v[10];
        std::fill(v, v + 10, kNaN);
        const int M = res->components[c];
        if (res->status[c] == VDFCG_OK && M > 0 && bins->in_range[c] > 0.0) {
          try {
            Model m;
            m.d = d;
            m.c.resize(M);
            for (int i = 0; i < M; ++i) {
              m.c[i].w = res->weights[c * K + i];
              for (int a = 0; a < d; ++a) m.c[i].mu[a] = res->means[(c * K + i) * d + a];
              for (int a = 0; a < d; ++a)
                for (int b = 0; b < d; ++b)
                  m.c[i].cov[a][b] = res->covariances[((c * K + i) * d + a) * d + b];
            }
            double area = 1.0;
            int64_t total = 1;
            for (int a = 0; a < d; ++a) {
              area *= (cells->hi[a] - cells->lo[a]) / nb;
              total *= nb;
            }
            const int64_t b0 = cells->cell_offsets[c];
            hist.assign(total, 0.0);
            for (int r = 0; r < bins->nnz[c]; ++r) hist[bins->keys[b0 + r]] = bins->counts[b0 + r];
            normalize_grid(hist, area);  // to_pdf (histogram.cpp:111-115)
            evaluate_grid(m, nb, cells->lo, cells->hi, model);
            normalize_grid(model, area);
            v[0] = jsd_impl(hist.data(), model.data(), total, area);
            v[1] = kl_impl(hist.data(), model.data(), total, area);
            v[2] = kl_impl(model.data(), hist.data(), total, area);
            const Points p = cell_points(cells, c, bins->keys, bins->counts, bins->nnz[c], bins->in_range[c]);
            const double ll = weighted_loglik_impl(m, p);
            const double k = static_cast<double>(M * (1 + d * (d + 3) / 2));
            v[3] = ll;
            v[4] = -2.0 * ll + k * std::log(p.total);
            v[5] = -2.0 * ll + k * std::log(static_cast<double>(total));
            moment_errors_impl(m, p, &v[6], &v[7]);
            const double mb = static_cast<double>(payload_bytes(M, d));
            v[8] = static_cast<double>(total * 8) / mb;
            v[9] = static_cast<double>((cells->cell_offsets[c + 1] - b0) * d * 8) / mb;
          } catch (const std::exception&) {
            std::fill(v, v + 10, kNaN);
          }
        }
        put(out->jsd, c, v[0]);
        put(out->kl_pq, c, v[1]);
        put(out->kl_qp, c, v[2]);
        put(out->loglik, c, v[3]);
        put(out->bic, c, v[4]);
        put(out->bic_bin_count, c, v[5]);
        put(out->mean_moment_error, c, v[6]);
        put(out->second_moment_error, c, v[7]);
        put(out->compression_ratio_vs_histogram, c, v[8]);
        put(out->compression_ratio_vs_raw, c, v[9]);
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
  });
}

}  // extern "C"
