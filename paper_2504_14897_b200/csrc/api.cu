// api.cu — the extern "C" entry points of include/vdfcg.h. Host code here only
// validates arguments (the reference's precondition checks and messages), stages host
// buffers through the context stream and launches the sm_100a kernels; every number the
// API returns is computed on the device.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "em.cuh"
#include "em_entry.cuh"
#include "hist.cuh"
#include "api.cuh"
#include "metrics.cuh"
#include "pack.cuh"

namespace vdfcg {
void launch_synth(vdfcg_ctx* ctx, int d, int n_cells, const int64_t* offsets, int64_t cell_base,
                  uint64_t seed, int species, double* u, double* v, double* w);
void launch_generate(vdfcg_ctx* ctx, int d, int m, int64_t n, uint64_t seed, uint64_t* uniforms,
                     int64_t n_uniforms, const double* params, double* vel);
double probe_fp64(vdfcg_ctx* ctx);
double probe_fp32(vdfcg_ctx* ctx);

namespace {

void begin(vdfcg_ctx* ctx) {
  if (!ctx) throw InvalidArgument("null vdfcg context");
  VDFCG_CUDA(cudaSetDevice(ctx->device));
  arena_reset(ctx);
}

bool range_ok(double lo, double hi) { return std::isfinite(lo) && std::isfinite(hi) && lo < hi; }

const char* plane_name(int p) { return p == 0 ? "uv" : p == 1 ? "vw" : "uw"; }

void plane_axes(int plane, int* ax, int* ay) {
  switch (plane) {
    case 0: *ax = 0; *ay = 1; return;
    case 1: *ax = 1; *ay = 2; return;
    case 2: *ax = 0; *ay = 2; return;
    default: throw InvalidArgument("unknown plane id " + std::to_string(plane));
  }
}

// FitConfig::validate (wgmm.cpp:65-76)
void validate_config(const vdfcg_fit_config* cfg, int d) {
  if (!cfg) throw InvalidArgument("null fit config");
  if (cfg->initial_components < 1) throw InvalidArgument("initial_components must be >= 1");
  if (cfg->initial_components > VDFCG_MAX_COMPONENTS)
    throw InvalidArgument("initial_components must be <= 16 on this implementation");
  if (cfg->max_em_iterations < 1) throw InvalidArgument("max_em_iterations must be >= 1");
  if (!(cfg->prune_threshold > 0.0)) throw InvalidArgument("prune_threshold must be > 0");
  if (cfg->prune_threshold >= 1.0 / cfg->initial_components)
    throw InvalidArgument("prune_threshold must be < 1/initial_components");
  if (cfg->prune_check_interval < 1) throw InvalidArgument("prune_check_interval must be >= 1");
  if (!(cfg->loglik_rel_tolerance > 0.0))
    throw InvalidArgument("loglik_rel_tolerance must be > 0");
  if (cfg->has_temperature)
    for (int a = 0; a < d; ++a)
      if (!(cfg->temperature[a] > 0.0))
        throw InvalidArgument("temperature must be > 0 on every axis");
  if (cfg->warm_start) {
    if (cfg->warm_start->dimension != d)
      throw InvalidArgument("warm-start model dimension does not match the data");
    if (cfg->warm_start->components < 1 || cfg->warm_start->components > VDFCG_MAX_COMPONENTS)
      throw InvalidArgument("warm-start model must have 1..16 components");
  }
}

// Device-side EmConfig: uniforms from mt19937_64(seed) and the canonical warm model.
EmConfig make_em_config(vdfcg_ctx* ctx, const vdfcg_fit_config* cfg, int d) {
  EmConfig e{};
  e.M = cfg->initial_components;
  e.max_it = cfg->max_em_iterations;
  e.prune_thr = cfg->prune_threshold;
  e.interval = cfg->prune_check_interval;
  e.tol = cfg->loglik_rel_tolerance;
  e.has_temp = cfg->has_temperature ? 1 : 0;
  for (int a = 0; a < 3; ++a) e.temp[a] = cfg->temperature[a];
  double* u = arena<double>(ctx, 64);
  launch_mt_uniforms(ctx, cfg->seed, VDFCG_MAX_COMPONENTS * 3, u);
  e.uniforms = u;
  e.exact_counter = ctx->diag;
  e.f32 = cfg->estep_fp32 ? 1 : 0;
  if (cfg->warm_start) {
    const vdfcg_model* w = cfg->warm_start;
    const int m = w->components;
    auto sw = stage_in(ctx, w->weights, m);
    auto smu = stage_in(ctx, w->means, size_t(m) * d);
    auto scv = stage_in(ctx, w->covariances, size_t(m) * d * d);
    auto ssc = stage_in(ctx, w->scale, w->scale ? d : 0);
    auto sof = stage_in(ctx, w->offset, w->offset ? d : 0);
    double* ow = arena<double>(ctx, m);
    double* omu = arena<double>(ctx, size_t(m) * d);
    double* ocv = arena<double>(ctx, size_t(m) * d * d);
    launch_canonicalize(ctx, d, m, sw.dev, smu.dev, scv.dev, (w->scale && w->offset) ? ssc.dev : nullptr,
                        (w->scale && w->offset) ? sof.dev : nullptr, ow, omu, ocv);
    e.warm_m = m;
    e.warm_w = ow;
    e.warm_mu = omu;
    e.warm_cov = ocv;
  }
  return e;
}

template <class T>
void copy_out(vdfcg_ctx* ctx, T* dst, const T* src, size_t count) {
  if (dst && count)
    VDFCG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDefault, ctx->stream));
}

template <class T>
T read_scalar(vdfcg_ctx* ctx, const T* dev) {
  T* h = static_cast<T*>(ctx->pinned);
  VDFCG_CUDA(cudaMemcpyAsync(h, dev, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  return *h;
}

struct EmOutDev {
  EmOut o;
  std::vector<int> dummy;
};

EmOut alloc_em_out(vdfcg_ctx* ctx, int n_cells, int d, int K, int trace_cap, bool events) {
  EmOut o{};
  o.K = K;
  o.trace_cap = trace_cap;
  o.status = arena<int32_t>(ctx, n_cells);
  o.comps = arena<int32_t>(ctx, n_cells);
  o.iters = arena<int32_t>(ctx, n_cells);
  o.conv = arena<int32_t>(ctx, n_cells);
  o.w = arena<double>(ctx, size_t(n_cells) * K);
  o.mu = arena<double>(ctx, size_t(n_cells) * K * d);
  o.cov = arena<double>(ctx, size_t(n_cells) * K * d * d);
  o.final_ll = arena<double>(ctx, n_cells);
  o.trace = trace_cap > 0 ? arena<double>(ctx, size_t(n_cells) * trace_cap) : nullptr;
  if (events) {
    o.n_events = arena<int32_t>(ctx, n_cells);
    o.ev_it = arena<int32_t>(ctx, size_t(n_cells) * K);
    o.ev_comp = arena<int32_t>(ctx, size_t(n_cells) * K);
    o.ev_w = arena<double>(ctx, size_t(n_cells) * K);
  }
  o.err_axis = arena<int32_t>(ctx, n_cells);
  o.err_value = arena<double>(ctx, n_cells);
  return o;
}

void throw_status(int status, int err_id, double err_value, bool fit_prefix) {
  const std::string msg = prologue_message(status, err_id, err_value, fit_prefix);
  if (status == VDFCG_INVALID_ARGUMENT) throw InvalidArgument(msg);
  if (status == VDFCG_REPAIR_FAILED) throw RepairFailed(msg);
  throw RuntimeError(msg);
}

CellsDev stage_cells(vdfcg_ctx* ctx, const vdfcg_cells* cells) {
  if (!cells) throw InvalidArgument("null cells");
  const int d = cells->dimension;
  if (d != 2 && d != 3) throw InvalidArgument("particle dimension must be 2 or 3");
  if (cells->n_bins < 2) throw InvalidArgument("n_bins must be >= 2");
  double nbd = 1.0;
  for (int a = 0; a < d; ++a) nbd *= cells->n_bins;
  if (nbd > 2147483647.0) throw InvalidArgument("n_bins^d must fit a 31-bit bin key");
  if (d == 3 && cells->n_bins > 1024) throw InvalidArgument("3V cells support n_bins <= 1024");
  for (int a = 0; a < d; ++a)
    if (!range_ok(cells->lo[a], cells->hi[a]))
      throw InvalidArgument("axis range must satisfy min < max");
  if (cells->n_cells < 0 || cells->n_particles < 0) throw InvalidArgument("negative sizes");
  if (!cells->cell_offsets) throw InvalidArgument("cell_offsets is required");
  CellsDev c{};
  c.d = d;
  c.n = cells->n_particles;
  for (int a = 0; a < d; ++a) {
    if (!cells->velocity[a] && c.n) throw InvalidArgument("missing velocity axis");
    c.vel[a] = stage_in(ctx, cells->velocity[a], c.n).dev;
  }
  for (int a = d; a < 3; ++a) c.vel[a] = c.vel[0];
  c.w = cells->weights ? stage_in(ctx, cells->weights, c.n).dev : nullptr;
  c.n_cells = cells->n_cells;
  c.offsets = stage_in(ctx, cells->cell_offsets, size_t(c.n_cells) + 1).dev;
  c.n_bins = cells->n_bins;
  for (int a = 0; a < 3; ++a) {
    c.lo[a] = cells->lo[a];
    c.hi[a] = cells->hi[a];
  }
  return c;
}

PackMeta make_pack_meta(vdfcg_ctx* ctx, const vdfcg_model_meta* meta, int d) {
  if (!meta) throw InvalidArgument("null model meta");
  if (meta->label_len < 0 || meta->label_len > 0xffff) throw InvalidArgument("species label too long");
  PackMeta pm{};
  pm.d = d;
  pm.plane = (meta->plane >= 0 && meta->plane <= 2) ? meta->plane : 255;
  pm.cycle = meta->cycle;
  for (int a = 0; a < 3; ++a) {
    pm.lo[a] = meta->range_lo[a];
    pm.hi[a] = meta->range_hi[a];
  }
  pm.label_len = meta->label_len;
  uint8_t* lab = arena<uint8_t>(ctx, std::max(meta->label_len, 1));
  if (meta->label_len)
    VDFCG_CUDA(cudaMemcpyAsync(lab, meta->species_label, meta->label_len, cudaMemcpyDefault, ctx->stream));
  pm.label = lab;
  return pm;
}

// GmmModel::validate (wgmm.cpp:46-63) on the device.
__global__ void validate_model_kernel(int d, int m, const double* w, const double* cov, int* code) {
  if (threadIdx.x != 0) return;
  int c = 0;
  if (m < 1) c = 1;
  double total = 0.0;
  for (int i = 0; i < m && !c; ++i) {
    if (!(w[i] > 0.0)) c = 2;
    for (int a = 0; a < d && !c; ++a)
      for (int b = 0; b < d; ++b)
        if (!(cov[(i * d + a) * d + b] == cov[(i * d + b) * d + a])) c = 3;
    total = __dadd_rn(total, w[i]);
  }
  if (!c && fabs(total - 1.0) > 1e-12) c = 4;
  *code = c;
}

}  // namespace
}  // namespace vdfcg

using namespace vdfcg;

extern "C" {

int vdfcg_validate_fit_config(const vdfcg_fit_config* cfg, int32_t d) {
  return guard_impl([&] { validate_config(cfg, d); });
}

int64_t vdfcg_model_payload_bytes(int32_t m, int32_t d) { return payload_bytes(m, d); }
int64_t vdfcg_model_header_bytes(int32_t d, int32_t l) { return header_bytes(d, l); }

// ------------------------------------------------------------------ histogram
int vdfcg_bin_particles(vdfcg_ctx* ctx, const double* velocities, int64_t n, int32_t d,
                        const double* weights, int32_t plane, int32_t n_bins, double xlo,
                        double xhi, double ylo, double yhi, double* counts, double* oor) {
  return guard_impl([&] {
    begin(ctx);
    if (d != 2 && d != 3) throw InvalidArgument("particle dimension must be 2 or 3");
    if (n_bins < 2) throw InvalidArgument("n_bins must be >= 2");
    if (!range_ok(xlo, xhi) || !range_ok(ylo, yhi))
      throw InvalidArgument("axis range must satisfy min < max");
    int ax, ay;
    plane_axes(plane, &ax, &ay);
    if (ay >= d)
      throw InvalidArgument(std::string("plane ") + plane_name(plane) +
                            " requires the w axis, but particles are " + std::to_string(d) +
                            "-dimensional");
    if (!counts || !oor) throw InvalidArgument("null output");
    auto v = stage_in(ctx, velocities, size_t(n) * d);
    auto w = stage_in(ctx, weights, weights ? size_t(n) : 0);
    const size_t nn = size_t(n_bins) * n_bins;
    auto c = stage_out(ctx, counts, nn);
    auto o = stage_out(ctx, oor, 1);
    launch_hist2d(ctx, v.dev, n, d, weights ? w.dev : nullptr, 1, &ax, &ay, n_bins, &xlo, &xhi,
                  &ylo, &yhi, c.dev, o.dev);
    finish(ctx, c);
    finish(ctx, o);
    sync(ctx);
  });
}

int vdfcg_all_planes(vdfcg_ctx* ctx, const double* velocities, int64_t n, int32_t d,
                     const double* weights, int32_t n_bins, double lo, double hi, double* counts3,
                     double* oor3) {
  return guard_impl([&] {
    begin(ctx);
    if (d != 3) throw InvalidArgument("all_planes requires d=3 particles; use bin_particles for d=2");
    if (n_bins < 2) throw InvalidArgument("n_bins must be >= 2");
    if (!range_ok(lo, hi)) throw InvalidArgument("axis range must satisfy min < max");
    auto v = stage_in(ctx, velocities, size_t(n) * d);
    auto w = stage_in(ctx, weights, weights ? size_t(n) : 0);
    const size_t nn = size_t(n_bins) * n_bins;
    auto c = stage_out(ctx, counts3, 3 * nn);
    auto o = stage_out(ctx, oor3, 3);
    const int ax[3] = {0, 1, 0}, ay[3] = {1, 2, 2};
    const double l3[3] = {lo, lo, lo}, h3[3] = {hi, hi, hi};
    launch_hist2d(ctx, v.dev, n, d, weights ? w.dev : nullptr, 3, ax, ay, n_bins, l3, h3, l3, h3,
                  c.dev, o.dev);
    finish(ctx, c);
    finish(ctx, o);
    sync(ctx);
  });
}

int vdfcg_to_weighted_points(vdfcg_ctx* ctx, const double* counts, int32_t n_bins, double xlo,
                             double xhi, double ylo, double yhi, int32_t drop_empty,
                             int64_t capacity, double* points, double* weights, int64_t* count,
                             double* total_weight) {
  return guard_impl([&] {
    begin(ctx);
    if (n_bins < 1) throw InvalidArgument("n_bins must be >= 1");
    if (!count || !total_weight) throw InvalidArgument("null output");
    const size_t nn = size_t(n_bins) * n_bins;
    auto c = stage_in(ctx, counts, nn);
    const size_t cap = static_cast<size_t>(std::max<int64_t>(capacity, 0));
    double* pd = arena<double>(ctx, 2 * cap);
    double* wd = arena<double>(ctx, cap);
    double* td = arena<double>(ctx, 1);
    const int64_t k = launch_to_weighted_points(ctx, c.dev, n_bins, xlo, xhi, ylo, yhi,
                                                drop_empty != 0, capacity, pd, wd, td);
    const double tot = read_scalar(ctx, td);
    if (!(tot > 0.0)) throw InvalidArgument("degenerate histogram: no in-range weight");
    if (k > capacity) throw InvalidArgument("to_weighted_points: capacity too small");
    copy_out(ctx, points, pd, size_t(2 * k));
    copy_out(ctx, weights, wd, size_t(k));
    sync(ctx);
    *count = k;
    *total_weight = tot;
  });
}

// ------------------------------------------------------------------ EM entry points
int vdfcg_normalize(vdfcg_ctx* ctx, const double* points, const double* weights, int64_t n,
                    int32_t d, double* out_points, double* scale, double* offset) {
  return guard_impl([&] {
    begin(ctx);
    if (d < 2 || d > 3) throw InvalidArgument("dimension must be 2 or 3");
    auto p = stage_in(ctx, points, size_t(n) * d);
    auto w = stage_in(ctx, weights, size_t(n));
    EmConfig cfg{};
    cfg.has_temp = 1;
    cfg.warm_m = 1;  // skips temperature + distinct count: normalize only
    double* z = arena<double>(ctx, size_t(std::max<int64_t>(n, 1)) * d);
    Frame* fr = arena<Frame>(ctx, 1);
    launch_fit_prologue(ctx, d, p.dev, w.dev, n, 0.0, cfg, z, fr);
    Frame F;
    VDFCG_CUDA(cudaMemcpyAsync(&F, fr, sizeof(Frame), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (F.status) throw_status(F.status, F.err_axis, F.err_value, false);
    copy_out(ctx, out_points, z, size_t(n) * d);
    sync(ctx);
    for (int a = 0; a < d; ++a) {
      scale[a] = F.scale[a];
      offset[a] = F.offset[a];
    }
  });
}

int vdfcg_denormalize_model(vdfcg_ctx* ctx, const vdfcg_model* in, vdfcg_model* out) {
  return guard_impl([&] {
    begin(ctx);
    if (!in || !out) throw InvalidArgument("null model");
    const int d = in->dimension, m = in->components;
    auto w = stage_in(ctx, in->weights, m);
    auto mu = stage_in(ctx, in->means, size_t(m) * d);
    auto cv = stage_in(ctx, in->covariances, size_t(m) * d * d);
    const bool map = in->scale && in->offset;
    auto sc = stage_in(ctx, in->scale, map ? d : 0);
    auto of = stage_in(ctx, in->offset, map ? d : 0);
    double* ow = arena<double>(ctx, m);
    double* omu = arena<double>(ctx, size_t(m) * d);
    double* ocv = arena<double>(ctx, size_t(m) * d * d);
    launch_canonicalize(ctx, d, m, w.dev, mu.dev, cv.dev, map ? sc.dev : nullptr, map ? of.dev : nullptr,
                        ow, omu, ocv);
    copy_out(ctx, out->weights, ow, m);
    copy_out(ctx, out->means, omu, size_t(m) * d);
    copy_out(ctx, out->covariances, ocv, size_t(m) * d * d);
    sync(ctx);
    out->dimension = d;
    out->components = m;
    if (out->scale && out->offset)
      for (int a = 0; a < d; ++a) {
        out->scale[a] = 1.0;
        out->offset[a] = 0.0;
      }
  });
}

int vdfcg_init_model(vdfcg_ctx* ctx, const double* normalized_points, int64_t n, int32_t d,
                     const vdfcg_fit_config* cfg, const double* temperature, const double* scale,
                     const double* offset, vdfcg_model* out) {
  return guard_impl([&] {
    begin(ctx);
    validate_config(cfg, d);
    if (!scale || !offset || !out) throw InvalidArgument("null argument");
    if (!cfg->warm_start) {
      for (int a = 0; a < d; ++a)
        if (!(temperature[a] > 0.0))
          throw InvalidArgument("temperature must be a positive per-axis variance");
    }
    EmConfig e = make_em_config(ctx, cfg, d);
    Frame F{};
    for (int a = 0; a < d; ++a) {
      F.scale[a] = scale[a];
      F.offset[a] = offset[a];
      F.temp[a] = temperature ? temperature[a] : 1.0;
    }
    auto z = stage_in(ctx, normalized_points, size_t(n) * d);
    const int K = std::max(cfg->initial_components, e.warm_m);
    double* w = arena<double>(ctx, K);
    double* mu = arena<double>(ctx, size_t(K) * d);
    double* cv = arena<double>(ctx, size_t(K) * d * d);
    int* m = arena<int>(ctx, 1);
    launch_init_model(ctx, d, z.dev, n, e, F, w, mu, cv, m);
    const int M = read_scalar(ctx, m);
    copy_out(ctx, out->weights, w, M);
    copy_out(ctx, out->means, mu, size_t(M) * d);
    copy_out(ctx, out->covariances, cv, size_t(M) * d * d);
    sync(ctx);
    out->dimension = d;
    out->components = M;
    if (out->scale && out->offset)
      for (int a = 0; a < d; ++a) {
        out->scale[a] = scale[a];
        out->offset[a] = offset[a];
      }
  });
}

int vdfcg_e_step(vdfcg_ctx* ctx, vdfcg_model* model, const double* points, const double* weights,
                 int64_t n, double* resp, double* loglik, int32_t* unrepairable,
                 int32_t* n_unrepairable) {
  return guard_impl([&] {
    begin(ctx);
    if (!model) throw InvalidArgument("null model");
    const int d = model->dimension, m = model->components;
    if (d < 1 || d > 3) throw InvalidArgument("model dimension must be 1..3");
    if (m < 1 || m > VDFCG_MAX_COMPONENTS) throw InvalidArgument("model must have 1..16 components");
    auto w = stage_in(ctx, model->weights, m);
    auto mu = stage_in(ctx, model->means, size_t(m) * d);
    auto cv = stage_in(ctx, model->covariances, size_t(m) * d * d);
    auto x = stage_in(ctx, points, size_t(n) * d);
    auto pw = stage_in(ctx, weights, size_t(n));
    double* r = arena<double>(ctx, size_t(m) * n);
    double* ll = arena<double>(ctx, 1);
    int* dead = arena<int>(ctx, VDFCG_MAX_COMPONENTS);
    int* nd = arena<int>(ctx, 1);
    if (d == 1) throw InvalidArgument("e_step supports d = 2 or 3");
    launch_e_step(ctx, d, m, w.dev, mu.dev, cv.dev, x.dev, pw.dev, n, r, ll, dead, nd);
    const int ndead = read_scalar(ctx, nd);
    if (ndead == m) throw RuntimeError("all mixture components are degenerate");
    copy_out(ctx, resp, r, size_t(m) * n);
    copy_out(ctx, model->covariances, cv.dev, size_t(m) * d * d);  // in-place repair
    std::vector<int> dl(VDFCG_MAX_COMPONENTS);
    VDFCG_CUDA(cudaMemcpyAsync(dl.data(), dead, sizeof(int) * VDFCG_MAX_COMPONENTS, cudaMemcpyDeviceToHost, ctx->stream));
    double llh = 0.0;
    VDFCG_CUDA(cudaMemcpyAsync(&llh, ll, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    *loglik = llh;
    for (int i = 0; i < ndead; ++i) unrepairable[i] = dl[i];
    *n_unrepairable = ndead;
  });
}

int vdfcg_m_step(vdfcg_ctx* ctx, const double* points, const double* weights, int64_t n,
                 double total_weight, const double* resp, const vdfcg_model* previous,
                 vdfcg_model* out, int32_t* degenerate, int32_t* n_degenerate) {
  return guard_impl([&] {
    begin(ctx);
    if (!previous || !out) throw InvalidArgument("null model");
    const int d = previous->dimension, m = previous->components;
    if (d < 2 || d > 3) throw InvalidArgument("m_step supports d = 2 or 3");
    if (!(total_weight > 0.0)) throw RuntimeError("m_step: zero total weight");
    auto x = stage_in(ctx, points, size_t(n) * d);
    auto pw = stage_in(ctx, weights, size_t(n));
    auto r = stage_in(ctx, resp, size_t(m) * n);
    auto pmu = stage_in(ctx, previous->means, size_t(m) * d);
    auto pcv = stage_in(ctx, previous->covariances, size_t(m) * d * d);
    double* ow = arena<double>(ctx, m);
    double* omu = arena<double>(ctx, size_t(m) * d);
    double* ocv = arena<double>(ctx, size_t(m) * d * d);
    int* dg = arena<int>(ctx, m);
    int* bad = arena<int>(ctx, 1);
    VDFCG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    launch_m_step(ctx, d, x.dev, pw.dev, n, total_weight, r.dev, m, pmu.dev, pcv.dev, ow, omu, ocv,
                  dg, bad);
    if (read_scalar(ctx, bad)) throw RuntimeError("m_step: invalid responsibility mass");
    copy_out(ctx, out->weights, ow, m);
    copy_out(ctx, out->means, omu, size_t(m) * d);
    copy_out(ctx, out->covariances, ocv, size_t(m) * d * d);
    std::vector<int> h(std::max(m, 1));
    VDFCG_CUDA(cudaMemcpyAsync(h.data(), dg, sizeof(int) * m, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    out->dimension = d;
    out->components = m;
    if (out->scale && out->offset && previous->scale && previous->offset)
      for (int a = 0; a < d; ++a) {
        out->scale[a] = previous->scale[a];
        out->offset[a] = previous->offset[a];
      }
    int k = 0;
    for (int i = 0; i < m; ++i)
      if (h[i]) {
        if (degenerate) degenerate[k] = i;
        ++k;
      }
    if (n_degenerate) *n_degenerate = k;
  });
}

int vdfcg_prune_one(vdfcg_ctx* ctx, vdfcg_model* model, double threshold, int32_t iteration,
                    int32_t* pruned, int32_t* event_component, double* event_weight) {
  (void)iteration;
  return guard_impl([&] {
    begin(ctx);
    if (!model) throw InvalidArgument("null model");
    const int d = model->dimension, m = model->components;
    if (d < 1 || d > 3 || m < 0 || m > VDFCG_MAX_COMPONENTS) throw InvalidArgument("bad model");
    double* w = arena<double>(ctx, VDFCG_MAX_COMPONENTS);
    double* mu = arena<double>(ctx, VDFCG_MAX_COMPONENTS * 3);
    double* cv = arena<double>(ctx, VDFCG_MAX_COMPONENTS * 9);
    copy_out(ctx, w, model->weights, m);
    copy_out(ctx, mu, model->means, size_t(m) * d);
    copy_out(ctx, cv, model->covariances, size_t(m) * d * d);
    int* mm = arena<int>(ctx, 4);
    double* ew = arena<double>(ctx, 1);
    VDFCG_CUDA(cudaMemcpyAsync(mm, &m, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    if (d == 1) throw InvalidArgument("prune_one supports d = 2 or 3");
    launch_prune_one(ctx, d, w, mu, cv, mm, threshold, mm + 1, mm + 2, ew);
    int hm[4];
    double hw;
    VDFCG_CUDA(cudaMemcpyAsync(hm, mm, sizeof(hm), cudaMemcpyDeviceToHost, ctx->stream));
    VDFCG_CUDA(cudaMemcpyAsync(&hw, ew, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    copy_out(ctx, model->weights, w, hm[0]);
    copy_out(ctx, model->means, mu, size_t(hm[0]) * d);
    copy_out(ctx, model->covariances, cv, size_t(hm[0]) * d * d);
    sync(ctx);
    model->components = hm[0];
    *pruned = hm[1];
    if (hm[1]) {
      *event_component = hm[2];
      *event_weight = hw;
    }
  });
}

int vdfcg_repair_covariance(vdfcg_ctx* ctx, const double* sigma, int32_t d, double* out,
                            int32_t* doublings) {
  return guard_impl([&] {
    begin(ctx);
    if (d < 1 || d > 3) throw InvalidArgument("repair_covariance supports d <= 3");
    auto s = stage_in(ctx, sigma, size_t(d) * d);
    double* o = arena<double>(ctx, 9);
    int* di = arena<int>(ctx, 2);
    launch_repair(ctx, d, s.dev, o, di, di + 1);
    int h[2];
    VDFCG_CUDA(cudaMemcpyAsync(h, di, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (!h[1]) throw RepairFailed("covariance repair failed after 60 doublings");
    copy_out(ctx, out, o, size_t(d) * d);
    sync(ctx);
    if (doublings) *doublings = h[0];
  });
}

int vdfcg_fit(vdfcg_ctx* ctx, const double* points, const double* weights, int64_t n, int32_t d,
              double total_weight, const vdfcg_fit_config* cfg, vdfcg_fit_result* res) {
  return guard_impl([&] {
    begin(ctx);
    if (d != 2 && d != 3) throw InvalidArgument("dimension must be 2 or 3");
    validate_config(cfg, d);
    if (!res) throw InvalidArgument("null result");
    const int K = std::max(cfg->initial_components, cfg->warm_start ? cfg->warm_start->components : 0);
    if (res->capacity_components < K) throw InvalidArgument("result capacity_components too small");
    if (res->capacity_trace < cfg->max_em_iterations)
      throw InvalidArgument("result capacity_trace too small");
    auto x = stage_in(ctx, points, size_t(n) * d);
    auto w = stage_in(ctx, weights, size_t(n));
    EmConfig e = make_em_config(ctx, cfg, d);
    EmOut o = alloc_em_out(ctx, 1, d, K, cfg->max_em_iterations, true);
    launch_em_points(ctx, d, x.dev, w.dev, n, total_weight, e, o);
    int st[4];  // status, comps, iters, conv
    VDFCG_CUDA(cudaMemcpyAsync(&st[0], o.status, 4, cudaMemcpyDeviceToHost, ctx->stream));
    VDFCG_CUDA(cudaMemcpyAsync(&st[1], o.comps, 4, cudaMemcpyDeviceToHost, ctx->stream));
    VDFCG_CUDA(cudaMemcpyAsync(&st[2], o.iters, 4, cudaMemcpyDeviceToHost, ctx->stream));
    VDFCG_CUDA(cudaMemcpyAsync(&st[3], o.conv, 4, cudaMemcpyDeviceToHost, ctx->stream));
    int ne = 0, eax = -1;
    double ev = 0.0;
    VDFCG_CUDA(cudaMemcpyAsync(&ne, o.n_events, 4, cudaMemcpyDeviceToHost, ctx->stream));
    VDFCG_CUDA(cudaMemcpyAsync(&eax, o.err_axis, 4, cudaMemcpyDeviceToHost, ctx->stream));
    VDFCG_CUDA(cudaMemcpyAsync(&ev, o.err_value, 8, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (st[0]) throw_status(st[0], eax, ev, true);
    const int M = st[1];
    copy_out(ctx, res->model.weights, o.w, M);
    copy_out(ctx, res->model.means, o.mu, size_t(M) * d);
    copy_out(ctx, res->model.covariances, o.cov, size_t(M) * d * d);
    copy_out(ctx, res->loglik_trace, o.trace, size_t(st[2]));
    copy_out(ctx, res->event_iteration, o.ev_it, size_t(ne));
    copy_out(ctx, res->event_component, o.ev_comp, size_t(ne));
    copy_out(ctx, res->event_weight, o.ev_w, size_t(ne));
    sync(ctx);
    res->model.dimension = d;
    res->model.components = M;
    res->trace_len = st[2];
    res->iterations_used = st[2];
    res->converged = st[3];
    res->n_events = ne;
  });
}

// ------------------------------------------------------------------ writer
int vdfcg_encode_model(vdfcg_ctx* ctx, const vdfcg_model* model, const vdfcg_model_meta* meta,
                       uint8_t* out, int64_t capacity, int64_t* length) {
  return guard_impl([&] {
    begin(ctx);
    if (!model || !meta || !length) throw InvalidArgument("null argument");
    const int d = model->dimension, m = model->components;
    if (d < 1) throw InvalidArgument("model dimension must be positive");
    if (m < 1) throw InvalidArgument("model has no components");
    if (d > 3) throw InvalidArgument("model dimension must be <= 3");
    auto w = stage_in(ctx, model->weights, m);
    auto mu = stage_in(ctx, model->means, size_t(m) * d);
    auto cv = stage_in(ctx, model->covariances, size_t(m) * d * d);
    int* code = arena<int>(ctx, 1);
    VDFCG_LAUNCH(ctx, "validate_model", validate_model_kernel<<<1, 32, 0, ctx->stream>>>(d, m, w.dev, cv.dev, code));
    const int c = read_scalar(ctx, code);
    if (c == 2) throw InvalidArgument("component weight must be > 0");
    if (c == 3) throw InvalidArgument("component covariance is not symmetric");
    if (c == 4) throw InvalidArgument("component weights must sum to 1");
    const bool map = model->scale && model->offset;
    const double* pw = w.dev;
    const double* pmu = mu.dev;
    const double* pcv = cv.dev;
    if (map) {
      auto sc = stage_in(ctx, model->scale, d);
      auto of = stage_in(ctx, model->offset, d);
      double* ow = arena<double>(ctx, m);
      double* omu = arena<double>(ctx, size_t(m) * d);
      double* ocv = arena<double>(ctx, size_t(m) * d * d);
      launch_canonicalize(ctx, d, m, w.dev, mu.dev, cv.dev, sc.dev, of.dev, ow, omu, ocv);
      pw = ow;
      pmu = omu;
      pcv = ocv;
    }
    PackMeta pm = make_pack_meta(ctx, meta, d);
    int32_t* comps = arena<int32_t>(ctx, 1);
    VDFCG_CUDA(cudaMemcpyAsync(comps, &m, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    PackIn in{1, m, nullptr, comps, pw, pmu, pcv};
    int64_t* offs = arena<int64_t>(ctx, 2);
    const int64_t total = launch_pack_offsets(ctx, in, pm, offs);
    if (total > capacity) throw InvalidArgument("encode_model: capacity too small");
    uint8_t* buf = arena<uint8_t>(ctx, total);
    launch_pack(ctx, in, pm, offs, buf);
    copy_out(ctx, out, buf, size_t(total));
    sync(ctx);
    *length = total;
  });
}

// ------------------------------------------------------------------ cells
static CellBinsDev bins_dev(vdfcg_ctx* ctx, const CellsDev& c, vdfcg_cell_bins* out,
                            std::vector<std::function<void()>>& fin) {
  CellBinsDev b{};
  const size_t nc = c.n_cells, n = size_t(c.n);
  if (out && out->nnz) {
    auto s1 = stage_out(ctx, out->nnz, nc);
    auto s2 = stage_out(ctx, out->keys, n);
    auto s3 = stage_out(ctx, out->counts, n);
    auto s4 = stage_out(ctx, out->out_of_range, nc);
    auto s5 = stage_out(ctx, out->in_range, nc);
    b = {s1.dev, s2.dev, s3.dev, s4.dev, s5.dev};
    fin.push_back([=] {
      finish(ctx, s1);
      finish(ctx, s2);
      finish(ctx, s3);
      finish(ctx, s4);
      finish(ctx, s5);
    });
  } else {
    b = {arena<int32_t>(ctx, nc), arena<uint32_t>(ctx, n), arena<double>(ctx, n),
         arena<double>(ctx, nc), arena<double>(ctx, nc)};
  }
  return b;
}

static EmOut results_dev(vdfcg_ctx* ctx, int n_cells, int d, vdfcg_cell_results* r,
                         std::vector<std::function<void()>>& fin) {
  if (!r) throw InvalidArgument("null cell results");
  const int K = r->capacity_components;
  const size_t nc = n_cells;
  EmOut o{};
  o.K = K;
  o.trace_cap = r->loglik_trace ? r->capacity_trace : 0;
  auto st = stage_out(ctx, r->status, nc);
  auto cm = stage_out(ctx, r->components, nc);
  auto it = stage_out(ctx, r->iterations, nc);
  auto cv = stage_out(ctx, r->converged, nc);
  auto w = stage_out(ctx, r->weights, nc * K);
  auto mu = stage_out(ctx, r->means, nc * K * d);
  auto co = stage_out(ctx, r->covariances, nc * K * d * d);
  auto fl = stage_out(ctx, r->final_loglik, nc);
  auto tr = stage_out(ctx, r->loglik_trace, o.trace_cap ? nc * o.trace_cap : 0);
  auto ne = stage_out(ctx, r->n_events, r->n_events ? nc : 0);
  auto ei = stage_out(ctx, r->event_iteration, r->event_iteration ? nc * K : 0);
  auto ec = stage_out(ctx, r->event_component, r->event_component ? nc * K : 0);
  auto ew = stage_out(ctx, r->event_weight, r->event_weight ? nc * K : 0);
  if (!st.dev || !cm.dev || !it.dev || !cv.dev || !w.dev || !mu.dev || !co.dev || !fl.dev)
    throw InvalidArgument("cell results: status/components/iterations/converged/weights/means/"
                          "covariances/final_loglik are required");
  o.status = st.dev;
  o.comps = cm.dev;
  o.iters = it.dev;
  o.conv = cv.dev;
  o.w = w.dev;
  o.mu = mu.dev;
  o.cov = co.dev;
  o.final_ll = fl.dev;
  o.trace = tr.dev;
  const bool ev = ne.dev && ei.dev && ec.dev && ew.dev;
  o.n_events = ev ? ne.dev : nullptr;
  o.ev_it = ev ? ei.dev : nullptr;
  o.ev_comp = ev ? ec.dev : nullptr;
  o.ev_w = ev ? ew.dev : nullptr;
  o.err_axis = nullptr;
  o.err_value = nullptr;
  fin.push_back([=] {
    finish(ctx, st);
    finish(ctx, cm);
    finish(ctx, it);
    finish(ctx, cv);
    finish(ctx, w);
    finish(ctx, mu);
    finish(ctx, co);
    finish(ctx, fl);
    finish(ctx, tr);
    finish(ctx, ne);
    finish(ctx, ei);
    finish(ctx, ec);
    finish(ctx, ew);
  });
  return o;
}

static bool any_host(const std::vector<std::function<void()>>& fin) { return !fin.empty(); }

static void fit_cells_dev(vdfcg_ctx* ctx, const CellsDev& c, const CellBinsDev& b,
                          const vdfcg_fit_config* cfg, const EmOut& o,
                          const vdfcg_cell_results* warm = nullptr,
                          uint32_t* packed_scratch = nullptr, const EmConfig* prebuilt = nullptr) {
  const int kw = warm ? warm->capacity_components : 0;
  if (warm && (kw < 1 || kw > VDFCG_MAX_COMPONENTS))
    throw InvalidArgument("warm cell results must have capacity_components in 1..16");
  if (o.K < std::max({cfg->initial_components, cfg->warm_start ? cfg->warm_start->components : 0, kw}))
    throw InvalidArgument("cell results capacity_components too small");
  if (o.trace_cap && o.trace_cap < cfg->max_em_iterations)
    throw InvalidArgument("cell results capacity_trace too small");
  EmConfig e = prebuilt ? *prebuilt : make_em_config(ctx, cfg, c.d);
  if (warm) {  // per-cell warm start from a previous (device or host) results buffer
    const size_t nc = c.n_cells;
    const int32_t* st = warm->status ? stage_in(ctx, warm->status, nc).dev : nullptr;
    if (!warm->components || !warm->weights || !warm->means || !warm->covariances)
      throw InvalidArgument("warm cell results need components, weights, means, covariances");
    const int32_t* cm = stage_in(ctx, warm->components, nc).dev;
    int32_t* wm = arena<int32_t>(ctx, nc);
    launch_warm_m(ctx, c.n_cells, st, cm, wm);
    e.cell_warm_m = wm;
    e.cell_warm_K = kw;
    e.cell_warm_w = stage_in(ctx, warm->weights, nc * kw).dev;
    e.cell_warm_mu = stage_in(ctx, warm->means, nc * kw * c.d).dev;
    e.cell_warm_cov = stage_in(ctx, warm->covariances, nc * kw * c.d * c.d).dev;
  }
  KeyCells kc{};
  kc.n_cells = c.n_cells;
  kc.offsets = c.offsets;
  kc.nnz = b.nnz;
  kc.keys = b.keys;
  kc.counts = b.counts;
  kc.in_range = b.in_range;
  // decoded-bin scratch, indexed by absolute particle offsets (full batch)
  kc.packed = packed_scratch ? packed_scratch : arena<uint32_t>(ctx, size_t(std::max<int64_t>(c.n, 1)));
  kc.n_bins = c.n_bins;
  for (int a = 0; a < 3; ++a) {
    kc.lo[a] = c.lo[a];
    kc.hi[a] = c.hi[a];
  }
  const double avg = c.shape_cells > 0 ? c.shape_avg : c.n_cells ? double(c.n) / c.n_cells : 0.0;
  launch_em_cells(ctx, c.d, kc, e, o, avg, c.shape_cells);
}

int vdfcg_bin_cells(vdfcg_ctx* ctx, const vdfcg_cells* cells, vdfcg_cell_bins* out) {
  return guard_impl([&] {
    begin(ctx);
    CellsDev c = stage_cells(ctx, cells);
    if (!out) throw InvalidArgument("null output");
    std::vector<std::function<void()>> fin;
    CellBinsDev b = bins_dev(ctx, c, out, fin);
    launch_bin_cells(ctx, c, b);
    for (auto& f : fin) f();
    sync(ctx);
  });
}

int vdfcg_fit_cells(vdfcg_ctx* ctx, const vdfcg_cells* cells, const vdfcg_cell_bins* bins,
                    const vdfcg_fit_config* cfg, vdfcg_cell_results* out) {
  return vdfcg_fit_cells_warm(ctx, cells, bins, cfg, nullptr, out);
}

int vdfcg_fit_cells_warm(vdfcg_ctx* ctx, const vdfcg_cells* cells, const vdfcg_cell_bins* bins,
                         const vdfcg_fit_config* cfg, const vdfcg_cell_results* warm,
                         vdfcg_cell_results* out) {
  return guard_impl([&] {
    begin(ctx);
    if (!cells || !bins) throw InvalidArgument("null argument");
    validate_config(cfg, cells->dimension);
    vdfcg_cells geom = *cells;
    geom.weights = nullptr;
    for (int a = 0; a < 3; ++a) geom.velocity[a] = nullptr;
    if (geom.n_particles == 0) geom.velocity[0] = nullptr;
    // geometry only: velocities are not read by the fitter
    CellsDev c{};
    c.d = cells->dimension;
    if (c.d != 2 && c.d != 3) throw InvalidArgument("particle dimension must be 2 or 3");
    c.n = cells->n_particles;
    c.n_cells = cells->n_cells;
    c.offsets = stage_in(ctx, cells->cell_offsets, size_t(c.n_cells) + 1).dev;
    c.n_bins = cells->n_bins;
    for (int a = 0; a < 3; ++a) {
      c.lo[a] = cells->lo[a];
      c.hi[a] = cells->hi[a];
    }
    CellBinsDev b{};
    b.nnz = stage_in(ctx, bins->nnz, c.n_cells).dev;
    b.keys = stage_in(ctx, bins->keys, size_t(c.n)).dev;
    b.counts = stage_in(ctx, bins->counts, size_t(c.n)).dev;
    b.in_range = stage_in(ctx, bins->in_range, c.n_cells).dev;
    std::vector<std::function<void()>> fin;
    EmOut o = results_dev(ctx, c.n_cells, c.d, out, fin);
    fit_cells_dev(ctx, c, b, cfg, o, warm);
    for (auto& f : fin) f();
    if (any_host(fin)) sync(ctx);
  });
}

static PackIn pack_in_from(vdfcg_ctx* ctx, int n_cells, int d, const vdfcg_cell_results* r) {
  const int K = r->capacity_components;
  const size_t nc = n_cells;
  PackIn in{};
  in.n_cells = n_cells;
  in.K = K;
  in.status = stage_in(ctx, r->status, nc).dev;
  in.comps = stage_in(ctx, r->components, nc).dev;
  in.w = stage_in(ctx, r->weights, nc * K).dev;
  in.mu = stage_in(ctx, r->means, nc * K * d).dev;
  in.cov = stage_in(ctx, r->covariances, nc * K * d * d).dev;
  return in;
}

int vdfcg_pack_cells(vdfcg_ctx* ctx, int32_t n_cells, int32_t d, const vdfcg_cell_results* res,
                     const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                     int64_t* record_offsets) {
  return guard_impl([&] {
    begin(ctx);
    if (!res || !record_offsets) throw InvalidArgument("null argument");
    if (d != 2 && d != 3) throw InvalidArgument("dimension must be 2 or 3");
    PackIn in = pack_in_from(ctx, n_cells, d, res);
    PackMeta pm = make_pack_meta(ctx, meta, d);
    auto offs = stage_out(ctx, record_offsets, size_t(n_cells) + 1);
    const int64_t total = launch_pack_offsets(ctx, in, pm, offs.dev);
    if (total > capacity) throw InvalidArgument("pack_cells: capacity too small");
    auto rec = stage_out(ctx, records, size_t(total));
    if (total) launch_pack(ctx, in, pm, offs.dev, rec.dev);
    finish(ctx, offs);
    finish(ctx, rec);
    sync(ctx);
  });
}

int vdfcg_compress_cells(vdfcg_ctx* ctx, const vdfcg_cells* cells, const vdfcg_fit_config* cfg,
                         vdfcg_cell_bins* bins, vdfcg_cell_results* out,
                         const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                         int64_t* record_offsets) {
  return vdfcg_compress_cells_warm(ctx, cells, cfg, nullptr, bins, out, meta, records, capacity,
                                   record_offsets);
}

// Sub-batch views of cells [c0, c1): the kernels index particles through cell_offsets,
// so only the per-cell arrays are offset.
static CellsDev sub_cells(const CellsDev& c, int c0, int c1) {
  CellsDev s = c;
  s.offsets = c.offsets + c0;
  s.n_cells = c1 - c0;
  return s;
}
static CellBinsDev sub_bins(const CellBinsDev& b, int c0) {
  CellBinsDev s = b;
  s.nnz += c0;
  s.oor += c0;
  s.in_range += c0;
  return s;
}
static EmOut sub_out(const EmOut& o, int c0, int d) {
  EmOut s = o;
  const int64_t K = o.K;
  s.status += c0;
  s.comps += c0;
  s.iters += c0;
  s.conv += c0;
  s.final_ll += c0;
  s.w += c0 * K;
  s.mu += c0 * K * d;
  s.cov += c0 * K * d * d;
  if (s.trace) s.trace += int64_t(c0) * o.trace_cap;
  if (s.n_events) {
    s.n_events += c0;
    s.ev_it += c0 * K;
    s.ev_comp += c0 * K;
    s.ev_w += c0 * K;
  }
  return s;
}
static vdfcg_cell_results sub_warm(const vdfcg_cell_results& w, int c0, int d) {
  vdfcg_cell_results s = w;
  const int64_t K = w.capacity_components;
  if (s.status) s.status += c0;
  s.components += c0;
  s.weights += c0 * K;
  s.means += c0 * K * d;
  s.covariances += c0 * K * d * d;
  return s;
}

static void pack_into(vdfcg_ctx* ctx, const CellsDev& c, const EmOut& o,
                      const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                      int64_t* record_offsets, std::vector<std::function<void()>>& fin) {
  if (!records && !record_offsets) return;
  if (!meta || !record_offsets) throw InvalidArgument("packing needs meta and record_offsets");
  PackIn in{c.n_cells, o.K, o.status, o.comps, o.w, o.mu, o.cov};
  PackMeta pm = make_pack_meta(ctx, meta, c.d);
  auto offs = stage_out(ctx, record_offsets, size_t(c.n_cells) + 1);
  const int64_t total = launch_pack_offsets(ctx, in, pm, offs.dev);
  if (total > capacity) throw InvalidArgument("compress_cells: record capacity too small");
  auto rec = stage_out(ctx, records, size_t(total));
  if (total) launch_pack(ctx, in, pm, offs.dev, rec.dev);
  fin.push_back([=] {
    finish(ctx, offs);
    finish(ctx, rec);
  });
}

// Events owned for the duration of one call (destroyed on every exit path).
struct EventPool {
  std::vector<cudaEvent_t> ev;
  cudaEvent_t make() {
    cudaEvent_t e;
    VDFCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev.push_back(e);
    return e;
  }
  ~EventPool() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

// On an exception, drain the side streams before the arena can be reused by the next call
// (their copies / kernels may still target this call's buffers).
struct SideStreamGuard {
  vdfcg_ctx* ctx;
  int pending = std::uncaught_exceptions();
  ~SideStreamGuard() {
    if (std::uncaught_exceptions() > pending) {
      cudaStreamSynchronize(ctx->copy_stream);
      cudaStreamSynchronize(ctx->aux_stream);
    }
  }
};

// Pageable host inputs (a plain numpy array / Eigen matrix): cudaMemcpyAsync from pageable
// memory blocks the calling thread, so every chunk's copy would finish before any compute is
// enqueued. Instead host threads copy pieces of each chunk into a ring of pinned slots and
// issue the H2D from there (truly asynchronous); a slot is reused once its previous H2D has
// completed. The main thread records chunk j's ready event as soon as all of chunk j's
// pieces are issued and enqueues its compute, so copy and compute overlap as for pinned input.
class PageableStager {
 public:
  struct Piece {
    const char* src;
    char* dst;
    size_t bytes;
    int chunk;
  };
  PageableStager(vdfcg_ctx* ctx, std::vector<Piece> pieces, int n_chunks)
      : ctx_(ctx), pieces_(std::move(pieces)), issued_(pieces_.size()), left_(n_chunks, 0) {
    constexpr size_t kSlot = size_t(64) << 20;
    constexpr int kSlots = 12;
    if (!ctx->ring) {
      VDFCG_CUDA(cudaHostAlloc(&ctx->ring, kSlot * kSlots, cudaHostAllocDefault));
      ctx->ring_slot = kSlot;
      ctx->ring_slots = kSlots;
      ctx->ring_ev.resize(kSlots);
      for (auto& e : ctx->ring_ev) VDFCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (auto& f : issued_) f.store(false);
    for (const auto& p : pieces_) ++left_[p.chunk];
    const int threads = std::min<int>(6, std::max<int>(1, static_cast<int>(pieces_.size())));
    for (int t = 0; t < threads; ++t) th_.emplace_back([this] { run(); });
  }
  ~PageableStager() {
    for (auto& t : th_) t.join();
  }
  // Blocks until every piece of chunk j has been issued on the copy stream.
  void wait_chunk(int j) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return left_[j] == 0 || failed_; });
    if (failed_) throw CudaError(err_);
  }
  static size_t slot_bytes() { return size_t(64) << 20; }

 private:
  void run() {
    cudaSetDevice(ctx_->device);
    for (;;) {
      const size_t i = next_.fetch_add(1);
      if (i >= pieces_.size() || failed_) return;
      const int slots = ctx_->ring_slots;
      const int slot = static_cast<int>(i % slots);
      // the slot's previous piece must have been issued (its event recorded) and copied
      if (i >= size_t(slots)) {
        while (!issued_[i - slots].load(std::memory_order_acquire)) {
          if (failed_) return;
          std::this_thread::yield();
        }
        if (cudaEventSynchronize(ctx_->ring_ev[slot]) != cudaSuccess) return fail("staging H2D failed");
      }
      char* buf = static_cast<char*>(ctx_->ring) + size_t(slot) * ctx_->ring_slot;
      const Piece& p = pieces_[i];
      std::memcpy(buf, p.src, p.bytes);
      {
        // one issuer at a time: the H2D and its slot event go onto the copy stream in order
        std::lock_guard<std::mutex> lk(issue_mu_);
        if (cudaMemcpyAsync(p.dst, buf, p.bytes, cudaMemcpyHostToDevice, ctx_->copy_stream) != cudaSuccess ||
            cudaEventRecord(ctx_->ring_ev[slot], ctx_->copy_stream) != cudaSuccess)
          return fail("staging H2D failed");
      }
      issued_[i].store(true, std::memory_order_release);
      {
        std::lock_guard<std::mutex> lk(mu_);
        --left_[p.chunk];
      }
      cv_.notify_all();
    }
  }
  void fail(const char* msg) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      failed_ = true;
      err_ = msg;
    }
    cv_.notify_all();
  }
  vdfcg_ctx* ctx_;
  std::vector<Piece> pieces_;
  std::vector<std::atomic<bool>> issued_;
  std::vector<int> left_;
  std::atomic<size_t> next_{0};
  std::mutex mu_, issue_mu_;
  std::condition_variable cv_;
  std::atomic<bool> failed_{false};
  std::string err_;
  std::vector<std::thread> th_;
};

static bool pageable_host(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// Host-resident particles: the velocity (and weight) ranges of successive cell chunks are
// copied on the context's copy stream while the compute stream bins and fits the chunks
// already resident, so the end-to-end time approaches max(H2D, compute) instead of the sum.
static bool compress_pipelined(vdfcg_ctx* ctx, const vdfcg_cells* cells,
                               const vdfcg_fit_config* cfg, const vdfcg_cell_results* warm,
                               vdfcg_cell_bins* bins, vdfcg_cell_results* out,
                               const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                               int64_t* record_offsets, const EmShape& shape) {
  const int d = cells->dimension;
  if (d != 2 && d != 3) return false;
  if (cells->n_particles < (int64_t(1) << 22) || cells->n_cells < 4) return false;
  for (int a = 0; a < d; ++a)
    if (!cells->velocity[a] || is_device_pointer(cells->velocity[a])) return false;
  if (is_device_pointer(cells->cell_offsets)) return false;
  if (cells->weights && is_device_pointer(cells->weights)) return false;
  // malformed offsets take the staged path, whose device checks raise the usual error
  const int64_t* ho = cells->cell_offsets;
  if (!ho || ho[0] < 0 || ho[cells->n_cells] > cells->n_particles) return false;
  for (int q = 0; q < cells->n_cells; ++q)
    if (ho[q + 1] < ho[q]) return false;
  // validation identical to stage_cells, without the bulk copies
  if (cells->n_bins < 2) throw InvalidArgument("n_bins must be >= 2");
  double nbd = 1.0;
  for (int a = 0; a < d; ++a) nbd *= cells->n_bins;
  if (nbd > 2147483647.0) throw InvalidArgument("n_bins^d must fit a 31-bit bin key");
  if (d == 3 && cells->n_bins > 1024) throw InvalidArgument("3V cells support n_bins <= 1024");
  for (int a = 0; a < d; ++a)
    if (!range_ok(cells->lo[a], cells->hi[a]))
      throw InvalidArgument("axis range must satisfy min < max");
  const int64_t n = cells->n_particles;
  const int nc = cells->n_cells;
  const int64_t* hoff = cells->cell_offsets;
  CellsDev c{};
  c.d = d;
  c.n = n;
  c.n_cells = nc;
  c.n_bins = cells->n_bins;
  for (int a = 0; a < 3; ++a) {
    c.lo[a] = cells->lo[a];
    c.hi[a] = cells->hi[a];
  }
  c.offsets = stage_in(ctx, hoff, size_t(nc) + 1).dev;
  double* dv[3] = {nullptr, nullptr, nullptr};
  for (int a = 0; a < d; ++a) dv[a] = arena<double>(ctx, size_t(n));
  double* dw = cells->weights ? arena<double>(ctx, size_t(n)) : nullptr;
  for (int a = 0; a < 3; ++a) c.vel[a] = a < d ? dv[a] : dv[0];
  c.w = dw;
  // whole-cell chunks growing geometrically (x2): the first is 1/(2^n - 1) of the
  // particles, so compute starts after a small copy, and every later copy (55 GB/s) is done
  // before the previous chunk's compute (~22 GB/s of input consumed) ends
  static const int pipe_chunks = [] {
    const char* e = getenv("VDFCG_PIPE_CHUNKS");
    return e ? std::min(20, std::max(2, atoi(e))) : 8;
  }();
  const int nch = std::min(pipe_chunks, nc);
  std::vector<int> bounds{0};
  for (int j = 1; j < nch; ++j) {
    const double f = double((1ll << j) - 1) / double((1ll << nch) - 1);
    const int64_t target = hoff[0] + static_cast<int64_t>(double(hoff[nc] - hoff[0]) * f);
    const int cb = static_cast<int>(std::upper_bound(hoff, hoff + nc + 1, target) - hoff) - 1;
    bounds.push_back(std::max(bounds.back(), std::min(cb, nc)));
  }
  bounds.push_back(nc);
  validate_config(cfg, d);
  // the copy stream starts after everything already queued on the compute stream
  EventPool events;
  SideStreamGuard side{ctx};
  cudaEvent_t start = events.make();
  VDFCG_CUDA(cudaEventRecord(start, ctx->stream));
  VDFCG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, start, 0));
  std::vector<cudaEvent_t> ready(bounds.size() - 1);
  for (auto& e : ready) e = events.make();
  bool pageable = cells->weights && pageable_host(cells->weights);
  for (int a = 0; a < d; ++a) pageable = pageable || pageable_host(cells->velocity[a]);
  std::unique_ptr<PageableStager> stager;
  if (pageable) {
    std::vector<PageableStager::Piece> pieces;
    const size_t slot = PageableStager::slot_bytes();
    for (size_t j = 0; j + 1 < bounds.size(); ++j) {
      const int64_t p0 = hoff[bounds[j]], p1 = hoff[bounds[j + 1]];
      const size_t bytes = size_t(p1 - p0) * sizeof(double);
      for (int a = 0; a <= d; ++a) {
        const double* src = a < d ? cells->velocity[a] : cells->weights;
        double* dst = a < d ? dv[a] : dw;
        if (!src) continue;
        for (size_t o = 0; o < bytes; o += slot)
          pieces.push_back({reinterpret_cast<const char*>(src + p0) + o, reinterpret_cast<char*>(dst + p0) + o,
                            std::min(slot, bytes - o), static_cast<int>(j)});
      }
    }
    stager = std::make_unique<PageableStager>(ctx, std::move(pieces), static_cast<int>(ready.size()));
  } else {
    for (size_t j = 0; j + 1 < bounds.size(); ++j) {
      const int64_t p0 = hoff[bounds[j]], p1 = hoff[bounds[j + 1]];
      const size_t bytes = size_t(p1 - p0) * sizeof(double);
      if (bytes) {
        for (int a = 0; a < d; ++a)
          VDFCG_CUDA(cudaMemcpyAsync(dv[a] + p0, cells->velocity[a] + p0, bytes,
                                     cudaMemcpyHostToDevice, ctx->copy_stream));
        if (dw)
          VDFCG_CUDA(cudaMemcpyAsync(dw + p0, cells->weights + p0, bytes, cudaMemcpyHostToDevice,
                                     ctx->copy_stream));
      }
      VDFCG_CUDA(cudaEventRecord(ready[j], ctx->copy_stream));
    }
  }
  std::vector<std::function<void()>> fin;
  CellBinsDev b = bins_dev(ctx, c, bins, fin);
  EmOut o = results_dev(ctx, nc, d, out, fin);
  uint32_t* packed = arena<uint32_t>(ctx, size_t(n));
  const EmConfig em = make_em_config(ctx, cfg, d);  // mt19937_64 uniforms once per call
  // Chunks alternate between the context stream and the aux stream so one chunk's fits
  // start while the previous chunk's last fits drain. Every fit is independent, so the
  // results do not depend on the interleaving.
  cudaStream_t main = ctx->stream;
  cudaEvent_t fork = events.make(), join = events.make();
  VDFCG_CUDA(cudaEventRecord(fork, main));
  VDFCG_CUDA(cudaStreamWaitEvent(ctx->aux_stream, fork, 0));
  try {
    for (size_t j = 0; j + 1 < bounds.size(); ++j) {
      const int c0 = bounds[j], c1 = bounds[j + 1];
      if (c1 <= c0) continue;
      ctx->stream = (j & 1) ? ctx->aux_stream : main;
      if (stager) {  // pageable input: chunk j's pieces issued -> its ready event
        stager->wait_chunk(static_cast<int>(j));
        VDFCG_CUDA(cudaEventRecord(ready[j], ctx->copy_stream));
      }
      VDFCG_CUDA(cudaStreamWaitEvent(ctx->stream, ready[j], 0));
      CellsDev sc = sub_cells(c, c0, c1);
      sc.n = hoff[c1] - hoff[c0];  // this chunk's particles (histogram launch shapes)
      sc.max_cell = 0;             // known on the host: no device round trip per chunk
      for (int q = c0; q < c1; ++q) sc.max_cell = std::max(sc.max_cell, hoff[q + 1] - hoff[q]);
      // EM launch shape of the whole batch (bitwise-identical results)
      sc.shape_cells = shape.cells > 0 ? shape.cells : nc;
      sc.shape_avg = shape.cells > 0 ? shape.avg : double(hoff[nc] - hoff[0]) / nc;
      launch_bin_cells(ctx, sc, sub_bins(b, c0));
      vdfcg_cell_results sw{};
      if (warm) sw = sub_warm(*warm, c0, d);
      fit_cells_dev(ctx, sc, sub_bins(b, c0), cfg, sub_out(o, c0, d), warm ? &sw : nullptr, packed,
                    &em);
    }
  } catch (...) {
    ctx->stream = main;
    throw;
  }
  ctx->stream = main;
  VDFCG_CUDA(cudaEventRecord(join, ctx->aux_stream));
  VDFCG_CUDA(cudaStreamWaitEvent(main, join, 0));
  pack_into(ctx, c, o, meta, records, capacity, record_offsets, fin);
  for (auto& f : fin) f();
  sync(ctx);
  return true;
}

}  // extern "C"

namespace vdfcg {
int compress_cells_shaped(vdfcg_ctx* ctx, const vdfcg_cells* cells, const vdfcg_fit_config* cfg,
                          const vdfcg_cell_results* warm, vdfcg_cell_bins* bins,
                          vdfcg_cell_results* out, const vdfcg_model_meta* meta, uint8_t* records,
                          int64_t capacity, int64_t* record_offsets, const EmShape& shape) {
  return guard_impl([&] {
    begin(ctx);
    if (!cells) throw InvalidArgument("null cells");
    if (compress_pipelined(ctx, cells, cfg, warm, bins, out, meta, records, capacity,
                           record_offsets, shape))
      return;
    CellsDev c = stage_cells(ctx, cells);
    c.shape_cells = shape.cells;
    c.shape_avg = shape.avg;
    validate_config(cfg, c.d);
    std::vector<std::function<void()>> fin;
    CellBinsDev b = bins_dev(ctx, c, bins, fin);
    EmOut o = results_dev(ctx, c.n_cells, c.d, out, fin);
    launch_bin_cells(ctx, c, b);
    fit_cells_dev(ctx, c, b, cfg, o, warm);
    pack_into(ctx, c, o, meta, records, capacity, record_offsets, fin);
    for (auto& f : fin) f();
    if (any_host(fin)) sync(ctx);
  });
}
}  // namespace vdfcg

extern "C" {

int vdfcg_compress_cells_warm(vdfcg_ctx* ctx, const vdfcg_cells* cells,
                              const vdfcg_fit_config* cfg, const vdfcg_cell_results* warm,
                              vdfcg_cell_bins* bins, vdfcg_cell_results* out,
                              const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                              int64_t* record_offsets) {
  return compress_cells_shaped(ctx, cells, cfg, warm, bins, out, meta, records, capacity,
                               record_offsets, EmShape{});
}

// ---- per-particle cell-index input (index.cu) ---------------------------------------
// Validation as stage_cells, plus the cell ids; returns the staged device view.
static IndexedDev stage_particles(vdfcg_ctx* ctx, const vdfcg_particles* p) {
  if (!p) throw InvalidArgument("null particles");
  const int d = p->dimension;
  if (d != 2 && d != 3) throw InvalidArgument("particle dimension must be 2 or 3");
  if (p->n_bins < 2) throw InvalidArgument("n_bins must be >= 2");
  double nbd = 1.0;
  for (int a = 0; a < d; ++a) nbd *= p->n_bins;
  if (nbd > 2147483647.0) throw InvalidArgument("n_bins^d must fit a 31-bit bin key");
  for (int a = 0; a < d; ++a)
    if (!range_ok(p->lo[a], p->hi[a])) throw InvalidArgument("axis range must satisfy min < max");
  if (p->n_cells < 1 || p->n_particles < 0) throw InvalidArgument("negative sizes");
  if (p->n_particles >= (int64_t(1) << 32)) throw InvalidArgument("cell-index input supports < 2^32 particles per call");
  if (p->n_particles && !p->cell) throw InvalidArgument("cell index array is required");
  IndexedDev in{};
  in.d = d;
  in.n = p->n_particles;
  for (int a = 0; a < d; ++a) {
    if (!p->velocity[a] && in.n) throw InvalidArgument("missing velocity axis");
    in.vel[a] = stage_in(ctx, p->velocity[a], size_t(in.n)).dev;
  }
  for (int a = d; a < 3; ++a) in.vel[a] = in.vel[0];
  in.w = p->weights ? stage_in(ctx, p->weights, size_t(in.n)).dev : nullptr;
  in.cell = stage_in(ctx, p->cell, size_t(in.n)).dev;
  in.n_cells = p->n_cells;
  in.n_bins = p->n_bins;
  for (int a = 0; a < 3; ++a) {
    in.lo[a] = p->lo[a];
    in.hi[a] = p->hi[a];
  }
  return in;
}

// Group by cell, then the CellsDev view of the grouped keys (velocities are not needed
// past the grouping: the bin key was computed while they were read).
static CellsDev group_particles(vdfcg_ctx* ctx, const IndexedDev& in, int64_t* offsets_dev, int* err) {
  GroupedDev g{arena<uint32_t>(ctx, size_t(std::max<int64_t>(in.n, 1))),
               in.w ? arena<double>(ctx, size_t(std::max<int64_t>(in.n, 1))) : nullptr, offsets_dev};
  launch_group_cells(ctx, in, g, err);
  CellsDev c{};
  c.d = in.d;
  c.n = in.n;
  for (int a = 0; a < 3; ++a) c.vel[a] = nullptr;
  c.w = g.w;
  c.n_cells = in.n_cells;
  c.offsets = offsets_dev;
  c.n_bins = in.n_bins;
  for (int a = 0; a < 3; ++a) {
    c.lo[a] = in.lo[a];
    c.hi[a] = in.hi[a];
  }
  c.keys = g.keys;
  return c;
}

static void check_group_error(vdfcg_ctx* ctx, const int* err) {
  const int e = read_scalar(ctx, err);
  if (e & 1) throw InvalidArgument("cell index out of range");
  if (e & 2) throw InvalidArgument("particle weights must all be > 0");
}

int vdfcg_bin_cells_indexed(vdfcg_ctx* ctx, const vdfcg_particles* particles, int64_t* cell_offsets,
                            vdfcg_cell_bins* out) {
  return guard_impl([&] {
    begin(ctx);
    IndexedDev in = stage_particles(ctx, particles);
    if (!out || !cell_offsets) throw InvalidArgument("null output");
    int* err = arena<int>(ctx, 1);
    VDFCG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
    auto offs = stage_out(ctx, cell_offsets, size_t(in.n_cells) + 1);
    CellsDev c = group_particles(ctx, in, offs.dev, err);
    check_group_error(ctx, err);
    std::vector<std::function<void()>> fin;
    CellBinsDev b = bins_dev(ctx, c, out, fin);
    launch_bin_cells(ctx, c, b);
    finish(ctx, offs);
    for (auto& f : fin) f();
    sync(ctx);
  });
}

int vdfcg_compress_cells_indexed(vdfcg_ctx* ctx, const vdfcg_particles* particles,
                                 const vdfcg_fit_config* cfg, int64_t* cell_offsets,
                                 vdfcg_cell_bins* bins, vdfcg_cell_results* out,
                                 const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                                 int64_t* record_offsets) {
  return vdfcg_compress_cells_indexed_warm(ctx, particles, cfg, nullptr, cell_offsets, bins, out, meta,
                                           records, capacity, record_offsets);
}

int vdfcg_compress_cells_indexed_warm(vdfcg_ctx* ctx, const vdfcg_particles* particles,
                                      const vdfcg_fit_config* cfg, const vdfcg_cell_results* warm,
                                      int64_t* cell_offsets, vdfcg_cell_bins* bins,
                                      vdfcg_cell_results* out, const vdfcg_model_meta* meta,
                                      uint8_t* records, int64_t capacity, int64_t* record_offsets) {
  return guard_impl([&] {
    begin(ctx);
    IndexedDev in = stage_particles(ctx, particles);
    validate_config(cfg, in.d);
    int* err = arena<int>(ctx, 1);
    VDFCG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
    auto offs = stage_out(ctx, cell_offsets, cell_offsets ? size_t(in.n_cells) + 1 : 0);
    int64_t* offs_dev = offs.dev ? offs.dev : arena<int64_t>(ctx, size_t(in.n_cells) + 1);
    CellsDev c = group_particles(ctx, in, offs_dev, err);
    check_group_error(ctx, err);
    std::vector<std::function<void()>> fin;
    CellBinsDev b = bins_dev(ctx, c, bins, fin);
    EmOut o = results_dev(ctx, c.n_cells, c.d, out, fin);
    launch_bin_cells(ctx, c, b);
    fit_cells_dev(ctx, c, b, cfg, o, warm);
    pack_into(ctx, c, o, meta, records, capacity, record_offsets, fin);
    finish(ctx, offs);
    for (auto& f : fin) f();
    sync(ctx);
  });
}

// ---- fit quality --------------------------------------------
// GmmModel::validate (wgmm.cpp:46-63) on the device, then the staged model.
static ModelDev staged_valid_model(vdfcg_ctx* ctx, const vdfcg_model* model) {
  if (!model) throw InvalidArgument("null model");
  const int d = model->dimension, m = model->components;
  if (d < 1) throw InvalidArgument("model dimension must be positive");
  if (m < 1) throw InvalidArgument("model has no components");
  if (d > 3) throw InvalidArgument("model dimension must be <= 3");
  if (m > VDFCG_MAX_COMPONENTS) throw InvalidArgument("model has more than 16 components");
  auto w = stage_in(ctx, model->weights, m);
  auto mu = stage_in(ctx, model->means, size_t(m) * d);
  auto cv = stage_in(ctx, model->covariances, size_t(m) * d * d);
  int* code = arena<int>(ctx, 1);
  VDFCG_LAUNCH(ctx, "validate_model", validate_model_kernel<<<1, 32, 0, ctx->stream>>>(d, m, w.dev, cv.dev, code));
  const int c = read_scalar(ctx, code);
  if (c == 2) throw InvalidArgument("component weight must be > 0");
  if (c == 3) throw InvalidArgument("component covariance is not symmetric");
  if (c == 4) throw InvalidArgument("component weights must sum to 1");
  ModelDev md{d, m, w.dev, mu.dev, cv.dev, nullptr, nullptr};
  if (model->scale && model->offset) {
    md.scale = stage_in(ctx, model->scale, d).dev;
    md.offset = stage_in(ctx, model->offset, d).dev;
  }
  return md;
}

int vdfcg_metrics_cells(vdfcg_ctx* ctx, const vdfcg_cells* cells, const vdfcg_cell_bins* bins,
                        const vdfcg_cell_results* res, vdfcg_cell_metrics* out) {
  return guard_impl([&] {
    begin(ctx);
    if (!cells || !bins || !res || !out) throw InvalidArgument("null argument");
    const int d = cells->dimension;
    if (d != 2 && d != 3) throw InvalidArgument("particle dimension must be 2 or 3");
    if (cells->n_bins < 2) throw InvalidArgument("n_bins must be >= 2");
    for (int a = 0; a < d; ++a)
      if (!range_ok(cells->lo[a], cells->hi[a])) throw InvalidArgument("axis range must satisfy min < max");
    if (cells->n_cells < 0 || cells->n_particles < 0) throw InvalidArgument("negative sizes");
    if (!cells->cell_offsets) throw InvalidArgument("cell_offsets is required");
    const int K = res->capacity_components;
    if (K < 1 || K > VDFCG_MAX_COMPONENTS) throw InvalidArgument("capacity_components must be 1..16");
    if (!bins->nnz || !bins->keys || !bins->counts || !bins->in_range)
      throw InvalidArgument("cell bins: nnz, keys, counts and in_range are required");
    if (!res->status || !res->components || !res->weights || !res->means || !res->covariances)
      throw InvalidArgument("cell results: status, components, weights, means, covariances are required");
    const size_t nc = cells->n_cells, n = cells->n_particles;
    CellsDev c{};
    c.d = d;
    c.n = cells->n_particles;
    c.n_cells = cells->n_cells;
    c.n_bins = cells->n_bins;
    for (int a = 0; a < 3; ++a) {
      c.lo[a] = cells->lo[a];
      c.hi[a] = cells->hi[a];
    }
    c.offsets = stage_in(ctx, cells->cell_offsets, nc + 1).dev;
    CellBinsDev b{};
    b.nnz = const_cast<int32_t*>(stage_in(ctx, bins->nnz, nc).dev);
    b.keys = const_cast<uint32_t*>(stage_in(ctx, bins->keys, n).dev);
    b.counts = const_cast<double*>(stage_in(ctx, bins->counts, n).dev);
    b.in_range = const_cast<double*>(stage_in(ctx, bins->in_range, nc).dev);
    CellModels r{K,
                 stage_in(ctx, res->status, nc).dev,
                 stage_in(ctx, res->components, nc).dev,
                 stage_in(ctx, res->weights, nc * K).dev,
                 stage_in(ctx, res->means, nc * K * d).dev,
                 stage_in(ctx, res->covariances, nc * K * d * d).dev};
    double* fields[kMetricFields] = {out->jsd, out->kl_pq, out->kl_qp, out->loglik, out->bic,
                                     out->bic_bin_count, out->mean_moment_error,
                                     out->second_moment_error, out->compression_ratio_vs_histogram,
                                     out->compression_ratio_vs_raw};
    MetricsOut mo{};
    std::vector<Staged<double>> st;
    for (int f = 0; f < kMetricFields; ++f) {
      st.push_back(stage_out(ctx, fields[f], fields[f] ? nc : 0));
      mo.f[f] = st.back().dev;
    }
    launch_cell_metrics(ctx, c, b, r, mo);
    bool host = false;
    for (auto& x : st) {
      finish(ctx, x);
      host = host || x.staged;
    }
    if (host) sync(ctx);
  });
}

int vdfcg_evaluate_pdf(vdfcg_ctx* ctx, const vdfcg_model* model, int32_t n_bins, double xlo,
                       double xhi, double ylo, double yhi, double* out) {
  return guard_impl([&] {
    begin(ctx);
    if (!out) throw InvalidArgument("null output");
    ModelDev m = staged_valid_model(ctx, model);
    if (m.d != 2) throw InvalidArgument("evaluate_pdf expects a 2-dimensional model");
    if (n_bins < 1 || !range_ok(xlo, xhi) || !range_ok(ylo, yhi)) throw InvalidArgument("invalid grid spec");
    auto o = stage_out(ctx, out, size_t(n_bins) * n_bins);
    int* err = arena<int>(ctx, 1);
    VDFCG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
    const double lo[2] = {xlo, ylo}, hi[2] = {xhi, yhi};
    launch_evaluate_pdf(ctx, m, n_bins, lo, hi, o.dev, err);
    if (read_scalar(ctx, err)) throw RuntimeError("model component covariance is not SPD");
    finish(ctx, o);
    sync(ctx);
  });
}

int vdfcg_weighted_loglik(vdfcg_ctx* ctx, const vdfcg_model* model, const double* points,
                          const double* weights, int64_t n, double* out) {
  return guard_impl([&] {
    begin(ctx);
    if (!model || !out) throw InvalidArgument("null argument");
    const int d = model->dimension, m = model->components;
    if (d != 2 && d != 3) throw InvalidArgument("model dimension must be 2 or 3");
    if (m < 1 || m > VDFCG_MAX_COMPONENTS) throw InvalidArgument("model components must be 1..16");
    if (n < 0 || (n > 0 && (!points || !weights))) throw InvalidArgument("null points");
    ModelDev md{d, m, stage_in(ctx, model->weights, m).dev, stage_in(ctx, model->means, size_t(m) * d).dev,
                stage_in(ctx, model->covariances, size_t(m) * d * d).dev, nullptr, nullptr};
    if (model->scale && model->offset) {
      md.scale = stage_in(ctx, model->scale, d).dev;
      md.offset = stage_in(ctx, model->offset, d).dev;
    }
    const double* px = stage_in(ctx, points, size_t(n) * d).dev;
    const double* pw = stage_in(ctx, weights, size_t(n)).dev;
    double* r = arena<double>(ctx, 1);
    launch_weighted_loglik(ctx, md, px, pw, n, r);
    *out = read_scalar(ctx, r);
  });
}

int vdfcg_pdf_divergences(vdfcg_ctx* ctx, const double* p, const double* q, int64_t n,
                          double area, double* jsd, double* kl_pq, double* kl_qp) {
  return guard_impl([&] {
    begin(ctx);
    if (n < 0 || (n > 0 && (!p || !q))) throw InvalidArgument("null grid");
    const double* dp = stage_in(ctx, p, size_t(n)).dev;
    const double* dq = stage_in(ctx, q, size_t(n)).dev;
    double* r = arena<double>(ctx, 3);
    launch_pdf_divergences(ctx, dp, dq, n, area, r);
    double h[3];
    VDFCG_CUDA(cudaMemcpyAsync(h, r, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (kl_pq) *kl_pq = h[1];
    if (kl_qp) *kl_qp = h[2];
    if (jsd) {  // metrics.cpp:41-45
      constexpr double ln2 = 0.6931471805599453;
      if (h[0] < -1e-9 || h[0] > ln2 + 1e-9)
        throw RuntimeError("jsd outside [0, ln 2] beyond numerical slack");
      *jsd = std::min(std::max(h[0], 0.0), ln2);
    }
  });
}

int vdfcg_synth_cells(vdfcg_ctx* ctx, int32_t d, int32_t n_cells, const int64_t* cell_offsets,
                      int64_t cell_base, uint64_t seed, int32_t species, double* u, double* v,
                      double* w) {
  return guard_impl([&] {
    begin(ctx);
    if (d != 2 && d != 3) throw InvalidArgument("dimension must be 2 or 3");
    if (!is_device_pointer(cell_offsets) || !is_device_pointer(u) || !is_device_pointer(v) ||
        (d == 3 && !is_device_pointer(w)))
      throw InvalidArgument("vdfcg_synth_cells takes device pointers");
    for (const void* q : {static_cast<const void*>(cell_offsets), static_cast<const void*>(u),
                          static_cast<const void*>(v), static_cast<const void*>(w)})
      if (q) check_pointer_device(ctx, q);
    if (n_cells > 0) launch_synth(ctx, d, n_cells, cell_offsets, cell_base, seed, species, u, v, w);
  });
}

// synthdata.cpp:54-86 (generate) after ScenarioSpec::validate (synthdata.cpp:32-52). The
// scenario (m fractions, means, covariances) is host parameter data: it is validated and
// factorised here exactly as the reference does before its particle loop; every particle
// is drawn on the device.
int vdfcg_generate(vdfcg_ctx* ctx, int32_t d, int32_t m, const double* fractions,
                   const double* means, const double* covs, int64_t n, uint64_t seed,
                   double* velocities, double* nominal_temperature) {
  return guard_impl([&] {
    begin(ctx);
    if (d != 2 && d != 3) throw InvalidArgument("scenario dimension must be 2 or 3");
    if (n < 1) throw InvalidArgument("particle_count must be >= 1");
    if (m < 1) throw InvalidArgument("scenario needs at least one component");
    if (!fractions || !means || !covs || !velocities) throw InvalidArgument("null argument");
    // params: cdf[m], mean[m][d], chol[m][3][3]
    std::vector<double> par(size_t(m) * (1 + d + 9), 0.0);
    double total = 0.0, acc = 0.0;
    for (int k = 0; k < m; ++k) {
      const std::string who = "component " + std::to_string(k);
      if (!(fractions[k] >= 0.0)) throw InvalidArgument(who + ": fraction must be >= 0");
      const double* c = covs + size_t(k) * d * d;
      double diff = 0.0, norm = 0.0;  // Eigen isApprox(transpose, 1e-12), Frobenius
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
          const double e = c[a * d + b] - c[b * d + a];
          diff += e * e;
          norm += c[a * d + b] * c[a * d + b];
        }
      if (!(diff <= 1e-24 * norm)) throw InvalidArgument(who + ": covariance is not symmetric");
      double* L = par.data() + m + size_t(m) * d + size_t(k) * 9;  // Eigen LLT, lower
      for (int j = 0; j < d; ++j) {
        double x = c[j * d + j];
        if (j > 0) {
          double sq = 0.0;
          for (int i = 0; i < j; ++i) sq += L[j * 3 + i] * L[j * 3 + i];
          x -= sq;
        }
        const double sj = std::sqrt(x);
        if (!(x > 0.0) || !std::isfinite(sj))
          throw InvalidArgument(who + ": covariance is not symmetric positive definite");
        L[j * 3 + j] = sj;
        for (int i = j + 1; i < d; ++i) {
          double v = c[i * d + j];
          for (int q = 0; q < j; ++q) v -= L[i * 3 + q] * L[j * 3 + q];
          L[i * 3 + j] = v / sj;
        }
      }
      for (int a = 0; a < d; ++a) par[m + size_t(k) * d + a] = means[size_t(k) * d + a];
      total += fractions[k];
      acc += fractions[k];
      par[k] = acc;
    }
    if (std::abs(total - 1.0) > 1e-12)
      throw InvalidArgument("fractions must sum to 1 (got " + std::to_string(total) + ")");
    par[m - 1] = 1.0;  // the last component owns the tail (synthdata.cpp:64)
    if (nominal_temperature) {  // synthdata.cpp:71-73
      for (int a = 0; a < d; ++a) nominal_temperature[a] = 0.0;
      for (int k = 0; k < m; ++k)
        for (int a = 0; a < d; ++a)
          nominal_temperature[a] += fractions[k] * covs[(size_t(k) * d + a) * d + a];
    }
    const int64_t n_uniforms = n + 2 * ((n * d + 1) / 2);
    double* dpar = arena<double>(ctx, par.size());
    VDFCG_CUDA(cudaMemcpyAsync(dpar, par.data(), par.size() * sizeof(double),
                               cudaMemcpyHostToDevice, ctx->stream));
    uint64_t* uni = arena<uint64_t>(ctx, size_t(n_uniforms));  // raw mt19937_64 words
    auto v = stage_out(ctx, velocities, size_t(n) * d);
    launch_generate(ctx, d, m, n, seed, uni, n_uniforms, dpar, v.dev);
    finish(ctx, v);
    sync(ctx);
  });
}

int vdfcg_probe_peaks(vdfcg_ctx* ctx, double* fp64, double* fp32) {
  return guard_impl([&] {
    begin(ctx);
    if (fp64) *fp64 = probe_fp64(ctx);
    if (fp32) *fp32 = probe_fp32(ctx);
  });
}

}  // extern "C"
