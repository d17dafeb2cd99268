// vdfcg.hpp — header-only C++ shim over the C-ABI (vdfcg.h) for the reference library's
// call sites. It keeps one context per (thread, device) — the reference API is pure and
// reentrant — and rethrows the reference's exception types:
//   VDFCG_INVALID_ARGUMENT -> std::invalid_argument
//   VDFCG_RUNTIME_ERROR    -> std::runtime_error
//   VDFCG_REPAIR_FAILED    -> vdfcg::CovarianceRepairError (derive/alias vdfc's, types.hpp:99)
//   VDFCG_CUDA_ERROR       -> vdfcg::CudaError (there is no CPU fallback)
// Buffers are plain pointers in the reference's Eigen (column-major) layouts, so an Eigen
// caller passes `.data()` directly; see INTEGRATION.md.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "vdfcg.h"

namespace vdfcg {

struct CovarianceRepairError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == VDFCG_OK) return;
  const std::string msg = vdfcg_last_error();
  switch (rc) {
    case VDFCG_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case VDFCG_REPAIR_FAILED: throw CovarianceRepairError(msg);
    case VDFCG_CUDA_ERROR: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

// RAII context (one CUDA stream + workspace on one device).
class Context {
 public:
  explicit Context(int device = 0) { check(vdfcg_ctx_create(device, &ctx_)); }
  ~Context() { vdfcg_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  vdfcg_ctx* get() const { return ctx_; }
  void set_stream(void* stream) { check(vdfcg_ctx_set_stream(ctx_, stream)); }
  void synchronize() { check(vdfcg_ctx_synchronize(ctx_)); }

  // Per-thread default context on `device`.
  static Context& thread_default(int device = 0) {
    thread_local std::vector<Context*> ctxs;
    if (static_cast<int>(ctxs.size()) <= device) ctxs.resize(device + 1, nullptr);
    if (!ctxs[device]) ctxs[device] = new Context(device);  // lives for the thread
    return *ctxs[device];
  }

 private:
  vdfcg_ctx* ctx_ = nullptr;
};

// Fit result with owning storage, mirroring vdfc::FitResult (wgmm.hpp:64-70).
struct FitOutput {
  int dimension = 0;
  int components = 0;
  std::vector<double> weights, means, covariances;  // component-major
  std::vector<double> loglik_trace;
  int iterations_used = 0;
  bool converged = false;
  struct Event {
    int iteration, component;
    double weight;
  };
  std::vector<Event> pruning_events;
};

// vdfc::fit (wgmm.hpp:126) on N x d column-major points.
inline FitOutput fit(const double* points, const double* weights, int64_t n, int d,
                     double total_weight, const vdfcg_fit_config& cfg,
                     Context& ctx = Context::thread_default()) {
  const int k = std::max(cfg.initial_components, cfg.warm_start ? cfg.warm_start->components : 0);
  FitOutput out;
  out.weights.resize(k);
  out.means.resize(size_t(k) * d);
  out.covariances.resize(size_t(k) * d * d);
  out.loglik_trace.resize(cfg.max_em_iterations);
  std::vector<int32_t> ev_it(k), ev_c(k);
  std::vector<double> ev_w(k);
  vdfcg_fit_result r{};
  r.capacity_components = k;
  r.capacity_trace = cfg.max_em_iterations;
  r.model.weights = out.weights.data();
  r.model.means = out.means.data();
  r.model.covariances = out.covariances.data();
  r.loglik_trace = out.loglik_trace.data();
  r.event_iteration = ev_it.data();
  r.event_component = ev_c.data();
  r.event_weight = ev_w.data();
  check(vdfcg_fit(ctx.get(), points, weights, n, d, total_weight, &cfg, &r));
  out.dimension = d;
  out.components = r.model.components;
  out.weights.resize(out.components);
  out.means.resize(size_t(out.components) * d);
  out.covariances.resize(size_t(out.components) * d * d);
  out.loglik_trace.resize(r.trace_len);
  out.iterations_used = r.iterations_used;
  out.converged = r.converged != 0;
  for (int e = 0; e < r.n_events; ++e) out.pruning_events.push_back({ev_it[e], ev_c[e], ev_w[e]});
  return out;
}

// vdfc::bin_particles (histogram.hpp:48-49): counts is n_bins x n_bins column-major.
inline double bin_particles(const double* velocities, int64_t n, int d, const double* weights,
                            int plane, int n_bins, double xlo, double xhi, double ylo, double yhi,
                            double* counts, Context& ctx = Context::thread_default()) {
  double oor = 0.0;
  check(vdfcg_bin_particles(ctx.get(), velocities, n, d, weights, plane, n_bins, xlo, xhi, ylo,
                            yhi, counts, &oor));
  return oor;
}

// vdfc::generate (synthdata.cpp:54-86): n x d column-major velocities drawn on the device
// from the reference's mt19937_64(seed) stream; returns the nominal temperature per axis.
inline std::vector<double> generate(int d, const std::vector<double>& fractions,
                                    const std::vector<double>& means,
                                    const std::vector<double>& covariances, int64_t n,
                                    uint64_t seed, double* velocities,
                                    Context& ctx = Context::thread_default()) {
  // ScenarioSpec::validate's shape checks (synthdata.cpp:39-43), before any pointer is read
  const size_t m = fractions.size(), dd = static_cast<size_t>(d > 0 ? d : 0);
  for (size_t k = 0; k < m; ++k) {
    const std::string who = "component " + std::to_string(k);
    if (means.size() < (k + 1) * dd) throw std::invalid_argument(who + ": mean dimension mismatch");
    if (covariances.size() < (k + 1) * dd * dd)
      throw std::invalid_argument(who + ": covariance shape mismatch");
  }
  if (means.size() != m * dd) throw std::invalid_argument("generate: means size != m*d");
  if (covariances.size() != m * dd * dd)
    throw std::invalid_argument("generate: covariances size != m*d*d");
  std::vector<double> temperature(dd);
  check(vdfcg_generate(ctx.get(), d, static_cast<int32_t>(fractions.size()), fractions.data(),
                       means.data(), covariances.data(), n, seed, velocities,
                       temperature.data()));
  return temperature;
}

// vdfc::encode_model (codec.hpp:48).
inline std::vector<uint8_t> encode_model(const vdfcg_model& model, const vdfcg_model_meta& meta,
                                         Context& ctx = Context::thread_default()) {
  const int64_t cap = vdfcg_model_header_bytes(model.dimension, meta.label_len) +
                      vdfcg_model_payload_bytes(model.components, model.dimension);
  std::vector<uint8_t> out(static_cast<size_t>(cap));
  int64_t len = 0;
  check(vdfcg_encode_model(ctx.get(), &model, &meta, out.data(), cap, &len));
  out.resize(static_cast<size_t>(len));
  return out;
}

}  // namespace vdfcg
