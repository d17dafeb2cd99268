// refem_shim.cpp — C entry point around the reference's own Eigen-free EM oracle
// (proj/tests/support/reference_em.{hpp,cpp}), which oracle/Makefile compiles from
// /root/reference into oracle/_ref/librefem.so. TEST INFRASTRUCTURE: used only to pin
// the oracle restatement (tests/test_oracle_vs_refem.py, tests/golden/make_golden.py).
#include <cstdint>
#include <vector>

#include "reference_em.hpp"

extern "C" int refem_fit_c(const double* xs, const double* ys, int64_t n, int32_t m,
                           int32_t max_iterations, double prune_threshold,
                           int32_t prune_interval, double tolerance, uint64_t seed,
                           double t0, double t1, int32_t cap_components, int32_t cap_trace,
                           double* alpha, double* means, double* covs, double* trace,
                           int32_t* n_components, int32_t* trace_len, int32_t* iterations,
                           int32_t* converged) {
  try {
    refem::Config cfg;
    cfg.initial_components = m;
    cfg.max_iterations = max_iterations;
    cfg.prune_threshold = prune_threshold;
    cfg.prune_interval = prune_interval;
    cfg.tolerance = tolerance;
    cfg.seed = seed;
    cfg.temperature[0] = t0;
    cfg.temperature[1] = t1;
    const std::vector<double> x(xs, xs + n), y(ys, ys + n);
    const refem::Result r = refem::fit(x, y, cfg);
    const int mc = static_cast<int>(r.components.size());
    if (mc > cap_components || static_cast<int>(r.loglik_trace.size()) > cap_trace) return 2;
    for (int i = 0; i < mc; ++i) {
      alpha[i] = r.components[i].alpha;
      means[2 * i] = r.components[i].mean[0];
      means[2 * i + 1] = r.components[i].mean[1];
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) covs[4 * i + 2 * a + b] = r.components[i].cov[a][b];
    }
    for (size_t t = 0; t < r.loglik_trace.size(); ++t) trace[t] = r.loglik_trace[t];
    *n_components = mc;
    *trace_len = static_cast<int32_t>(r.loglik_trace.size());
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    return 0;
  } catch (...) {
    return 1;
  }
}
