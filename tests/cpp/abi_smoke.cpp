// C++ consumer of the drop-in shim (include/vdfcg.hpp): what a vdfc call site compiles
// against. Built by tests/test_cpp_shim.py (CPU: compile + link); run on the GPU box.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../../include/vdfcg.hpp"

int main() {
  try {
    // two Gaussian blobs, unit weights, N x 2 column-major (Eigen's default layout)
    const int n = 4000;
    std::mt19937_64 eng(7);
    std::normal_distribution<double> g;
    std::vector<double> pts(2 * n), w(n, 1.0);
    for (int i = 0; i < n; ++i) {
      pts[i] = g(eng) + (i % 2 ? 2.5 : -2.5);
      pts[n + i] = g(eng);
    }
    vdfcg_fit_config cfg{};
    cfg.initial_components = 2;
    cfg.max_em_iterations = 100;
    cfg.prune_threshold = 0.005;
    cfg.prune_check_interval = 10;
    cfg.loglik_rel_tolerance = 1e-6;
    cfg.seed = 3;
    cfg.has_temperature = 1;
    cfg.temperature[0] = cfg.temperature[1] = 1.0;
    const vdfcg::FitOutput r = vdfcg::fit(pts.data(), w.data(), n, 2, double(n), cfg);
    std::printf("components=%d iterations=%d converged=%d w0=%.6f\n", r.components,
                r.iterations_used, int(r.converged), r.weights[0]);
    // the reference's error path: zero spread on axis 0 -> std::invalid_argument "fit: ..."
    std::vector<double> bad = {1, 1, 1, 0, 1, 2};
    std::vector<double> bw(3, 1.0);
    try {
      vdfcg::fit(bad.data(), bw.data(), 3, 2, 3.0, cfg);
      std::printf("FAIL: no exception\n");
      return 1;
    } catch (const std::invalid_argument& e) {
      std::printf("invalid_argument: %s\n", e.what());
    }
    return (r.components == 2 && std::fabs(r.weights[0] + r.weights[1] - 1.0) < 1e-12) ? 0 : 1;
  } catch (const vdfcg::CudaError& e) {
    std::printf("cuda: %s\n", e.what());
    return 3;
  }
}
