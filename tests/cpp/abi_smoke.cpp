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
    if (!(r.components == 2 && std::fabs(r.weights[0] + r.weights[1] - 1.0) < 1e-12)) return 1;

    // batched path from C++: 64 cells x 2000 3V particles on the host -> compress (bins,
    // fits, .gmmc records) -> per-cell metrics -> record stream with index
    const int nc = 64, per = 2000, K = 4;
    std::vector<double> u(nc * per), v(nc * per), ww(nc * per);
    std::vector<int64_t> off(nc + 1);
    for (int c = 0; c <= nc; ++c) off[c] = int64_t(c) * per;
    for (int i = 0; i < nc * per; ++i) {
      u[i] = g(eng) + (i % 3 == 0 ? 2.0 : 0.0);
      v[i] = g(eng);
      ww[i] = g(eng);
    }
    vdfcg_cells cells{3, int64_t(nc) * per, {u.data(), v.data(), ww.data()}, nullptr, nc, off.data(), 32,
                      {-6, -6, -6}, {6, 6, 6}};
    vdfcg_fit_config cc = cfg;
    cc.initial_components = K;
    cc.temperature[2] = 1.0;
    std::vector<int32_t> st(nc), cm(nc), it(nc), cv(nc);
    std::vector<double> rw(nc * K), rm(nc * K * 3), rc(nc * K * 9), fl(nc);
    vdfcg_cell_results res{K, 0, st.data(), cm.data(), it.data(), cv.data(), rw.data(), rm.data(),
                           rc.data(), fl.data(), nullptr, nullptr, nullptr, nullptr, nullptr};
    std::vector<int32_t> nnz(nc);
    std::vector<uint32_t> keys(nc * per);
    std::vector<double> counts(nc * per), oor(nc), inr(nc);
    vdfcg_cell_bins bins{nnz.data(), keys.data(), counts.data(), oor.data(), inr.data()};
    const char label[] = "e";
    vdfcg_model_meta meta{label, 1, -1, 7, {-6, -6, -6}, {6, 6, 6}};
    const int64_t cap = int64_t(nc) * (vdfcg_model_header_bytes(3, 1) + vdfcg_model_payload_bytes(K, 3));
    std::vector<uint8_t> rec(cap);
    std::vector<int64_t> roff(nc + 1);
    vdfcg::Context& ctx = vdfcg::Context::thread_default();
    vdfcg::check(vdfcg_compress_cells(ctx.get(), &cells, &cc, &bins, &res, &meta, rec.data(), cap,
                                      roff.data()));
    std::vector<double> jsd(nc), bic(nc);
    vdfcg_cell_metrics met{jsd.data(), nullptr, nullptr, nullptr, bic.data(),
                           nullptr, nullptr, nullptr, nullptr, nullptr};
    vdfcg::check(vdfcg_metrics_cells(ctx.get(), &cells, &bins, &res, &met));
    vdfcg_stream* s = nullptr;
    vdfcg::check(vdfcg_stream_open("/tmp/abi_smoke.gmmcs", VDFCG_STREAM_GMMC, &s));
    vdfcg::check(vdfcg_stream_append_records(s, ctx.get(), rec.data(), roff.data(), nc, 0));
    int64_t n_rec = 0, n_bytes = 0;
    vdfcg::check(vdfcg_stream_close(s, &n_rec, &n_bytes));
    std::vector<double> gv(2 * 1000);  // vdfc::generate on the device
    const auto temp = vdfcg::generate(2, {0.8, 0.2}, {0, 0, 3, 0}, {1, 0, 0, 1, 0.25, 0, 0, 0.25},
                                      1000, 11, gv.data());
    std::printf("generate T=(%.3f,%.3f)\n", temp[0], temp[1]);
    try {
      vdfcg::generate(2, {0.5, 0.4}, {0, 0, 1, 1}, {1, 0, 0, 1, 1, 0, 0, 1}, 10, 1, gv.data());
    } catch (const std::invalid_argument& e) {
      std::printf("invalid_argument: %s\n", e.what());
    }
    int ok = 0;
    for (int c = 0; c < nc; ++c) ok += st[c] == 0 && jsd[c] >= 0 && jsd[c] <= std::log(2.0) && std::isfinite(bic[c]);
    std::printf("cells ok=%d records=%lld bytes=%lld\n", ok, (long long)n_rec, (long long)n_bytes);
    return (ok == nc && n_rec == nc && n_bytes == roff[nc]) ? 0 : 1;
  } catch (const vdfcg::CudaError& e) {
    std::printf("cuda: %s\n", e.what());
    return 3;
  }
}
