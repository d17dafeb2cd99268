// metrics.cuh — fit-quality kernels: the per-cell
// assemble_metrics report (pipeline.cpp:106-128) and the single-fit evaluate_pdf,
// weighted_loglik and kl/jsd entry points.
#pragma once

#include "ctx.cuh"
#include "hist.cuh"

namespace vdfcg {

constexpr int kMetricFields = 10;  // vdfcg_cell_metrics field order

// Read-only view of a cell-results buffer (device pointers).
struct CellModels {
  int K;
  const int32_t* status;
  const int32_t* comps;
  const double* w;
  const double* mu;
  const double* cov;
};

struct MetricsOut {
  double* f[kMetricFields];  // jsd, kl_pq, kl_qp, loglik, bic, bic_bin_count,
                             // mean_err, m2_err, cr_hist, cr_raw (each [n_cells] or null)
};

// A single model on the device (data space unless scale/offset are given).
struct ModelDev {
  int d, m;
  const double* w;
  const double* mu;
  const double* cov;
  const double* scale;   // null = identity map
  const double* offset;
};

void launch_cell_metrics(vdfcg_ctx* ctx, const CellsDev& c, const CellBinsDev& b,
                         const CellModels& r, const MetricsOut& o);
// out: n x n column-major; err: device int set to 1 when a covariance is not SPD.
void launch_evaluate_pdf(vdfcg_ctx* ctx, const ModelDev& m, int nb, const double* lo,
                         const double* hi, double* out, int* err);
// out: device double (the weighted log-likelihood).
void launch_weighted_loglik(vdfcg_ctx* ctx, const ModelDev& m, const double* pts,
                            const double* wts, int64_t n, double* out);
// out: device double[3] = {jsd (unclamped), kl_pq, kl_qp}.
void launch_pdf_divergences(vdfcg_ctx* ctx, const double* p, const double* q, int64_t n,
                            double area, double* out);

}  // namespace vdfcg
