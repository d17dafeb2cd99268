// em_entry.cuh — launchers for the fine-grained EM entry points (em_entry.cu).
#pragma once

#include "em.cuh"

namespace vdfcg {

void launch_init_model(vdfcg_ctx* ctx, int d, const double* z, int64_t n, const EmConfig& cfg,
                       const Frame& f, double* w, double* mu, double* cov, int* m_out);
void launch_e_step(vdfcg_ctx* ctx, int d, int m, const double* alpha, const double* mu,
                   double* cov, const double* x, const double* w, int64_t n, double* resp,
                   double* loglik, int* dead_list, int* n_dead);
void launch_m_step(vdfcg_ctx* ctx, int d, const double* x, const double* w, int64_t n,
                   double total, const double* resp, int m, const double* prev_mu,
                   const double* prev_cov, double* out_w, double* out_mu, double* out_cov,
                   int* degen, int* bad);
void launch_prune_one(vdfcg_ctx* ctx, int d, double* alpha, double* mu, double* cov, int* m_io,
                      double thr, int* pruned, int* idx, double* weight);
void launch_repair(vdfcg_ctx* ctx, int d, const double* sigma, double* out, int* doublings,
                   int* ok);

}  // namespace vdfcg
