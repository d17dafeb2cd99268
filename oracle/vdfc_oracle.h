/*
 * vdfc_oracle.h — CPU restatement of the reference histogram -> weighted-EM -> writer
 * path. TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may call it, always as the checker or as the
 * timed CPU baseline, never as the product path.
 *
 * Parity is PINNED: the EM restatement is checked against the reference's own
 * Eigen-free oracle `refem::fit` (proj/tests/support/reference_em.cpp, compiled from
 * /root/reference into oracle/_ref by oracle/Makefile), the histogram restatement
 * against the KATs of proj/tests/unit/test_histogram.cpp and the writer against the
 * FORMATS.md:35-47 hex vector (see tests/test_oracle_*.py).
 *
 * Structs are shared with the product ABI (include/vdfcg.h) so the tests feed both
 * sides the same buffers. Host pointers only.
 */
#ifndef VDFC_ORACLE_H
#define VDFC_ORACLE_H

#include "../include/vdfcg.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* oracle_last_error(void);

/* rng.hpp:22 — n uniforms from mt19937_64(seed), top 53 bits. */
void oracle_uniforms(uint64_t seed, int64_t n, double* out);

/* synthdata.cpp:54-86 — Gaussian-mixture generator (fixture producer).
 * means [m*d], covs [m*d*d]; out velocities N x d column-major; nominal_temperature [d]. */
int oracle_generate(int32_t d, int32_t m, const double* fractions, const double* means,
                    const double* covs, int64_t n, uint64_t seed, double* velocities,
                    double* nominal_temperature);

/* histogram.cpp:45-76 */
int oracle_bin_particles(const double* velocities, int64_t n, int32_t d, const double* weights,
                         int32_t plane, int32_t n_bins, double xlo, double xhi, double ylo,
                         double yhi, double* counts, double* out_of_range);
/* histogram.cpp:78-84 */
int oracle_all_planes(const double* velocities, int64_t n, int32_t d, const double* weights,
                      int32_t n_bins, double lo, double hi, double* counts3, double* oor3);
/* histogram.cpp:86-109 */
int oracle_to_weighted_points(const double* counts, int32_t n_bins, double xlo, double xhi,
                              double ylo, double yhi, int32_t drop_empty, int64_t capacity,
                              double* points, double* weights, int64_t* count,
                              double* total_weight);

/* wgmm.cpp:65-76 */
int oracle_validate_fit_config(const vdfcg_fit_config* cfg, int32_t dimension);
/* wgmm.cpp:78-100 */
int oracle_normalize(const double* points, const double* weights, int64_t n, int32_t d,
                     double* out_points, double* scale, double* offset);
/* wgmm.cpp:102-120 */
int oracle_denormalize_model(const vdfcg_model* in, vdfcg_model* out);
/* wgmm.cpp:136-191 */
int oracle_init_model(const double* normalized_points, int64_t n, int32_t d,
                      const vdfcg_fit_config* cfg, const double* temperature, const double* scale,
                      const double* offset, vdfcg_model* out);
/* wgmm.cpp:233-255 */
int oracle_e_step(vdfcg_model* model, const double* points, const double* weights, int64_t n,
                  double* resp, double* loglik, int32_t* unrepairable, int32_t* n_unrepairable);
/* wgmm.cpp:269-318 */
int oracle_m_step(const double* points, const double* weights, int64_t n, double total_weight,
                  const double* resp, const vdfcg_model* previous, vdfcg_model* out,
                  int32_t* degenerate, int32_t* n_degenerate);
/* wgmm.cpp:320-333 */
int oracle_prune_one(vdfcg_model* model, double threshold, int32_t iteration, int32_t* pruned,
                     int32_t* event_component, double* event_weight);
/* wgmm.cpp:340-362 */
int oracle_repair_covariance(const double* sigma, int32_t d, double* out, int32_t* doublings);
/* wgmm.cpp:364-423 */
int oracle_fit(const double* points, const double* weights, int64_t n, int32_t d,
               double total_weight, const vdfcg_fit_config* cfg, vdfcg_fit_result* result);
/* wgmm.cpp:455-471 / 473-480: mixture and weighted data moments (test helpers). */
int oracle_mixture_moments(const vdfcg_model* model, double* mean, double* m2);
int oracle_weighted_data_moments(const double* points, const double* weights, int64_t n,
                                 int32_t d, double* mean, double* m2);

/* codec.cpp:86-136 */
int64_t oracle_model_payload_bytes(int32_t components, int32_t dimension);
int oracle_encode_model(const vdfcg_model* model, const vdfcg_model_meta* meta, uint8_t* out,
                        int64_t capacity, int64_t* length);

/* 3V/2V per-cell generalisation: bin + compact each cell. */
int oracle_bin_cells(const vdfcg_cells* cells, vdfcg_cell_bins* out);
/* Per-particle cell ids: stable group-by-cell, then oracle_bin_cells. offsets [n_cells+1]. */
int oracle_bin_cells_indexed(const vdfcg_particles* particles, int64_t* offsets,
                             vdfcg_cell_bins* out);
/* The CPU baseline unit (pipeline.cpp:130-151): per cell bin + compact + fit, on a pool
 * of `threads` workers (0 = hardware concurrency), cells [cell_begin, cell_end). */
int oracle_compress_cells(const vdfcg_cells* cells, const vdfcg_fit_config* cfg,
                          int32_t cell_begin, int32_t cell_end, int32_t threads,
                          vdfcg_cell_bins* bins, vdfcg_cell_results* out);
/* Pack like vdfcg_pack_cells. */
int oracle_pack_cells(int32_t n_cells, int32_t dimension, const vdfcg_cell_results* res,
                      const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                      int64_t* record_offsets);

/* wgmm.cpp:425-453 evaluate_pdf (d = 2): out n x n column-major, out(i,j) at i + j*n. */
int oracle_evaluate_pdf(const vdfcg_model* model, int32_t n_bins, double xlo, double xhi,
                        double ylo, double yhi, double* out);
/* wgmm.cpp:257-267 weighted_loglik (repair on a copy; Kahan over points). */
int oracle_weighted_loglik(const vdfcg_model* model, const double* points, const double* weights,
                           int64_t n, double* out);
/* metrics.cpp:12-46 over two aligned normalised grids of n values (any layout, same order). */
int oracle_pdf_divergences(const double* p, const double* q, int64_t n, double area,
                           double* jsd, double* kl_pq, double* kl_qp);
/* pipeline.cpp:106-128 assemble_metrics per cell over the bins^d grid (d = 2 is the
 * reference's plane case; d = 3 the same formulas over the 3V grid). */
int oracle_cell_metrics(const vdfcg_cells* cells, const vdfcg_cell_bins* bins,
                        const vdfcg_cell_results* res, int32_t cell_begin, int32_t cell_end,
                        int32_t threads, vdfcg_cell_metrics* out);

#ifdef __cplusplus
}
#endif
#endif
