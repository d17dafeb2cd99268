/*
 * vdfcg.h — C-ABI of the B200-native histogram -> weighted-GMM compression path.
 *
 * Drop-in boundary for the reference library `vdfc` (C++20, /root/reference/proj).
 * Every entry point below replaces one reference function; the citation next to it
 * names the reference interface (file:line, relative to proj/). Plain pointers and
 * sizes only: no Eigen, no torch types.
 *
 * Matrix layouts follow the reference's Eigen defaults (column-major):
 *   - particle velocities  N x d   -> velocity[a*N + n]  (SoA: u[N], v[N], w[N])
 *   - Histogram2D::counts  n x n   -> counts[i + j*n]    (i = x bin, j = y bin)
 *   - WeightedPoints::points N x d -> points[a*N + r]
 *   - EStep::responsibilities M x N -> resp[i + n*M]
 * Model parameters are component-major: weights[i], means[i*d + a],
 * covariances[i*d*d + a*d + b] (symmetric, so row/col-major coincide).
 *
 * Pointers may be host (pageable or pinned) or device memory; each call detects
 * the memory kind and stages host buffers through the context's stream. All
 * compute runs in sm_100a kernels; there is no CPU fallback — without a usable
 * CUDA device every compute call returns VDFCG_CUDA_ERROR.
 *
 * Errors mirror the reference's exception classes (return code + message from
 * vdfcg_last_error(), thread-local). The C++ shim include/vdfcg.hpp rethrows them
 * as std::invalid_argument / std::runtime_error / vdfc::CovarianceRepairError.
 *
 * Threading: a context owns one CUDA stream and a grow-only workspace; use one
 * context per host thread (the reference is reentrant).
 */
#ifndef VDFCG_H
#define VDFCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VDFCG_ABI_VERSION 1

/* Return codes. */
enum {
  VDFCG_OK = 0,
  VDFCG_INVALID_ARGUMENT = 1, /* std::invalid_argument                        */
  VDFCG_RUNTIME_ERROR = 2,    /* std::runtime_error                           */
  VDFCG_REPAIR_FAILED = 3,    /* vdfc::CovarianceRepairError (types.hpp:99)   */
  VDFCG_CUDA_ERROR = 4,       /* no device / launch failure                   */
  VDFCG_CODEC_ERROR = 5       /* vdfc::CodecError (types.hpp:93)              */
};

/* Plane ids, identical to vdfc::Plane (types.hpp:18). */
enum { VDFCG_PLANE_UV = 0, VDFCG_PLANE_VW = 1, VDFCG_PLANE_UW = 2, VDFCG_PLANE_NONE = 255 };

/* Largest component count a fit may start with (FitConfig::initial_components). */
#define VDFCG_MAX_COMPONENTS 16

typedef struct vdfcg_ctx vdfcg_ctx;

/* A GmmModel view (wgmm.hpp:27-39). Arrays are caller-owned. `scale`/`offset`
 * carry the AffineMap (types.hpp:59-81); NULL means the identity map. */
typedef struct vdfcg_model {
  int32_t dimension;
  int32_t components;
  double* weights;     /* [components]           */
  double* means;       /* [components * d]       */
  double* covariances; /* [components * d * d]   */
  double* scale;       /* [d] or NULL (identity) */
  double* offset;      /* [d] or NULL (identity) */
} vdfcg_model;

/* FitConfig (wgmm.hpp:41-56). `warm_start` is a canonical (data-space) model or NULL. */
typedef struct vdfcg_fit_config {
  int32_t initial_components;   /* default 12   */
  int32_t max_em_iterations;    /* default 100  */
  double prune_threshold;       /* default 0.005 */
  int32_t prune_check_interval; /* default 10   */
  double loglik_rel_tolerance;  /* default 1e-6 */
  uint64_t seed;                /* default 0    */
  int32_t has_temperature;      /* 0: weighted variance of the points (wgmm.cpp:374) */
  double temperature[3];        /* per-axis variance, data units */
  const vdfcg_model* warm_start;
  /* NOT in the reference: 1 = FP32 E-step (log-densities, log-sum-exp, responsibilities in
   * single precision; sufficient statistics, M-step and protocol in FP64) on the cell-
   * batched path, parity tolerance 1e-4 relative instead of 1e-9. 0 (default) = FP64. */
  int32_t estep_fp32;
} vdfcg_fit_config;

/* FitResult (wgmm.hpp:64-70). Capacities are set by the caller. */
typedef struct vdfcg_fit_result {
  int32_t capacity_components; /* >= initial_components (or warm-start M) */
  int32_t capacity_trace;      /* >= max_em_iterations */
  vdfcg_model model;           /* out: canonical model, identity map (scale/offset ignored) */
  double* loglik_trace;        /* [capacity_trace] */
  int32_t trace_len;
  int32_t iterations_used;
  int32_t converged;
  int32_t n_events;            /* pruning events, capacity = capacity_components */
  int32_t* event_iteration;
  int32_t* event_component;
  double* event_weight;
} vdfcg_fit_result;

/* ModelMeta (codec.hpp:20-25). */
typedef struct vdfcg_model_meta {
  const char* species_label; /* UTF-8, not NUL-terminated necessarily */
  int32_t label_len;
  int32_t plane;             /* VDFCG_PLANE_* */
  int64_t cycle;
  double range_lo[3];
  double range_hi[3];
} vdfcg_model_meta;

/* ------------------------------------------------------------------------- */
/* Context, errors                                                            */
/* ------------------------------------------------------------------------- */
const char* vdfcg_last_error(void);
int vdfcg_abi_version(void);
int vdfcg_ctx_create(int device, vdfcg_ctx** out);
int vdfcg_ctx_destroy(vdfcg_ctx* ctx);
/* Ordering: a call whose inputs and outputs are all device memory is asynchronous — it
 * is enqueued on the context stream and returns; results are ready for work ordered
 * after it on that stream (or after vdfcg_ctx_synchronize). Calls with any host buffer
 * return after their host outputs are written. Set the context stream to the caller's
 * stream (e.g. torch.cuda.current_stream().cuda_stream) to order library work with the
 * caller's kernels; NULL restores the context's own stream. */
int vdfcg_ctx_set_stream(vdfcg_ctx* ctx, void* cuda_stream);
int vdfcg_ctx_synchronize(vdfcg_ctx* ctx);
/* Per-kernel device timing (CUDA events on the context stream). When enabled, every
 * kernel launch is bracketed by events; vdfcg_ctx_kernel_times reports, per kernel
 * family, the summed milliseconds and launch count since the last reset. */
int vdfcg_ctx_enable_timing(vdfcg_ctx* ctx, int enable);
int vdfcg_ctx_reset_timing(vdfcg_ctx* ctx);
int vdfcg_ctx_kernel_times(vdfcg_ctx* ctx, int32_t max_entries, char* names /* max_entries*32 */,
                           double* ms, int64_t* launches, int32_t* n_entries);
/* Total kernel launches issued by this context since creation. */
int64_t vdfcg_ctx_launch_count(vdfcg_ctx* ctx);
/* Diagnostics since creation/last reset: number of (fit, iteration) pairs that ran the
 * exact second M-step pass. reset != 0 zeroes the counters. */
int vdfcg_ctx_diagnostics(vdfcg_ctx* ctx, int64_t* exact_passes, int reset);

/* ------------------------------------------------------------------------- */
/* Histogram (histogram.hpp / histogram.cpp)                                  */
/* ------------------------------------------------------------------------- */

/* bin_particles (histogram.hpp:48-49, histogram.cpp:45-76). velocities: N x d
 * column-major; weights NULL = unit weights. counts: n_bins^2 column-major. */
int vdfcg_bin_particles(vdfcg_ctx* ctx, const double* velocities, int64_t n, int32_t d,
                        const double* weights, int32_t plane, int32_t n_bins, double xlo,
                        double xhi, double ylo, double yhi, double* counts,
                        double* out_of_range);

/* all_planes (histogram.hpp:53, histogram.cpp:78-84): the uv, vw, uw marginals in
 * ONE pass over the particles. counts3: 3 consecutive n_bins^2 column-major grids. */
int vdfcg_all_planes(vdfcg_ctx* ctx, const double* velocities, int64_t n, int32_t d,
                     const double* weights, int32_t n_bins, double lo, double hi,
                     double* counts3, double* out_of_range3);

/* to_weighted_points (histogram.hpp:55, histogram.cpp:86-109). `points` is
 * count x 2 column-major with leading dimension = *count (the non-empty bin count
 * when drop_empty, else n_bins^2); capacity bounds *count. */
int vdfcg_to_weighted_points(vdfcg_ctx* ctx, const double* counts, int32_t n_bins, double xlo,
                             double xhi, double ylo, double yhi, int32_t drop_empty,
                             int64_t capacity, double* points, double* weights, int64_t* count,
                             double* total_weight);

/* ------------------------------------------------------------------------- */
/* Weighted EM (wgmm.hpp / wgmm.cpp)                                          */
/* ------------------------------------------------------------------------- */

/* FitConfig::validate (wgmm.cpp:65-76); host-only, no device needed. */
int vdfcg_validate_fit_config(const vdfcg_fit_config* cfg, int32_t dimension);

/* normalize (wgmm.hpp:74, wgmm.cpp:78-100). out_points N x d column-major. */
int vdfcg_normalize(vdfcg_ctx* ctx, const double* points, const double* weights, int64_t n,
                    int32_t d, double* out_points, double* scale, double* offset);

/* denormalize_model (wgmm.hpp:78, wgmm.cpp:102-120). out->scale/offset ignored. */
int vdfcg_denormalize_model(vdfcg_ctx* ctx, const vdfcg_model* in, vdfcg_model* out);

/* init_model (wgmm.hpp:85-86, wgmm.cpp:136-191). `normalized_points` N x d; the map is
 * (scale, offset); out->components receives the (possibly reduced) M. */
int vdfcg_init_model(vdfcg_ctx* ctx, const double* normalized_points, int64_t n, int32_t d,
                     const vdfcg_fit_config* cfg, const double* temperature,
                     const double* scale, const double* offset, vdfcg_model* out);

/* e_step (wgmm.hpp:97, wgmm.cpp:233-255). MUTATES `model` covariances (in-place
 * repair). resp: M x N column-major. unrepairable: capacity M. */
int vdfcg_e_step(vdfcg_ctx* ctx, vdfcg_model* model, const double* points, const double* weights,
                 int64_t n, double* resp, double* loglik, int32_t* unrepairable,
                 int32_t* n_unrepairable);

/* m_step (wgmm.hpp:106-107, wgmm.cpp:269-318). degenerate: capacity M (may be NULL). */
int vdfcg_m_step(vdfcg_ctx* ctx, const double* points, const double* weights, int64_t n,
                 double total_weight, const double* resp, const vdfcg_model* previous,
                 vdfcg_model* out, int32_t* degenerate, int32_t* n_degenerate);

/* prune_one (wgmm.hpp:112, wgmm.cpp:320-333). In place; *pruned = 1 when an event happened. */
int vdfcg_prune_one(vdfcg_ctx* ctx, vdfcg_model* model, double threshold, int32_t iteration,
                    int32_t* pruned, int32_t* event_component, double* event_weight);

/* repair_covariance (wgmm.hpp:120, wgmm.cpp:340-362). doublings may be NULL. */
int vdfcg_repair_covariance(vdfcg_ctx* ctx, const double* sigma, int32_t d, double* out,
                            int32_t* doublings);

/* fit (wgmm.hpp:126, wgmm.cpp:364-423). points N x d column-major. */
int vdfcg_fit(vdfcg_ctx* ctx, const double* points, const double* weights, int64_t n, int32_t d,
              double total_weight, const vdfcg_fit_config* cfg, vdfcg_fit_result* result);

/* ------------------------------------------------------------------------- */
/* Writer (codec.hpp / codec.cpp, FORMATS.md)                                  */
/* ------------------------------------------------------------------------- */
/* model_payload_bytes (codec.hpp:36, codec.cpp:86-89). */
int64_t vdfcg_model_payload_bytes(int32_t components, int32_t dimension);
/* Header bytes of a .gmmc record: 4+4+4+8+16d+2+L+4 (FORMATS.md:11-24). */
int64_t vdfcg_model_header_bytes(int32_t dimension, int32_t label_len);
/* encode_model (codec.hpp:48, codec.cpp:103-136). */
int vdfcg_encode_model(vdfcg_ctx* ctx, const vdfcg_model* model, const vdfcg_model_meta* meta,
                       uint8_t* out, int64_t capacity, int64_t* length);

/* ------------------------------------------------------------------------- */
/* Cell-batched path (new: the GPU generalisation of the per-subdomain fan-out, */
/* pipeline.cpp:76-104,130-160,340-349; 3V bins per SURVEY.md Appendix A)      */
/* ------------------------------------------------------------------------- */

/* Particles of one species, grouped by spatial cell (PIC ownership order). */
typedef struct vdfcg_cells {
  int32_t dimension;            /* 2 or 3 velocity axes */
  int64_t n_particles;
  const double* velocity[3];    /* SoA axis arrays u, v, w; each n_particles */
  const double* weights;        /* NULL = unit weights */
  int32_t n_cells;
  const int64_t* cell_offsets;  /* [n_cells+1]; cell c owns particles [off[c], off[c+1]) */
  int32_t n_bins;               /* per axis; bins^d flat index (i*n+j)*n+k */
  double lo[3];
  double hi[3];
} vdfcg_cells;

/* Compacted per-cell histograms: cell c's non-empty bins, ascending flat key
 * (= to_weighted_points(drop_empty) order), stored at [off[c], off[c]+nnz[c]). */
typedef struct vdfcg_cell_bins {
  int32_t* nnz;          /* [n_cells] */
  uint32_t* keys;        /* [n_particles] */
  double* counts;        /* [n_particles] */
  double* out_of_range;  /* [n_cells] */
  double* in_range;      /* [n_cells] (Histogram2D::in_range_count) */
} vdfcg_cell_bins;

/* Per-cell fit results, SoA with stride K = capacity_components. */
typedef struct vdfcg_cell_results {
  int32_t capacity_components;
  int32_t capacity_trace;   /* 0: no trace stored */
  int32_t* status;          /* [n_cells] VDFCG_* per cell */
  int32_t* components;      /* [n_cells] M-hat */
  int32_t* iterations;      /* [n_cells] */
  int32_t* converged;       /* [n_cells] */
  double* weights;          /* [n_cells*K] */
  double* means;            /* [n_cells*K*d] */
  double* covariances;      /* [n_cells*K*d*d] */
  double* final_loglik;     /* [n_cells] last E-step loglik (fitting frame) */
  double* loglik_trace;     /* [n_cells*capacity_trace] or NULL */
  int32_t* n_events;        /* [n_cells] or NULL */
  int32_t* event_iteration; /* [n_cells*K] or NULL */
  int32_t* event_component; /* [n_cells*K] or NULL */
  double* event_weight;     /* [n_cells*K] or NULL */
} vdfcg_cell_results;

/* Histogram every cell (bins^d, exact integer counts for unit weights). */
int vdfcg_bin_cells(vdfcg_ctx* ctx, const vdfcg_cells* cells, vdfcg_cell_bins* out);

/* Fit every cell's compacted histogram with the same FitConfig (pipeline.cpp:144 copies
 * cfg.fit unchanged for every part). temperature: [d] or NULL (cfg / weighted variance). */
int vdfcg_fit_cells(vdfcg_ctx* ctx, const vdfcg_cells* cells, const vdfcg_cell_bins* bins,
                    const vdfcg_fit_config* cfg, vdfcg_cell_results* out);

/* Time-series warm start (pipeline.cpp:482-564, wgmm.cpp:142-161 per cell): cell c starts
 * from `warm`'s model of cell c (the previous cycle's results, canonical data space) when
 * warm->status[c] == 0 and warm->components[c] > 0, else from the seeded random init. */
int vdfcg_fit_cells_warm(vdfcg_ctx* ctx, const vdfcg_cells* cells, const vdfcg_cell_bins* bins,
                         const vdfcg_fit_config* cfg, const vdfcg_cell_results* warm,
                         vdfcg_cell_results* out);

/* Pack every cell's fitted model as a .gmmc record (FORMATS.md). records: capacity
 * bytes; record_offsets: [n_cells+1]. Cells with status != 0 get an empty record. */
int vdfcg_pack_cells(vdfcg_ctx* ctx, int32_t n_cells, int32_t dimension,
                     const vdfcg_cell_results* res, const vdfcg_model_meta* meta,
                     uint8_t* records, int64_t capacity, int64_t* record_offsets);

/* ---- Record streams ----------------------------------------
 * A stream file is a plain concatenation of standard FORMATS.md payloads — .gmmc
 * records (kind 0) or .h2d histogram payloads (kind 1, n_bins^2 f64, x bin = row) — so
 * every record stays decodable by the reference's decode_model / decode_histogram.
 * `<path>.idx` indexes it: "GMIX", u8 version (1), u8 kind, u16 reserved, u64 count, then
 * per record {i64 cell, u64 offset, u32 length, u32 crc32 (zlib) of the record bytes,
 * f64 aux (h2d: out_of_range_count; gmmc: 0)}, little-endian. Cells whose fit failed
 * have length 0. Appends copy device data to pinned staging on the context stream and
 * return; a per-stream IO thread waits for each copy and writes it, so file IO
 * overlaps the next batch's kernels. A stream is used by one host thread at a time. */
typedef struct vdfcg_stream vdfcg_stream;

#define VDFCG_STREAM_GMMC 0
#define VDFCG_STREAM_H2D 1

int vdfcg_stream_open(const char* path, int32_t kind, vdfcg_stream** out);
/* Records of cells [cell_base, cell_base + n_cells) as produced by vdfcg_pack_cells /
 * vdfcg_compress_cells (host or device buffers). */
int vdfcg_stream_append_records(vdfcg_stream* s, vdfcg_ctx* ctx, const uint8_t* records,
                                const int64_t* record_offsets, int32_t n_cells,
                                int64_t cell_base);
/* One .h2d payload per 2V cell (encode_histogram, codec.cpp:260-267) from compacted
 * cell histograms (vdfcg_bin_cells output; host or device). */
int vdfcg_stream_append_h2d(vdfcg_stream* s, vdfcg_ctx* ctx, const vdfcg_cells* cells,
                            const vdfcg_cell_bins* bins, int64_t cell_base);
/* Wait for every pending write, write the index, close the files. */
int vdfcg_stream_close(vdfcg_stream* s, int64_t* n_records, int64_t* n_bytes);

/* ---- Fit quality ------------------------------------------- */

/* Per-cell MetricsReport (metrics.hpp:39-54) as assemble_metrics computes it
 * (pipeline.cpp:106-128), over each cell's bins^d grid: d = 2 is the reference's plane
 * case, d = 3 applies the same formulas to the 3V grid. Arrays are [n_cells]; any may be
 * NULL. Cells with status != 0, no components or an empty histogram get NaN. `cells`
 * supplies the grid (n_bins, lo, hi), cell_offsets (bins CSR + raw particle counts) and
 * dimension; its particle arrays are not read. */
typedef struct vdfcg_cell_metrics {
  double* jsd;                 /* metrics.cpp:28-46, clamped to [0, ln 2] */
  double* kl_pq;               /* metrics.cpp:12-26, D(hist || model); +inf = divergent */
  double* kl_qp;               /* D(model || hist) */
  double* loglik;              /* weighted_loglik (wgmm.cpp:257-267) over the cell's points */
  double* bic;                 /* metrics.cpp:52-56 with n = total weight */
  double* bic_bin_count;       /* ... with n = n_bins^d */
  double* mean_moment_error;   /* metrics.cpp:58-65 */
  double* second_moment_error;
  double* compression_ratio_vs_histogram;  /* n_bins^d * 8 / payload bytes */
  double* compression_ratio_vs_raw;        /* cell particles * d * 8 / payload bytes */
} vdfcg_cell_metrics;

int vdfcg_metrics_cells(vdfcg_ctx* ctx, const vdfcg_cells* cells, const vdfcg_cell_bins* bins,
                        const vdfcg_cell_results* res, vdfcg_cell_metrics* out);

/* evaluate_pdf (wgmm.hpp:130, wgmm.cpp:425-453): d = 2 model (normalisation map honoured)
 * on the n_bins x n_bins grid; out column-major, out(i,j) at i + j*n_bins. */
int vdfcg_evaluate_pdf(vdfcg_ctx* ctx, const vdfcg_model* model, int32_t n_bins, double xlo,
                       double xhi, double ylo, double yhi, double* out);

/* weighted_loglik (wgmm.cpp:257-267): sum_n w_n log sum_k alpha_k N(x_n), points N x d
 * column-major; covariances are repaired on a copy like the reference. */
int vdfcg_weighted_loglik(vdfcg_ctx* ctx, const vdfcg_model* model, const double* points,
                          const double* weights, int64_t n, double* out);

/* kl_divergence / jsd (metrics.cpp:12-46) of two aligned normalised grids of n values
 * (PdfGrid values; bin mass = value * area). Any output may be NULL. */
int vdfcg_pdf_divergences(vdfcg_ctx* ctx, const double* p, const double* q, int64_t n,
                          double area, double* jsd, double* kl_pq, double* kl_qp);

/* The whole compression step: bin_cells -> fit_cells (-> pack_cells when records != NULL),
 * one stream, no host round trip in between. */
int vdfcg_compress_cells(vdfcg_ctx* ctx, const vdfcg_cells* cells, const vdfcg_fit_config* cfg,
                         vdfcg_cell_bins* bins, vdfcg_cell_results* out,
                         const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                         int64_t* record_offsets);

/* compress_cells with the per-cell warm start of vdfcg_fit_cells_warm. */
int vdfcg_compress_cells_warm(vdfcg_ctx* ctx, const vdfcg_cells* cells,
                              const vdfcg_fit_config* cfg, const vdfcg_cell_results* warm,
                              vdfcg_cell_bins* bins, vdfcg_cell_results* out,
                              const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                              int64_t* record_offsets);

/* ---- Per-particle cell-index input (north_star: "streams particle (u,v,w) and cell-index
 * arrays"). The particles of one species in ANY order, each with an int32 cell id — the
 * device-side equivalent of the reference's per-part fan-out (split_subdomains then
 * fit_one_plane per part, pipeline.cpp:76-104,130-160,340-345) for a caller that owns a PIC
 * particle array. The library groups the particles by cell with a stable device sort (each
 * cell keeps its particles in input order, so fractional weights are summed in the order of
 * the reference's sequential `counts(i,j) += w`, histogram.cpp:66-74), then bins and fits
 * exactly like the cell-grouped path. Cell c of the results is cell id c. */
typedef struct vdfcg_particles {
  int32_t dimension;            /* 2 or 3 velocity axes */
  int64_t n_particles;          /* < 2^32 per call */
  const double* velocity[3];    /* SoA axis arrays u, v, w; each n_particles, any order */
  const double* weights;        /* NULL = unit weights */
  const int32_t* cell;          /* [n_particles] cell id of each particle, in [0, n_cells) */
  int32_t n_cells;
  int32_t n_bins;               /* per axis; bins^d flat index (i*n+j)*n+k */
  double lo[3];
  double hi[3];
} vdfcg_particles;

/* Histogram every cell of an unsorted particle array. cell_offsets (out, [n_cells+1]) is
 * the CSR of the grouped particles (cell c owned off[c+1]-off[c] of them); `out` is indexed
 * by it exactly as vdfcg_bin_cells' output, so vdfcg_fit_cells / vdfcg_metrics_cells accept
 * (a vdfcg_cells with these offsets, out). A cell id outside [0, n_cells) is an
 * invalid_argument ("cell index out of range"). */
int vdfcg_bin_cells_indexed(vdfcg_ctx* ctx, const vdfcg_particles* particles,
                            int64_t* cell_offsets, vdfcg_cell_bins* out);

/* bin_cells_indexed -> fit_cells (-> pack_cells when records != NULL) on one stream.
 * cell_offsets and bins may be NULL (workspace). */
int vdfcg_compress_cells_indexed(vdfcg_ctx* ctx, const vdfcg_particles* particles,
                                 const vdfcg_fit_config* cfg, int64_t* cell_offsets,
                                 vdfcg_cell_bins* bins, vdfcg_cell_results* out,
                                 const vdfcg_model_meta* meta, uint8_t* records,
                                 int64_t capacity, int64_t* record_offsets);
/* ... with the per-cell warm start of vdfcg_fit_cells_warm (the in-situ time series,
 * pipeline.cpp:482-564): cell id c restarts from warm's model of cell c. */
int vdfcg_compress_cells_indexed_warm(vdfcg_ctx* ctx, const vdfcg_particles* particles,
                                      const vdfcg_fit_config* cfg, const vdfcg_cell_results* warm,
                                      int64_t* cell_offsets, vdfcg_cell_bins* bins,
                                      vdfcg_cell_results* out, const vdfcg_model_meta* meta,
                                      uint8_t* records, int64_t capacity, int64_t* record_offsets);

/* ---- Several devices from one host process (run_pipeline's fan-out over
 * parts and final gather, pipeline.cpp:340-353). Cells are independent, so a batch is split
 * into contiguous cell ranges balanced by particle count and each device bins, fits and
 * packs its range on its own context and host thread; no collective on the data path. The
 * records of all devices are gathered in cell order into one host buffer with global
 * offsets — byte-identical to a one-device call. */
typedef struct vdfcg_multi vdfcg_multi;

/* Contiguous cell ranges [cell_begin[r], cell_begin[r+1]) for n_parts workers with about
 * (off[n_cells] - off[0]) / n_parts particles each (the cell boundary whose particle prefix
 * is nearest r * total / n_parts). Host-only: needs no device. cell_begin: [n_parts + 1]. */
int vdfcg_partition_cells(const int64_t* cell_offsets, int32_t n_cells, int32_t n_parts,
                          int32_t* cell_begin);
int vdfcg_multi_create(const int32_t* devices, int32_t n_devices, vdfcg_multi** out);
int vdfcg_multi_destroy(vdfcg_multi* m);
int32_t vdfcg_multi_device_count(const vdfcg_multi* m);
/* The context of device slot `index` (e.g. to enable per-kernel timing). */
int vdfcg_multi_context(vdfcg_multi* m, int32_t index, vdfcg_ctx** out);
/* vdfcg_compress_cells over every device of `m`. Host buffers (cells->cell_offsets must be
 * host memory); bins may be NULL; records/record_offsets as vdfcg_compress_cells over the
 * whole batch. cell_begin (may be NULL) receives the partition used, [n_devices + 1]. */
int vdfcg_multi_compress_cells(vdfcg_multi* m, const vdfcg_cells* cells, const vdfcg_fit_config* cfg,
                               vdfcg_cell_bins* bins, vdfcg_cell_results* out,
                               const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                               int64_t* record_offsets, int32_t* cell_begin);

/* Synthetic cell data for tests/bench (counter-based, deterministic per (seed, species,
 * global particle index)): each cell draws from a 2-component mixture whose drift and
 * temperature vary with the global cell index. cell_offsets are GLOBAL particle offsets
 * of cells [cell_base, cell_base + n_cells); particle p is written at p - cell_offsets[0].
 * Device pointers only. */
int vdfcg_synth_cells(vdfcg_ctx* ctx, int32_t dimension, int32_t n_cells,
                      const int64_t* cell_offsets, int64_t cell_base, uint64_t seed,
                      int32_t species, double* velocity_u, double* velocity_v,
                      double* velocity_w);

/* Replaces vdfc::generate (synthdata.hpp / synthdata.cpp:54-86; validation as
 * ScenarioSpec::validate, synthdata.cpp:32-52): the reference's Gaussian-mixture particle
 * generator drawing from the same single mt19937_64(seed) stream (rng.hpp:17-48), on the
 * device. fractions[m], means[m*d], covs[m*d*d] (row-major per component) are host
 * arrays; velocities (n x d column-major = SoA) is a host or device buffer;
 * nominal_temperature[d] (host, may be null). Component choice and stream positions are
 * bit-identical to the reference; values agree to the last few ulp (CUDA's log/sin/cos vs
 * the host libm). Needs (n + 2*ceil(n*d/2)) * 8 bytes of device workspace. */
int vdfcg_generate(vdfcg_ctx* ctx, int32_t dimension, int32_t m, const double* fractions,
                   const double* means, const double* covs, int64_t n, uint64_t seed,
                   double* velocities, double* nominal_temperature);

/* Roofline denominators: FP64 and FP32 FMA throughput of this device, measured with a
 * dependent-chain-free FMA loop on every SM (TFLOP/s, FMA = 2 flops). */
int vdfcg_probe_peaks(vdfcg_ctx* ctx, double* fp64_tflops, double* fp32_tflops);

#ifdef __cplusplus
}
#endif

#endif /* VDFCG_H */
