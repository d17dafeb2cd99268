// em.cuh — batched weighted-EM fitter (wgmm.cpp:364-423 per cell) launchers.
#pragma once

#include "ctx.cuh"

namespace vdfcg {

// Per-fit frame produced by a prologue (normalize + init inputs), wgmm.cpp:78-100,136-191.
struct Frame {
  double offset[3], scale[3], zlo[3], zhi[3], temp[3];
  double total;      // points.total_weight
  double err_value;  // value printed in the zero-spread message
  int32_t m_init;    // min(M, distinct points)
  int32_t status;    // VDFCG_* of the prologue
  int32_t err_axis;  // axis of a zero-spread error, or a message id
  int32_t pad;
};

// Prologue error ids carried in Frame::err_axis when status != 0.
enum PrologueMsg {
  kMsgZeroSpread = 0,       // "degenerate data: axis a has zero spread (all values x)"
  kMsgEmpty = 100,          // "weighted points: empty"
  kMsgNegWeight = 101,      // "weighted points: weights must be >= 0"
  kMsgNoPosWeight = 102,    // "weighted points: at least one weight must be > 0"
  kMsgTemperature = 103,    // "temperature must be a positive per-axis variance"
  kMsgDegenerateHist = 104, // "degenerate histogram: no in-range weight"
  kMsgAllDegenerate = 200,  // "all mixture components are degenerate"
  kMsgInvalidMass = 201,    // "m_step: invalid responsibility mass"
};

struct EmConfig {
  int M;
  int max_it;
  double prune_thr;
  int interval;
  double tol;
  int has_temp;
  double temp[3];
  int warm_m;               // 0: random init
  const double* warm_w;     // canonical warm model (device)
  const double* warm_mu;
  const double* warm_cov;
  const double* uniforms;   // [16*3] mt19937_64(seed) uniforms (device)
  unsigned long long* exact_counter;  // optional diagnostics: exact second passes run
  int f32;                  // FP32 E-step with FP64 accumulation (cells path; tolerance 1e-4)
  // Per-cell warm start (time series, pipeline.cpp:482-564): cell c starts from its own
  // canonical model when cell_warm_m[c] > 0 (else the seeded random init). Device arrays
  // with component stride cell_warm_K.
  const int32_t* cell_warm_m;
  const double* cell_warm_w;
  const double* cell_warm_mu;
  const double* cell_warm_cov;
  int cell_warm_K;
};


struct EmOut {
  int K;
  int trace_cap;
  int32_t* status;
  int32_t* comps;
  int32_t* iters;
  int32_t* conv;
  double* w;
  double* mu;
  double* cov;
  double* final_ll;
  double* trace;
  int32_t* n_events;
  int32_t* ev_it;
  int32_t* ev_comp;
  double* ev_w;
  int32_t* err_axis;   // optional [n_cells]
  double* err_value;   // optional [n_cells]
};

struct KeyCells {
  int n_cells;
  const int64_t* offsets;  // region start of each cell's compacted bins
  const int32_t* nnz;
  const uint32_t* keys;
  const double* counts;
  const double* in_range;
  uint32_t* packed;        // scratch [n_particles]: decoded bin indices (device)
  int n_bins;
  double lo[3], hi[3];
  int cluster = 1;         // CTAs per cell (thread-block cluster) when few, large cells
};

struct CoordArgs {
  const double* z;  // SoA normalized points [D][n]
  int64_t n;
  const double* w;
  const Frame* frame;
};

// uniforms[0..n) = mt19937_64(seed) top-53-bit doubles (rng.hpp:22), on the device.
void launch_mt_uniforms(vdfcg_ctx* ctx, uint64_t seed, int n, double* out);

// cell_warm_m[c] = previous status[c] == 0 ? previous components[c] : 0 (device).
void launch_warm_m(vdfcg_ctx* ctx, int n_cells, const int32_t* status, const int32_t* comps,
                   int32_t* m);

// Fit every cell of a compacted histogram batch.
// avg_particles: mean particles per cell (bounds the points per fit for the launch shape);
// shape_fits: number of fits the shape is chosen for (0 = kc.n_cells). Chunked calls pass
// the whole batch's figures so every chunk runs the launch shape the whole batch would.
void launch_em_cells(vdfcg_ctx* ctx, int d, const KeyCells& kc, const EmConfig& cfg,
                     const EmOut& out, double avg_particles, int shape_fits = 0);

// Fit one set of explicit points (N x d column-major, data space) — vdfcg_fit.
void launch_em_points(vdfcg_ctx* ctx, int d, const double* pts, const double* w, int64_t n,
                      double total_weight, const EmConfig& cfg, const EmOut& out);

// normalize + validation + bounding box of z + temperature + distinct count (one CTA).
void launch_fit_prologue(vdfcg_ctx* ctx, int d, const double* pts, const double* w, int64_t n,
                         double total_weight, const EmConfig& cfg, double* z, Frame* fr);

// Canonicalise a warm-start model (denormalize if it carries a map), device buffers.
void launch_canonicalize(vdfcg_ctx* ctx, int d, int m, const double* w, const double* mu,
                         const double* cov, const double* scale, const double* offset,
                         double* ow, double* omu, double* ocov);

std::string prologue_message(int status, int err_axis, double err_value, bool fit_prefix);

}  // namespace vdfcg
