// hist.cuh — histogram kernels (declarations of the host-side launchers).
#pragma once

#include "ctx.cuh"

namespace vdfcg {

// 2D marginal histograms over one pass (bin_particles: 1 plane; all_planes: 3 planes).
// vel: N x d column-major device array. counts_out: nplanes * n^2 doubles, column-major
// per plane. oor_out: nplanes doubles. Throws InvalidArgument on a non-positive weight.
void launch_hist2d(vdfcg_ctx* ctx, const double* vel, int64_t n, int d, const double* w,
                   int nplanes, const int* ax, const int* ay, int n_bins, const double* xlo,
                   const double* xhi, const double* ylo, const double* yhi, double* counts_out,
                   double* oor_out);

// to_weighted_points on a column-major n x n count grid (device). Returns the count.
int64_t launch_to_weighted_points(vdfcg_ctx* ctx, const double* counts, int n_bins, double xlo,
                                  double xhi, double ylo, double yhi, bool drop_empty,
                                  int64_t capacity, double* points, double* weights,
                                  double* total_weight_dev);

// Cell batch histogram + compaction (all pointers device).
struct CellsDev {
  int d;
  int64_t n;
  const double* vel[3];
  const double* w;
  int n_cells;
  const int64_t* offsets;
  int n_bins;
  double lo[3], hi[3];
  int64_t max_cell = -1;   // largest cell, when the host already knows it (else computed)
  int shape_cells = 0;     // EM launch shape from the whole batch when > 0 (chunked calls)
  double shape_avg = 0.0;
  const uint32_t* keys = nullptr;  // precomputed bin keys (cell-index path): vel unused
};
struct CellBinsDev {
  int32_t* nnz;
  uint32_t* keys;
  double* counts;
  double* oor;
  double* in_range;
};
void launch_bin_cells(vdfcg_ctx* ctx, const CellsDev& c, const CellBinsDev& out);

// Cell-index input (index.cu): particles in any order with an int32 cell id each.
struct IndexedDev {
  int d;
  int64_t n;  // < 2^32
  const double* vel[3];
  const double* w;
  const int32_t* cell;
  int n_cells;
  int n_bins;
  double lo[3], hi[3];
};
// Stable group-by-cell: keys (u32 bin key per particle, 0xffffffff = out of range) and
// weights in cell order, offsets[n_cells+1]. err |= 1 on a cell id outside [0, n_cells),
// |= 2 on a weight that is not > 0.
struct GroupedDev {
  uint32_t* keys;
  double* w;
  int64_t* offsets;
};
void launch_group_cells(vdfcg_ctx* ctx, const IndexedDev& in, const GroupedDev& out, int* err);

// Exclusive scan of n int64 values (device), total written to out[n].
void launch_scan_i64(vdfcg_ctx* ctx, const int64_t* in, int64_t* out, int64_t n);
// max over cells of (off[c+1]-off[c]) (device -> host, synchronizes).
int64_t max_cell_size(vdfcg_ctx* ctx, const int64_t* offsets, int n_cells);

}  // namespace vdfcg
