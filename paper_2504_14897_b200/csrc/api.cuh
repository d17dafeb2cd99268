// api.cuh — internal entry points shared by the C-ABI translation units (not exported).
#pragma once

#include "ctx.cuh"

namespace vdfcg {

// EM launch shape of a sub-batch: the (cells, mean particles per cell) of the batch it is
// part of, so every part runs the launch shape the whole batch would (bitwise-identical
// fits). cells = 0: the sub-batch's own shape.
struct EmShape {
  int cells = 0;
  double avg = 0.0;
};

// vdfcg_compress_cells_warm with an explicit EM launch shape.
int compress_cells_shaped(vdfcg_ctx* ctx, const vdfcg_cells* cells, const vdfcg_fit_config* cfg,
                          const vdfcg_cell_results* warm, vdfcg_cell_bins* bins,
                          vdfcg_cell_results* out, const vdfcg_model_meta* meta, uint8_t* records,
                          int64_t capacity, int64_t* record_offsets, const EmShape& shape);

}  // namespace vdfcg
