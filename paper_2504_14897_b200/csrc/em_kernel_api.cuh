// em_kernel_api.cuh — per-dimension EM launch entry points (em_d2.cu, em_d3.cu).
#pragma once

#include "em.cuh"

namespace vdfcg {
void launch_em_dim2(vdfcg_ctx* ctx, bool keys, int K, const KeyCells& kc, const CoordArgs& ca,
                    const EmConfig& cfg, const EmOut& out, int n_cells, int G, int n_bins);
void launch_em_dim3(vdfcg_ctx* ctx, bool keys, int K, const KeyCells& kc, const CoordArgs& ca,
                    const EmConfig& cfg, const EmOut& out, int n_cells, int G, int n_bins);
}  // namespace vdfcg
