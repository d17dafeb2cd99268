// em_d3.cu — instantiations of the fused EM kernel for d = 3 velocity axes.
#include "em_kernel.cuh"
#include "em_kernel_api.cuh"

namespace vdfcg {
void launch_em_dim3(vdfcg_ctx* ctx, bool keys, int K, const KeyCells& kc, const CoordArgs& ca,
                    const EmConfig& cfg, const EmOut& out, int n_cells, int G, int n_bins) {
  if (keys) launch_em_k<3, true>(ctx, K, kc, ca, cfg, out, n_cells, G, n_bins);
  else launch_em_k<3, false>(ctx, K, kc, ca, cfg, out, n_cells, G, n_bins);
}
}  // namespace vdfcg
