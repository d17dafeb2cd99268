// hist.cu — velocity histogram kernels (sm_100a).
//
// K1 hist2d: bin_particles / all_planes (histogram.cpp:45-84). One pass over the
//    particle columns (all three marginals from one read for all_planes), per-CTA
//    shared-memory privatised u32 counters (unit weights: exact integers) merged into
//    global memory with one atomic per non-empty bin, out-of-range mass per CTA.
//    Fractional weights: per-particle bin -> stable device group-by (index.cu) -> every
//    bin summed sequentially in particle order = the reference's `+=`, bit for bit.
// K2 cells_dense: per-cell bins^d histograms for cells much larger than the grid
//    (SURVEY.md App. A), work items = (cell, chunk), shared-memory privatised counters;
//    fractional weights take the ordered composite-id path (cells_weighted_ordered).
// K3 cells_sort: per-cell sort of composite (bin, particle) keys for cells much
//    smaller than the grid (48^3, 64^3): the sorted runs ARE the compacted histogram in
//    ascending bin order (= to_weighted_points(drop_empty) order), and fractional
//    weights are summed in particle order, i.e. bit-identical to the reference's
//    sequential `counts(i,j) += w` (histogram.cpp:70-73).
// K4 compaction of dense grids (histogram.cpp:86-109 order: i outer, j, k inner).
#include <cub/block/block_exchange.cuh>
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <string>

#include "common.cuh"
#include "hist.cuh"

namespace vdfcg {

// ---------------------------------------------------------------------------- K1
struct Hist2dParams {
  int ax[3], ay[3];
  int n_bins;
  double xlo[3], xhi[3], ylo[3], yhi[3], invx[3], invy[3];
};

template <int NP, bool W, bool SMEM>
__global__ void __launch_bounds__(512) hist2d_kernel(const double* __restrict__ vel, int64_t n,
                                                     const double* __restrict__ w, Hist2dParams p,
                                                     unsigned* __restrict__ gcnt,
                                                     double* __restrict__ gcntw,
                                                     unsigned long long* __restrict__ goor,
                                                     double* __restrict__ goorw, int* err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nb = p.n_bins;
  const int nn = nb * nb;
  unsigned* sh = reinterpret_cast<unsigned*>(smem_raw);
  double* shw = reinterpret_cast<double*>(smem_raw);
  if (SMEM) {
    for (int f = threadIdx.x; f < NP * nn; f += blockDim.x) {
      if (W) shw[f] = 0.0; else sh[f] = 0u;
    }
    __syncthreads();
  }
  unsigned long long oor[NP];
  double oorw[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    oor[q] = 0;
    oorw[q] = 0.0;
  }
  bool bad = false;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    double wt = 1.0;
    if (W) {
      wt = __ldg(w + i);
      bad |= !(wt > 0.0);
    }
    // Load each needed axis once (all_planes: u, v, w read once for three planes).
    double v[3];
    int idx[3][2];
#pragma unroll
    for (int a = 0; a < 3; ++a) v[a] = 0.0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const double vx = __ldg(vel + static_cast<int64_t>(p.ax[q]) * n + i);
      const double vy = __ldg(vel + static_cast<int64_t>(p.ay[q]) * n + i);
      idx[q][0] = bin_index(vx, p.xlo[q], p.xhi[q], nb, p.invx[q]);
      idx[q][1] = bin_index(vy, p.ylo[q], p.yhi[q], nb, p.invy[q]);
    }
    (void)v;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int bi = idx[q][0], bj = idx[q][1];
      if (bi < 0 || bj < 0) {
        if (W) oorw[q] += wt; else oor[q] += 1;
      } else {
        const int f = q * nn + bi + bj * nb;  // column-major counts(i, j)
        if (SMEM) {
          if (W) atomicAdd(shw + f, wt); else atomicAdd(sh + f, 1u);
        } else {
          if (W) atomicAdd(gcntw + f, wt); else atomicAdd(gcnt + f, 1u);
        }
      }
    }
  }
  if (W && bad) atomicOr(err, 1);
  if (SMEM) {
    __syncthreads();
    for (int f = threadIdx.x; f < NP * nn; f += blockDim.x) {
      if (W) {
        const double c = shw[f];
        if (c != 0.0) atomicAdd(gcntw + f, c);
      } else {
        const unsigned c = sh[f];
        if (c) atomicAdd(gcnt + f, c);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    if (W) {
      const double s = warp_sum(oorw[q]);
      if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(goorw + q, s);
    } else {
      const unsigned long long s = warp_sum(oor[q]);
      if ((threadIdx.x & 31) == 0 && s) atomicAdd(goor + q, s);
    }
  }
}

__global__ void u32_to_f64_kernel(const unsigned* __restrict__ in, double* __restrict__ out,
                                  int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<double>(in[i]);
}

__global__ void u64_to_f64_kernel(const unsigned long long* in, double* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<double>(in[i]);
}

template <int NP, bool W, bool SMEM>
static void hist2d_dispatch(vdfcg_ctx* ctx, int grid, int block, size_t smem, const double* vel,
                            int64_t n, const double* w, const Hist2dParams& p, unsigned* gcnt,
                            double* gcntw, unsigned long long* goor, double* goorw, int* err) {
  auto k = hist2d_kernel<NP, W, SMEM>;
  if (smem > 48 * 1024)
    VDFCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
  VDFCG_LAUNCH(ctx, "hist2d", k<<<grid, block, smem, ctx->stream>>>(vel, n, w, p, gcnt, gcntw,
                                                                     goor, goorw, err));
}

// Weighted bin_particles / all_planes in the reference's summation order: every bin (and the
// out-of-range total) is the sequential sum `counts(i,j) += w` over the particles in input
// order (histogram.cpp:66-74). Per plane: each particle's column-major bin (or n^2 for out
// of range) -> the stable device group-by (index.cu) puts every bin's weights contiguous in
// particle order -> one thread per bin adds them in that order from 0.0. Bit-identical to
// the reference and run-to-run deterministic (the atomic scatter is neither).
__global__ void plane_bin_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                                 int nb, double xlo, double xhi, double ylo, double yhi, double invx,
                                 double invy, int32_t* __restrict__ bin) {
  const int32_t oor = nb * nb;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int bi = bin_index(__ldg(x + i), xlo, xhi, nb, invx);
    const int bj = bin_index(__ldg(y + i), ylo, yhi, nb, invy);
    bin[i] = (bi < 0 || bj < 0) ? oor : bi + bj * nb;  // column-major counts(i, j)
  }
}

__global__ void ordered_bin_sum_kernel(const double* __restrict__ wg, const int64_t* __restrict__ off,
                                       int32_t nn, double* __restrict__ counts, double* __restrict__ oor) {
  for (int32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= nn; b += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t p = off[b]; p < off[b + 1]; ++p) s = __dadd_rn(s, __ldg(wg + p));
    if (b < nn) counts[b] = s;
    else *oor = s;
  }
}

static void hist2d_weighted_ordered(vdfcg_ctx* ctx, const double* vel, int64_t n, const double* w, int nplanes,
                                    const int* ax, const int* ay, int n_bins, const double* xlo,
                                    const double* xhi, const double* ylo, const double* yhi,
                                    double* counts_out, double* oor_out, int* err) {
  const int32_t nn = n_bins * n_bins;
  int32_t* bin = arena<int32_t>(ctx, size_t(std::max<int64_t>(n, 1)));
  uint32_t* keys = arena<uint32_t>(ctx, size_t(std::max<int64_t>(n, 1)));
  double* wg = arena<double>(ctx, size_t(std::max<int64_t>(n, 1)));
  int64_t* off = arena<int64_t>(ctx, size_t(nn) + 2);
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(ctx->sm_count) * 8)));
  for (int q = 0; q < nplanes; ++q) {
    const double* x = vel + static_cast<int64_t>(ax[q]) * n;
    const double* y = vel + static_cast<int64_t>(ay[q]) * n;
    if (n > 0)
      VDFCG_LAUNCH(ctx, "hist2d_bin",
                   plane_bin_kernel<<<grid, 256, 0, ctx->stream>>>(x, y, n, n_bins, xlo[q], xhi[q], ylo[q], yhi[q],
                                                                   n_bins / (xhi[q] - xlo[q]),
                                                                   n_bins / (yhi[q] - ylo[q]), bin));
    IndexedDev in{};
    in.d = 2;
    in.n = n;
    in.vel[0] = x;
    in.vel[1] = y;
    in.vel[2] = x;
    in.w = w;
    in.cell = bin;
    in.n_cells = nn + 1;  // + the out-of-range bin
    in.n_bins = 2;
    in.lo[0] = in.lo[1] = in.lo[2] = 0.0;
    in.hi[0] = in.hi[1] = in.hi[2] = 1.0;
    launch_group_cells(ctx, in, GroupedDev{keys, wg, off}, err);
    const int g2 = std::max(1, std::min((nn + 256) / 256, ctx->sm_count * 8));
    VDFCG_LAUNCH(ctx, "hist2d_ordered_sum",
                 ordered_bin_sum_kernel<<<g2, 256, 0, ctx->stream>>>(wg, off, nn, counts_out + size_t(q) * nn,
                                                                   oor_out + q));
  }
}

void launch_hist2d(vdfcg_ctx* ctx, const double* vel, int64_t n, int d, const double* w,
                   int nplanes, const int* ax, const int* ay, int n_bins, const double* xlo,
                   const double* xhi, const double* ylo, const double* yhi, double* counts_out,
                   double* oor_out) {
  (void)d;
  Hist2dParams p{};
  p.n_bins = n_bins;
  for (int q = 0; q < nplanes; ++q) {
    p.ax[q] = ax[q];
    p.ay[q] = ay[q];
    p.xlo[q] = xlo[q];
    p.xhi[q] = xhi[q];
    p.ylo[q] = ylo[q];
    p.yhi[q] = yhi[q];
    p.invx[q] = n_bins / (xhi[q] - xlo[q]);  // histogram.cpp:64-65
    p.invy[q] = n_bins / (yhi[q] - ylo[q]);
  }
  const int64_t nn = static_cast<int64_t>(n_bins) * n_bins * nplanes;
  const bool weighted = w != nullptr;
  const size_t elem = weighted ? 8 : 4;
  const size_t smem = static_cast<size_t>(nn) * elem;
  const bool use_smem = smem <= 112 * 1024;
  int* err = arena<int>(ctx, 1);
  VDFCG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
  if (weighted) {  // reference summation order (bit-exact), see hist2d_weighted_ordered
    hist2d_weighted_ordered(ctx, vel, n, w, nplanes, ax, ay, n_bins, xlo, xhi, ylo, yhi, counts_out,
                            oor_out, err);
    int* h = static_cast<int*>(ctx->pinned);
    VDFCG_CUDA(cudaMemcpyAsync(h, err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (*h & 2) throw InvalidArgument("particle weights must all be > 0");
    return;
  }
  unsigned* gcnt = nullptr;
  unsigned long long* goor = nullptr;
  if (weighted) {
    VDFCG_CUDA(cudaMemsetAsync(counts_out, 0, nn * sizeof(double), ctx->stream));
    VDFCG_CUDA(cudaMemsetAsync(oor_out, 0, nplanes * sizeof(double), ctx->stream));
  } else {
    gcnt = arena<unsigned>(ctx, nn);
    goor = arena<unsigned long long>(ctx, nplanes);
    VDFCG_CUDA(cudaMemsetAsync(gcnt, 0, nn * sizeof(unsigned), ctx->stream));
    VDFCG_CUDA(cudaMemsetAsync(goor, 0, nplanes * sizeof(unsigned long long), ctx->stream));
  }
  const int block = 512;
  int per_sm = 1;
  if (use_smem) per_sm = std::max(1, std::min(4, static_cast<int>((200 * 1024) / std::max<size_t>(smem, 1))));
  else per_sm = 4;
  int64_t want = (n + block - 1) / block;
  int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(ctx->sm_count) * per_sm)));
  const size_t sm = use_smem ? smem : 0;
#define VDFCG_H2D(NP)                                                                         \
  if (weighted) {                                                                             \
    if (use_smem) hist2d_dispatch<NP, true, true>(ctx, grid, block, sm, vel, n, w, p, gcnt,   \
                                                  counts_out, goor, oor_out, err);            \
    else hist2d_dispatch<NP, true, false>(ctx, grid, block, sm, vel, n, w, p, gcnt,           \
                                          counts_out, goor, oor_out, err);                    \
  } else {                                                                                    \
    if (use_smem) hist2d_dispatch<NP, false, true>(ctx, grid, block, sm, vel, n, w, p, gcnt,  \
                                                   counts_out, goor, oor_out, err);           \
    else hist2d_dispatch<NP, false, false>(ctx, grid, block, sm, vel, n, w, p, gcnt,          \
                                           counts_out, goor, oor_out, err);                   \
  }
  if (n > 0) {
    if (nplanes == 1) {
      VDFCG_H2D(1)
    } else {
      VDFCG_H2D(3)
    }
  }
#undef VDFCG_H2D
  if (!weighted) {
    const int g2 = static_cast<int>(std::min<int64_t>((nn + 255) / 256, ctx->sm_count * 8));
    VDFCG_LAUNCH(ctx, "hist2d_finalize",
                 u32_to_f64_kernel<<<std::max(g2, 1), 256, 0, ctx->stream>>>(gcnt, counts_out, nn));
    VDFCG_LAUNCH(ctx, "hist2d_finalize",
                 u64_to_f64_kernel<<<1, 32, 0, ctx->stream>>>(goor, oor_out, nplanes));
  }
  if (weighted) {
    int* h = static_cast<int*>(ctx->pinned);
    VDFCG_CUDA(cudaMemcpyAsync(h, err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (*h) throw InvalidArgument("particle weights must all be > 0");
  }
}

// ------------------------------------------------------- to_weighted_points (2D)
__global__ void __launch_bounds__(1024) twp_kernel(const double* __restrict__ counts, int nb,
                                                   double xlo, double xhi, double ylo,
                                                   double yhi, int drop_empty, int64_t capacity,
                                                   double* __restrict__ points,
                                                   double* __restrict__ weights,
                                                   int64_t* count_out, double* total_out) {
  using Reduce = cub::BlockReduce<long long, 1024>;
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Reduce::TempStorage rs;
  __shared__ typename Scan::TempStorage ss;
  __shared__ long long s_kept;
  __shared__ int s_run;
  const int64_t nn = static_cast<int64_t>(nb) * nb;
  // Pass 1: count kept bins; in-range total summed in column-major storage order by
  // one thread (Histogram2D::in_range_count, histogram.hpp:25).
  long long kept = 0;
  double part = 0.0;
  for (int64_t f = threadIdx.x; f < nn; f += blockDim.x) {
    const double c = counts[f];
    kept += (c > 0.0) ? 1 : 0;
    part += c;
  }
  long long tot_kept = Reduce(rs).Sum(kept);
  // in_range_count (Eigen sum(), histogram.hpp:25) in a fixed tree order: exact for integer
  // counts, deterministic for fractional ones
  __shared__ typename cub::BlockReduce<double, 1024>::TempStorage rds;
  const double total = cub::BlockReduce<double, 1024>(rds).Sum(part);
  if (threadIdx.x == 0) {
    s_kept = drop_empty ? tot_kept : nn;
    *total_out = total;
    *count_out = s_kept;
    s_run = 0;
  }
  __syncthreads();
  const int64_t ld = s_kept;
  if (ld > capacity) return;
  // Pass 2: i outer, j inner (histogram.cpp:97-106), ordered compaction per tile.
  for (int64_t base = 0; base < nn; base += blockDim.x) {
    const int64_t f = base + threadIdx.x;  // f = i*nb + j
    double c = 0.0;
    int keep = 0;
    int i = 0, j = 0;
    if (f < nn) {
      i = static_cast<int>(f / nb);
      j = static_cast<int>(f % nb);
      c = counts[i + static_cast<int64_t>(j) * nb];
      keep = (!drop_empty || c > 0.0) ? 1 : 0;
    }
    int pos, total;
    Scan(ss).ExclusiveSum(keep, pos, total);
    const int r = s_run + pos;
    if (keep) {
      points[r] = bin_center(xlo, xhi, nb, i);
      points[ld + r] = bin_center(ylo, yhi, nb, j);
      weights[r] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_run += total;
    __syncthreads();
  }
}

int64_t launch_to_weighted_points(vdfcg_ctx* ctx, const double* counts, int n_bins, double xlo,
                                  double xhi, double ylo, double yhi, bool drop_empty,
                                  int64_t capacity, double* points, double* weights,
                                  double* total_weight_dev) {
  int64_t* cnt = arena<int64_t>(ctx, 1);
  VDFCG_LAUNCH(ctx, "to_weighted_points",
               twp_kernel<<<1, 1024, 0, ctx->stream>>>(counts, n_bins, xlo, xhi, ylo, yhi,
                                                       drop_empty ? 1 : 0, capacity, points,
                                                       weights, cnt, total_weight_dev));
  int64_t* h = static_cast<int64_t*>(ctx->pinned);
  VDFCG_CUDA(cudaMemcpyAsync(h, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  return *h;
}

// ---------------------------------------------------------------------- cells
struct CellGeom {
  int n_bins;
  double lo[3], hi[3], inv[3];
};

struct VelPtrs {
  const double* v[3];
  const uint32_t* keys;  // D == 0: precomputed bin keys (0xffffffff = out of range)
};

// Flat bin key of particle i, -1 when out of range. D == 0 reads a key
// computed upstream (the cell-index path, index.cu) instead of the velocities.
template <int D>
VDFCG_DEV int64_t cell_key(const VelPtrs& vp, int64_t i, const CellGeom& g) {
  if constexpr (D == 0) {
    const uint32_t k = __ldg(vp.keys + i);
    return k == 0xffffffffu ? int64_t(-1) : int64_t(k);
  } else {
    int64_t key = 0;
    bool out = false;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int b = bin_index(__ldg(vp.v[a] + i), g.lo[a], g.hi[a], g.n_bins, g.inv[a]);
      out |= b < 0;
      key = key * g.n_bins + b;
    }
    return out ? -1 : key;
  }
}

// K2: work item = (cell, chunk of `chunk` particles).
template <int D, bool SMEM>
__global__ void __launch_bounds__(1024) cells_dense_kernel(
    VelPtrs vp, const double* __restrict__ w, const int64_t* __restrict__ offsets, int n_cells,
    const int64_t* __restrict__ item_off, int64_t chunk, CellGeom g, int64_t bins,
    unsigned* __restrict__ dense, double* __restrict__ densew,
    unsigned long long* __restrict__ oor_cnt, double* __restrict__ oorw, int* err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned* sh = reinterpret_cast<unsigned*>(smem_raw);
  const int64_t n_items = item_off[n_cells];
  const bool weighted = w != nullptr;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    // cell = last c with item_off[c] <= item
    int lo = 0, hi = n_cells - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (item_off[mid] <= item) lo = mid; else hi = mid - 1;
    }
    const int c = lo;
    const int64_t k = item - item_off[c];
    const int64_t b = offsets[c] + k * chunk;
    const int64_t e = min(offsets[c + 1], b + chunk);
    if (SMEM) {
      for (int64_t f = threadIdx.x; f < bins; f += blockDim.x) sh[f] = 0u;
      __syncthreads();
    }
    unsigned long long oor = 0;
    double ow = 0.0;
    bool bad = false;
    constexpr int U = 4;  // 4 particles per thread in flight: 12 independent 8-byte loads
    for (int64_t i0 = b + threadIdx.x; i0 < e; i0 += int64_t(U) * blockDim.x) {
      int64_t key[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + int64_t(u) * blockDim.x;
        key[u] = i < e ? cell_key<D>(vp, i, g) : -2;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + int64_t(u) * blockDim.x;
        if (key[u] == -2) continue;
        if (weighted) {
          const double wt = __ldg(w + i);
          bad |= !(wt > 0.0);
          if (key[u] < 0) ow += wt;
          else atomicAdd(densew + static_cast<int64_t>(c) * bins + key[u], wt);
        } else {
          if (key[u] < 0) ++oor;
          else if (SMEM) atomicAdd(sh + key[u], 1u);
          else atomicAdd(dense + static_cast<int64_t>(c) * bins + key[u], 1u);
        }
      }
    }
    if (bad) atomicOr(err, 1);
    if (SMEM) {
      __syncthreads();
      for (int64_t f = threadIdx.x; f < bins; f += blockDim.x) {
        const unsigned v = sh[f];
        if (v) atomicAdd(dense + static_cast<int64_t>(c) * bins + f, v);
      }
      __syncthreads();
    }
    if (weighted) {
      const double s = warp_sum(ow);
      if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(oorw + c, s);
    } else {
      const unsigned long long s = warp_sum(oor);
      if ((threadIdx.x & 31) == 0 && s) atomicAdd(oor_cnt + c, s);
    }
  }
}

// K4: ordered compaction of dense per-cell grids into the cell's CSR region.
template <bool W>
__global__ void __launch_bounds__(512) cells_compact_kernel(
    int n_cells, int64_t bins, const unsigned* __restrict__ dense,
    const double* __restrict__ densew, const unsigned long long* __restrict__ oor_cnt,
    const double* __restrict__ oorw, const int64_t* __restrict__ offsets, int32_t* nnz,
    uint32_t* __restrict__ keys, double* __restrict__ counts, double* oor_out, double* in_range) {
  using Scan = cub::BlockScan<int, 512>;
  using Reduce = cub::BlockReduce<unsigned long long, 512>;
  using ReduceD = cub::BlockReduce<double, 512>;
  __shared__ typename Scan::TempStorage ss;
  __shared__ typename Reduce::TempStorage rs;
  __shared__ typename ReduceD::TempStorage rds;
  __shared__ int64_t s_run;
  for (int c = blockIdx.x; c < n_cells; c += gridDim.x) {
    const int64_t base = offsets[c];
    const int64_t cap = offsets[c + 1] - base;
    if (threadIdx.x == 0) s_run = 0;
    __syncthreads();
    unsigned long long tot = 0;
    double totw = 0.0;
    for (int64_t t0 = 0; t0 < bins; t0 += blockDim.x) {
      const int64_t f = t0 + threadIdx.x;
      unsigned v = 0;
      double vw = 0.0;
      if (f < bins) {
        if (W) vw = densew[static_cast<int64_t>(c) * bins + f];
        else v = dense[static_cast<int64_t>(c) * bins + f];
      }
      const int keep = W ? (vw > 0.0) : (v > 0u);
      tot += v;
      totw += vw;
      int pos, total;
      Scan(ss).ExclusiveSum(keep, pos, total);
      const int64_t r = s_run + pos;
      if (keep && r < cap) {
        keys[base + r] = static_cast<uint32_t>(f);
        counts[base + r] = W ? vw : static_cast<double>(v);
      }
      __syncthreads();
      if (threadIdx.x == 0) s_run += total;
      __syncthreads();
    }
    const unsigned long long t = Reduce(rs).Sum(tot);
    __syncthreads();
    const double tw = ReduceD(rds).Sum(totw);
    if (threadIdx.x == 0) {
      nnz[c] = static_cast<int32_t>(s_run);
      oor_out[c] = W ? oorw[c] : static_cast<double>(oor_cnt[c]);
      in_range[c] = W ? tw : static_cast<double>(t);
    }
    __syncthreads();
  }
}

// K3: per-cell composite-key sort. key = (bin << IDXB) | local index; OOR bin = SENT.
// Unit weights sort the bin key alone (counts = run lengths; order within a run is
// irrelevant); fractional weights sort (bin, particle) so each run is summed in particle
// order. CUB's 4-bit digits: 5- and 6-bit digits measured slower at 64^3 (2.06 / 3.09
// vs 1.97 ms per 65536 cells; the wider rank counters cost occupancy).
template <int D, int BLOCK, int IPT, bool W>
__global__ void __launch_bounds__(BLOCK) cells_sort_kernel(
    VelPtrs vp, const double* __restrict__ w, const int64_t* __restrict__ offsets, int n_cells,
    CellGeom g, int binbits, int idxbits, int32_t* nnz, uint32_t* __restrict__ keys_out,
    double* __restrict__ counts_out, double* oor_out, double* in_range, int* err) {
  constexpr int CAP = BLOCK * IPT;
  using Sort = cub::BlockRadixSort<uint32_t, BLOCK, IPT>;
  using Scan = cub::BlockScan<int, BLOCK>;
  using ReduceD = cub::BlockReduce<double, BLOCK>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Exchange = cub::BlockExchange<uint32_t, BLOCK, IPT>;
  auto& sort_ts = *reinterpret_cast<typename Sort::TempStorage*>(smem_raw);
  auto& exch_ts = *reinterpret_cast<typename Exchange::TempStorage*>(smem_raw);
  uint32_t* sk = reinterpret_cast<uint32_t*>(smem_raw);  // reused after the sort
  uint32_t* pos = sk + CAP;                               // run heads [CAP + 1]
  __shared__ typename Scan::TempStorage ss;
  __shared__ typename ReduceD::TempStorage rds;
  __shared__ int s_valid, s_nnz;
  const uint32_t sent = (binbits >= 32) ? 0xffffffffu : ((1u << binbits) - 1u);
  const uint32_t idxmask = (1u << idxbits) - 1u;
  for (int c = blockIdx.x; c < n_cells; c += gridDim.x) {
    const int64_t b = offsets[c];
    const int nc = static_cast<int>(offsets[c + 1] - b);
    uint32_t k[IPT];
    bool bad = false;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int li = i * BLOCK + threadIdx.x;  // striped, coalesced loads
      if (li < nc) {
        const int64_t key = cell_key<D>(vp, b + li, g);
        const uint32_t bin = key < 0 ? sent : static_cast<uint32_t>(key);
        k[i] = W ? ((bin << idxbits) | static_cast<uint32_t>(li)) : bin;
        if (W) bad |= !(__ldg(w + b + li) > 0.0);
      } else {
        k[i] = W ? 0xffffffffu : sent;  // padding sorts with (after) the out-of-range keys
      }
    }
    if (W && bad) atomicOr(err, 1);
    __syncthreads();
    if constexpr (W) {
      // blocked = particle order, so a stable sort on the bin bits alone keeps every
      // bin's particles in order (5 digit passes at 48^3 instead of 7 over bin + index)
      Exchange(exch_ts).StripedToBlocked(k);
      __syncthreads();
      Sort(sort_ts).Sort(k, idxbits, idxbits + binbits);
    } else {
      Sort(sort_ts).Sort(k, 0, binbits);
    }
    __syncthreads();
    // blocked arrangement: thread t holds sorted positions t*IPT + i
#pragma unroll
    for (int i = 0; i < IPT; ++i) sk[threadIdx.x * IPT + i] = k[i];
    __syncthreads();
    int heads = 0, valid = 0;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int p = threadIdx.x * IPT + i;
      if (p < nc) {
        const uint32_t bin = sk[p] >> idxbits;
        if (bin != sent) {
          ++valid;
          if (p == 0 || (sk[p - 1] >> idxbits) != bin) ++heads;
        }
      }
    }
    int hpos, htot;
    Scan(ss).ExclusiveSum(heads, hpos, htot);
    int vtot = 0;
    {
      __syncthreads();
      int vp2;
      Scan(ss).ExclusiveSum(valid, vp2, vtot);
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int p = threadIdx.x * IPT + i;
      if (p < nc) {
        const uint32_t bin = sk[p] >> idxbits;
        if (bin != sent && (p == 0 || (sk[p - 1] >> idxbits) != bin)) pos[hpos++] = p;
      }
    }
    if (threadIdx.x == 0) {
      s_nnz = htot;
      s_valid = vtot;
      pos[htot] = vtot;
    }
    __syncthreads();
    const int nz = s_nnz;
    double part = 0.0;
    for (int r = threadIdx.x; r < nz; r += BLOCK) {
      const int p0 = pos[r], p1 = pos[r + 1];
      double v;
      if (W) {
        v = 0.0;  // particle order within the run: exact reference summation
        for (int p = p0; p < p1; ++p) v += __ldg(w + b + (sk[p] & idxmask));
      } else {
        v = static_cast<double>(p1 - p0);
      }
      keys_out[b + r] = sk[p0] >> idxbits;
      counts_out[b + r] = v;
      part += v;
    }
    double tw = 0.0;
    if (W) tw = ReduceD(rds).Sum(part);
    if (threadIdx.x == 0) {
      nnz[c] = nz;
      if (W) {
        double o = 0.0;
        for (int p = s_valid; p < nc; ++p) o += __ldg(w + b + (sk[p] & idxmask));
        oor_out[c] = o;
        in_range[c] = tw;
      } else {
        oor_out[c] = static_cast<double>(nc - s_valid);
        in_range[c] = static_cast<double>(s_valid);
      }
    }
    __syncthreads();
  }
}

// K3b: sparse unit-weight cells without sorting. A shared-memory occupancy bitmap over
// the cell's bins^d grid (1 bit per bin), a block prefix of per-word popcounts gives
// every occupied bin its rank in ascending key order (= to_weighted_points order), a
// second pass counts particles per rank, and set bits are emitted in order. Cost per
// cell: bins/32 words + 2 shared atomics per particle; particles are read once.
template <int D, int BLOCK>
__global__ void __launch_bounds__(BLOCK) cells_bitmap_kernel(
    VelPtrs vp, const int64_t* __restrict__ offsets, int n_cells, CellGeom g, int words, int ccap,
    int cap, int32_t* nnz, uint32_t* __restrict__ keys_out, double* __restrict__ counts_out,
    double* oor_out, double* in_range) {
  using Scan = cub::BlockScan<unsigned, BLOCK>;
  __shared__ typename Scan::TempStorage ss;
  __shared__ unsigned s_oor;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned* bitmap = reinterpret_cast<unsigned*>(smem_raw);  // [words]
  unsigned* wpre = bitmap + words;                           // [words] exclusive prefix
  unsigned* cnt = wpre + words;                              // [ccap >= max nnz] per-rank counts
  unsigned* kbuf = cnt + ccap;                               // [cap] keys of this cell
  const int wpt = (words + BLOCK - 1) / BLOCK;
  // bitmap and counters start zero and are re-zeroed by the emit phase of every cell
  for (int t = threadIdx.x; t < words; t += BLOCK) bitmap[t] = 0u;
  for (int t = threadIdx.x; t < ccap; t += BLOCK) cnt[t] = 0u;
  if (threadIdx.x == 0) s_oor = 0u;
  __syncthreads();
  for (int c = blockIdx.x; c < n_cells; c += gridDim.x) {
    const int64_t b = offsets[c];
    const int nc = static_cast<int>(offsets[c + 1] - b);
    // 1. occupancy bits (8 particles = 24 independent loads in flight per thread)
    unsigned oor = 0;
    constexpr int U = 8;
    for (int l0 = threadIdx.x; l0 < nc; l0 += U * BLOCK) {
      int64_t key[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int li = l0 + u * BLOCK;
        key[u] = li < nc ? cell_key<D>(vp, b + li, g) : -2;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int li = l0 + u * BLOCK;
        if (key[u] == -2) continue;
        if (key[u] < 0) ++oor;
        else atomicOr(bitmap + (key[u] >> 5), 1u << (key[u] & 31));
        if (li < cap) kbuf[li] = key[u] < 0 ? 0xffffffffu : static_cast<unsigned>(key[u]);
      }
    }
    oor = warp_sum(oor);
    if ((threadIdx.x & 31) == 0 && oor) atomicAdd(&s_oor, oor);
    __syncthreads();
    // 2. rank of every occupied bin = exclusive prefix of per-word popcounts
    unsigned local = 0;
    for (int k = 0; k < wpt; ++k) {
      const int wi = threadIdx.x * wpt + k;
      if (wi < words) local += __popc(bitmap[wi]);
    }
    unsigned pre, total;
    Scan(ss).ExclusiveSum(local, pre, total);
    for (int k = 0; k < wpt; ++k) {
      const int wi = threadIdx.x * wpt + k;
      if (wi < words) {
        wpre[wi] = pre;
        pre += __popc(bitmap[wi]);
      }
    }
    __syncthreads();
    // 3. count per rank; each particle writes its bin key at its rank (duplicates write
    //    the same value), so keys come out in ascending order without an emit loop
    for (int li = threadIdx.x; li < nc; li += BLOCK) {
      unsigned key;
      if (li < cap) {
        key = kbuf[li];
      } else {
        const int64_t k2 = cell_key<D>(vp, b + li, g);
        key = k2 < 0 ? 0xffffffffu : static_cast<unsigned>(k2);
      }
      if (key != 0xffffffffu) {
        const unsigned wd = key >> 5, bit = key & 31;
        const unsigned r = wpre[wd] + __popc(bitmap[wd] & ((1u << bit) - 1u));
        atomicAdd(cnt + r, 1u);
        keys_out[b + r] = key;
      }
    }
    __syncthreads();
    // 4. coalesced emit of the counts; re-zero counters and bitmap for the next cell
    for (unsigned r = threadIdx.x; r < total; r += BLOCK) {
      counts_out[b + r] = static_cast<double>(cnt[r]);
      cnt[r] = 0u;
    }
    for (int t = threadIdx.x; t < words; t += BLOCK) bitmap[t] = 0u;
    if (threadIdx.x == 0) {
      const unsigned to = s_oor;
      nnz[c] = static_cast<int32_t>(total);
      oor_out[c] = static_cast<double>(to);
      in_range[c] = static_cast<double>(nc - static_cast<int>(to));
      s_oor = 0u;
    }
    __syncthreads();
  }
}

// K3c: K3b with the particle loads moved to the Tensor Memory Accelerator. Phase 1 of
// cell c reads u/v/w from shared memory; right after it, one thread issues three 1-D
// bulk copies (cp.async.bulk, completion counted on an mbarrier) of the NEXT cell's axis
// slices into the same buffer, so the HBM reads of cell c+grid overlap the rank / count
// / emit phases of cell c and no warp waits on global-load latency. Slices are widened
// to 16-byte boundaries (bulk-copy granularity); `skew` locates the cell inside them.
// D == 0 stages the cell's precomputed u32 bin keys instead (cell-index path).
VDFCG_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

VDFCG_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

VDFCG_DEV void bar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

VDFCG_DEV void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Stage cell c's axis slices (D == 0: its precomputed u32 keys). Axis a's base address is
// `sh[a]` elements past a 16-byte boundary (an Eigen N x 3 column of odd N starts 8 bytes
// off), so element x is 16-byte aligned iff (x + sh[a]) % A == 0, A = 16 / element size.
// The staged window is [B, E) with B = floor_A(b + sh) - sh, E = ceil_A(e + sh) - sh, kept
// at pbuf[a][x - B] (skew b - B); the part a bulk copy may not touch — before element 0 or
// past element lim-1 (lim = offsets[n_cells]) — is loaded by this thread directly.
template <int D>
struct Stage {
  static constexpr int kArrays = D == 0 ? 1 : D;
  static constexpr int kElem = D == 0 ? 4 : 8;
  static constexpr int kA = 16 / kElem;
};

// Every array 16-byte aligned (sh == 0): the window starts at the even (D > 0) / 4-aligned
// (keys) element at or below b; only an element past lim-1 at the very end is loaded directly.
template <int D>
VDFCG_DEV void issue_cell_copy_aligned(const VelPtrs& vp, const int64_t* offsets, int c, int64_t lim,
                                       unsigned char* pbuf, int capp, uint64_t* bar) {
  using S = Stage<D>;
  constexpr int A = S::kA;
  const int64_t b = offsets[c], e = offsets[c + 1];
  const int64_t b0 = b & ~int64_t(A - 1);
  int64_t e0 = (e + A - 1) & ~int64_t(A - 1);
  int64_t ed = e0;  // directly loaded tail [ed, e)
  if (e0 > lim) {
    e0 -= A;
    ed = e0;
  }
  const uint32_t bytes = e0 > b0 ? static_cast<uint32_t>((e0 - b0) * S::kElem) : 0u;
  for (int64_t x = ed; x < e; ++x) {
#pragma unroll
    for (int a = 0; a < S::kArrays; ++a) {
      if constexpr (D == 0)
        reinterpret_cast<uint32_t*>(pbuf)[x - b0] = __ldg(vp.keys + x);
      else
        reinterpret_cast<double*>(pbuf)[a * capp + (x - b0)] = __ldg(vp.v[a] + x);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  bar_expect(bar, bytes * S::kArrays);
  if (bytes)
#pragma unroll
    for (int a = 0; a < S::kArrays; ++a) {
      if constexpr (D == 0)
        bulk_g2s(reinterpret_cast<uint32_t*>(pbuf), vp.keys + b0, bytes, bar);
      else
        bulk_g2s(reinterpret_cast<double*>(pbuf) + a * capp, vp.v[a] + b0, bytes, bar);
    }
}

template <int D>
VDFCG_DEV void issue_cell_copy(const VelPtrs& vp, const int64_t* offsets, int c, int64_t lim,
                               unsigned char* pbuf, int capp, const int* sh, uint64_t* bar) {
  using S = Stage<D>;
  constexpr int A = S::kA;
  const int64_t b = offsets[c], e = offsets[c + 1];
  uint32_t total = 0;
  int64_t bb[S::kArrays], ee[S::kArrays], B[S::kArrays];
#pragma unroll
  for (int a = 0; a < S::kArrays; ++a) {
    B[a] = ((b + sh[a]) / A) * A - sh[a];
    const int64_t E = ((e + sh[a] + A - 1) / A) * A - sh[a];
    bb[a] = B[a] < 0 ? B[a] + A : B[a];
    ee[a] = E > lim ? E - A : E;
    if (ee[a] < bb[a]) ee[a] = bb[a];
    // direct loads of [b, e) outside the bulk window [bb, ee)
    for (int64_t x = b; x < e; ++x) {
      if (x >= bb[a] && x < ee[a]) {
        x = ee[a] - 1;
        continue;
      }
      if constexpr (D == 0)
        reinterpret_cast<uint32_t*>(pbuf)[x - B[a]] = __ldg(vp.keys + x);
      else
        reinterpret_cast<double*>(pbuf)[a * capp + (x - B[a])] = __ldg(vp.v[a] + x);
    }
    total += static_cast<uint32_t>((ee[a] - bb[a]) * S::kElem);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  bar_expect(bar, total);
#pragma unroll
  for (int a = 0; a < S::kArrays; ++a) {
    const uint32_t bytes = static_cast<uint32_t>((ee[a] - bb[a]) * S::kElem);
    if (!bytes) continue;
    if constexpr (D == 0)
      bulk_g2s(reinterpret_cast<uint32_t*>(pbuf) + (bb[a] - B[a]), vp.keys + bb[a], bytes, bar);
    else
      bulk_g2s(reinterpret_cast<double*>(pbuf) + a * capp + (bb[a] - B[a]), vp.v[a] + bb[a], bytes, bar);
  }
}

struct StageShift {
  int sh[3];
};

template <int D, int BLOCK, int kTmaWpt, bool GEN, int MINB, bool PK = false, int GW = 1>  // kTmaWpt >=
// bitmap words per thread; GEN: some array base is not 16-byte aligned (per-array skew),
// else the aligned fast form; MINB: CTAs per SM the shared memory allows (3 caps registers
// at 40 for 512 threads: small bitmaps run three CTAs, larger ones two with more
// registers); PK: per-rank counts packed as u16 pairs (a staged cell has < 2^16
// particles) — only where the 2 bytes per rank saved make room for a third CTA (32^3:
// 0.567 -> 0.628 of HBM); elsewhere the shift/mask costs ~2%. GW = 4: one exclusive prefix
// per 4-word group (a rank adds the popcounts of the group's earlier words, read as one
// 16-byte load), so a 64^3 bitmap's prefix array shrinks 4x and two CTAs fit per SM
__global__ void __launch_bounds__(BLOCK) __maxnreg__(MINB == 3 ? 40 : GW == 4 ? 64 : 48) cells_bitmap_tma_kernel(
    VelPtrs vp, const int64_t* __restrict__ offsets, int n_cells, CellGeom g, int words, int ccap,
    int capp, StageShift ss_, int32_t* nnz, uint32_t* __restrict__ keys_out,
    double* __restrict__ counts_out, double* oor_out, double* in_range) {
  using Scan = cub::BlockScan<unsigned, BLOCK>;
  __shared__ typename Scan::TempStorage ss;
  __shared__ unsigned s_oor;
  __shared__ __align__(8) uint64_t bar;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using S = Stage<D>;
  unsigned char* pbuf = smem_raw;                                        // [arrays][capp]
  unsigned* bitmap = reinterpret_cast<unsigned*>(pbuf + size_t(S::kArrays) * capp * S::kElem);
  unsigned* wpre = bitmap + words;                                       // [words / GW]
  const int cw = PK ? (ccap + 1) >> 1 : ccap;
  unsigned* cnt2 = wpre + (words + GW - 1) / GW;                         // [cw]
  unsigned* kbuf = cnt2 + cw;                                            // [capp]
  unsigned* keyr = kbuf + capp;                                          // [ccap] key of rank r
  unsigned short* cnt16 = reinterpret_cast<unsigned short*>(cnt2);
  const int wpt = (words + BLOCK - 1) / BLOCK;
  // GW = 4: word w lives at w ^ ((w >> 5) & 15) — thread t's k-th prefix word 16t + k then
  // hits 32 distinct banks across a warp (a plain stride of 16 words is a 16-way conflict)
#ifndef VDFCG_HIST_NOSWZ
  auto swz = [](unsigned w) { return GW == 4 ? (w ^ ((w >> 5) & 15u)) : w; };
#else  // measurement variant only (tools/build_variant.sh hist.cu -DVDFCG_HIST_NOSWZ)
  auto swz = [](unsigned w) { return w; };
#endif
  const int64_t lim = offsets[n_cells];
  for (int t = threadIdx.x; t < words; t += BLOCK) bitmap[t] = 0u;
  for (int t = threadIdx.x; t < cw; t += BLOCK) cnt2[t] = 0u;
  if (threadIdx.x == 0) {
    s_oor = 0u;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x < n_cells) {
      if constexpr (GEN) issue_cell_copy<D>(vp, offsets, blockIdx.x, lim, pbuf, capp, ss_.sh, &bar);
      else issue_cell_copy_aligned<D>(vp, offsets, blockIdx.x, lim, pbuf, capp, &bar);
    }
  }
  __syncthreads();
  uint32_t parity = 0;
  for (int c = blockIdx.x; c < n_cells; c += gridDim.x) {
    const int64_t b = offsets[c];
    const int nc = static_cast<int>(offsets[c + 1] - b);
    int skew[S::kArrays];
#pragma unroll
    for (int a = 0; a < S::kArrays; ++a)
      skew[a] = GEN ? static_cast<int>((b + ss_.sh[a]) % S::kA) : static_cast<int>(b & (S::kA - 1));
    bar_wait(&bar, parity);
    parity ^= 1u;
    // 1. occupancy bits from the staged slices
    unsigned oor = 0;
    for (int li = threadIdx.x; li < nc; li += BLOCK) {
      int64_t key = 0;
      bool out = false;
      if constexpr (D == 0) {
        const uint32_t k = reinterpret_cast<const uint32_t*>(pbuf)[skew[0] + li];
        out = k == 0xffffffffu;
        key = k;
      } else {
        const double* pb = reinterpret_cast<const double*>(pbuf);
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const int bi = bin_index(pb[a * capp + skew[a] + li], g.lo[a], g.hi[a], g.n_bins, g.inv[a]);
          out |= bi < 0;
          key = key * g.n_bins + bi;
        }
      }
      if (out) {
        ++oor;
        kbuf[li] = 0xffffffffu;
      } else {
        atomicOr(bitmap + swz(static_cast<unsigned>(key >> 5)), 1u << (key & 31));
        kbuf[li] = static_cast<unsigned>(key);
      }
    }
    oor = warp_sum(oor);
    if ((threadIdx.x & 31) == 0 && oor) atomicAdd(&s_oor, oor);
    __syncthreads();
    // the staging buffer is free: fetch the next cell while this one is ranked
    if (threadIdx.x == 0 && c + static_cast<int>(gridDim.x) < n_cells)
    {
      if constexpr (GEN) issue_cell_copy<D>(vp, offsets, c + gridDim.x, lim, pbuf, capp, ss_.sh, &bar);
      else issue_cell_copy_aligned<D>(vp, offsets, c + gridDim.x, lim, pbuf, capp, &bar);
    }
    // 2. ranks; the word popcounts stay in registers for the prefix and the re-zeroing
    unsigned local = 0, pc[kTmaWpt];
#pragma unroll
    for (int k = 0; k < kTmaWpt; ++k) {
      const int wi = threadIdx.x * wpt + k;
      pc[k] = (k < wpt && wi < words) ? __popc(bitmap[swz(wi)]) : 0u;
      local += pc[k];
    }
    unsigned pre, total;
    Scan(ss).ExclusiveSum(local, pre, total);
#pragma unroll
    for (int k = 0; k < kTmaWpt; ++k) {
      if constexpr (GW == 1) {
        if (pc[k]) wpre[threadIdx.x * wpt + k] = pre;  // only occupied words are ever read
      } else {  // wpt is a multiple of GW (host): groups never straddle threads
        if (k % GW == 0 && k < wpt && threadIdx.x * wpt + k < words) wpre[(threadIdx.x * wpt + k) / GW] = pre;
      }
      pre += pc[k];
    }
    __syncthreads();
    // 3. counts per rank; each rank's key goes to shared memory (the scattered global
    //    stores of the key per particle cost ~10% of the kernel), emitted coalesced below
    for (int li = threadIdx.x; li < nc; li += BLOCK) {
      const unsigned key = kbuf[li];
      if (key != 0xffffffffu) {
        const unsigned wd = key >> 5, bit = key & 31;
        unsigned r;
        if constexpr (GW == 1) {
          r = wpre[wd] + __popc(bitmap[wd] & ((1u << bit) - 1u));
        } else {
          static_assert(GW == 4, "4-word groups");
          // the group's 4 words sit in one swizzled 16-byte slot, slot p holding word p ^ s3
          const unsigned sx = swz(wd) ^ wd, s3 = sx & 3u;  // the swizzle of this row
          const uint4 q = reinterpret_cast<const uint4*>(bitmap)[((wd & ~3u) ^ (sx & 12u)) >> 2];
          const unsigned j = wd & 3u, lt = (1u << bit) - 1u;
          auto msk = [&](unsigned p) { const unsigned l = p ^ s3; return l < j ? ~0u : l == j ? lt : 0u; };
          r = wpre[wd >> 2] + __popc(q.x & msk(0)) + __popc(q.y & msk(1)) + __popc(q.z & msk(2)) +
              __popc(q.w & msk(3));
        }
        if constexpr (PK) atomicAdd(cnt2 + (r >> 1), 1u << ((r & 1u) << 4));
        else atomicAdd(cnt2 + r, 1u);
        keyr[r] = key;  // duplicates store the same value
      }
    }
    __syncthreads();
    // 4. emit counts, re-zero
    for (unsigned r = threadIdx.x; r < total; r += BLOCK) {  // coalesced keys + counts
      keys_out[b + r] = keyr[r];
      if constexpr (PK) {
        counts_out[b + r] = static_cast<double>(cnt16[r]);
        cnt16[r] = 0;
      } else {
        counts_out[b + r] = static_cast<double>(cnt2[r]);
        cnt2[r] = 0u;
      }
    }
#pragma unroll
    for (int k = 0; k < kTmaWpt; ++k)
      if (pc[k]) bitmap[swz(threadIdx.x * wpt + k)] = 0u;
    if (threadIdx.x == 0) {
      const unsigned to = s_oor;
      nnz[c] = static_cast<int32_t>(total);
      oor_out[c] = static_cast<double>(to);
      in_range[c] = static_cast<double>(nc - static_cast<int>(to));
      s_oor = 0u;
    }
    __syncthreads();
  }
}

__global__ void chunks_per_cell_kernel(const int64_t* offsets, int n_cells, int64_t chunk,
                                       int64_t* out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += gridDim.x * blockDim.x) {
    const int64_t nc = offsets[c + 1] - offsets[c];
    out[c] = (nc + chunk - 1) / chunk;
  }
}

// Exclusive scan of n int64 values, total at out[n]: one CTA walking 4096-element tiles with
// coalesced loads and a running prefix (n = cells of a batch).
__global__ void __launch_bounds__(1024) scan_i64_kernel(const int64_t* in, int64_t* out, int64_t n) {
  using Scan = cub::BlockScan<long long, 1024>;
  __shared__ typename Scan::TempStorage ss;
  __shared__ long long s_run;
  if (threadIdx.x == 0) s_run = 0;
  __syncthreads();
  for (int64_t t0 = 0; t0 < n; t0 += 4096) {
    long long x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t k = t0 + threadIdx.x + i * 1024;  // coalesced
      x[i] = k < n ? in[k] : 0;
    }
    // thread t owns elements t, t+1024, ...: four block scans in (i, t) order
    long long run = s_run;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      long long pre, tot;
      Scan(ss).ExclusiveSum(x[i], pre, tot);
      const int64_t k = t0 + threadIdx.x + i * 1024;
      if (k < n) out[k] = run + pre;
      run += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) s_run = run;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = s_run;
}

void launch_scan_i64(vdfcg_ctx* ctx, const int64_t* in, int64_t* out, int64_t n) {
  VDFCG_LAUNCH(ctx, "scan", scan_i64_kernel<<<1, 1024, 0, ctx->stream>>>(in, out, n));
}

__global__ void max_cell_kernel(const int64_t* offsets, int n_cells, unsigned long long* out) {
  unsigned long long m = 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += gridDim.x * blockDim.x)
    m = max(m, static_cast<unsigned long long>(offsets[c + 1] - offsets[c]));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

int64_t max_cell_size(vdfcg_ctx* ctx, const int64_t* offsets, int n_cells) {
  unsigned long long* d = arena<unsigned long long>(ctx, 1);
  VDFCG_CUDA(cudaMemsetAsync(d, 0, 8, ctx->stream));
  const int grid = std::max(1, std::min((n_cells + 255) / 256, ctx->sm_count * 4));
  VDFCG_LAUNCH(ctx, "max_cell", max_cell_kernel<<<grid, 256, 0, ctx->stream>>>(offsets, n_cells, d));
  auto* h = static_cast<unsigned long long*>(ctx->pinned);
  VDFCG_CUDA(cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  return static_cast<int64_t>(*h);
}

static int bits_for(uint64_t v) {  // smallest b with 2^b > v
  int b = 0;
  while (b < 64 && (uint64_t(1) << b) <= v) ++b;
  return b;
}

template <int D, int BLOCK, int IPT, bool W>
static void launch_sort(vdfcg_ctx* ctx, const CellsDev& c, const CellBinsDev& out,
                        const CellGeom& g, int binbits, int* err) {
  using Sort = cub::BlockRadixSort<uint32_t, BLOCK, IPT>;
  constexpr int CAP = BLOCK * IPT;
  const size_t smem = std::max({sizeof(typename Sort::TempStorage),
                                sizeof(typename cub::BlockExchange<uint32_t, BLOCK, IPT>::TempStorage),
                                size_t(2 * CAP + 2) * 4});
  auto k = cells_sort_kernel<D, BLOCK, IPT, W>;
  VDFCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int occ = 0;
  VDFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, BLOCK, smem));
  const int grid = std::max(1, std::min(c.n_cells, ctx->sm_count * std::max(occ, 1)));
  const int idxbits = W ? bits_for(CAP - 1) : 0;
  VelPtrs vp{{c.vel[0], c.vel[1], c.vel[2]}, c.keys};
  VDFCG_LAUNCH(ctx, "cells_sort",
               k<<<grid, BLOCK, smem, ctx->stream>>>(vp, c.w, c.offsets, c.n_cells, g, binbits,
                                                     idxbits, out.nnz, out.keys, out.counts,
                                                     out.oor, out.in_range, err));
}

template <int D, bool W>
static bool try_sort_path(vdfcg_ctx* ctx, const CellsDev& c, const CellBinsDev& out,
                          const CellGeom& g, int binbits, int64_t maxc, int* err) {
  auto fits = [&](int cap) { return maxc <= cap && binbits + bits_for(cap - 1) <= 32; };
  if (fits(1024)) launch_sort<D, 128, 8, W>(ctx, c, out, g, binbits, err);
  else if (fits(2048)) launch_sort<D, 256, 8, W>(ctx, c, out, g, binbits, err);
  else if (fits(4096)) launch_sort<D, 256, 16, W>(ctx, c, out, g, binbits, err);
  else if (fits(8192)) launch_sort<D, 512, 16, W>(ctx, c, out, g, binbits, err);
  else return false;
  return true;
}

// Weighted cells too large for the per-cell sort (> 8192 particles): every (cell, bin) sum
// in particle order (histogram.cpp:66-74) through the stable device group-by over the
// composite id c * (bins + 1) + bin (bins = the cell's out-of-range slot); then one thread
// per id adds its weights sequentially into the dense per-cell grid the compaction reads.
__global__ void fill_i32_kernel(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

template <int D>
__global__ void cell_composite_kernel(VelPtrs vp, const int64_t* __restrict__ offsets, int n_cells,
                                      CellGeom g, int64_t bins, int32_t* __restrict__ ids) {
  for (int c = blockIdx.x; c < n_cells; c += gridDim.x) {
    const int64_t b = offsets[c], e = offsets[c + 1];
    const int64_t base = static_cast<int64_t>(c) * (bins + 1);
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      const int64_t key = cell_key<D>(vp, i, g);
      ids[i] = static_cast<int32_t>(base + (key < 0 ? bins : key));
    }
  }
}

__global__ void composite_sum_kernel(const double* __restrict__ wg, const int64_t* __restrict__ off,
                                     int64_t n_ids, int64_t bins, double* __restrict__ densew,
                                     double* __restrict__ oorw) {
  for (int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; id < n_ids;
       id += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p0 = off[id], p1 = off[id + 1];
    double s = 0.0;
    for (int64_t p = p0; p < p1; ++p) s = __dadd_rn(s, __ldg(wg + p));
    const int64_t c = id / (bins + 1), k = id - c * (bins + 1);
    if (k == bins) oorw[c] = s;
    else densew[c * bins + k] = s;
  }
}

template <int D>
static void cells_weighted_ordered(vdfcg_ctx* ctx, const CellsDev& c, const CellGeom& g, int64_t bins,
                                   double* densew, double* oorw, int* err) {
  const int64_t n_ids = int64_t(c.n_cells) * (bins + 1);
  const int64_t n = std::max<int64_t>(c.n, 1);
  int32_t* ids = arena<int32_t>(ctx, size_t(n));
  uint32_t* keys = arena<uint32_t>(ctx, size_t(n));
  double* wg = arena<double>(ctx, size_t(n));
  int64_t* off = arena<int64_t>(ctx, size_t(n_ids) + 2);
  const int g1 = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(ctx->sm_count) * 8)));
  // particles outside every cell range get the extra id n_ids (grouped, never summed)
  VDFCG_LAUNCH(ctx, "cells_ordered_ids",
               fill_i32_kernel<<<g1, 256, 0, ctx->stream>>>(ids, c.n, static_cast<int32_t>(n_ids)));
  VelPtrs vp{{c.vel[0], c.vel[1], c.vel[2]}, c.keys};
  const int gc = std::max(1, std::min(c.n_cells, ctx->sm_count * 8));
  VDFCG_LAUNCH(ctx, "cells_ordered_ids",
               cell_composite_kernel<D><<<gc, 512, 0, ctx->stream>>>(vp, c.offsets, c.n_cells, g, bins, ids));
  IndexedDev in{};
  in.d = 2;
  in.n = c.n;
  in.vel[0] = in.vel[1] = in.vel[2] = c.w;  // read-only dummy: the group keys are not used
  in.w = c.w;
  in.cell = ids;
  in.n_cells = static_cast<int>(n_ids + 1);
  in.n_bins = 2;
  in.lo[0] = in.lo[1] = in.lo[2] = 0.0;
  in.hi[0] = in.hi[1] = in.hi[2] = 1.0;
  launch_group_cells(ctx, in, GroupedDev{keys, wg, off}, err);
  const int g2 = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n_ids + 255) / 256, int64_t(ctx->sm_count) * 16)));
  VDFCG_LAUNCH(ctx, "cells_ordered_sum",
               composite_sum_kernel<<<g2, 256, 0, ctx->stream>>>(wg, off, n_ids, bins, densew, oorw));
}

// D = velocity axes read by the kernels, or 0 when the bin keys were computed upstream
// (c.keys, the cell-index path); the grid dimension is c.d either way.
template <int D>
static void bin_cells_d(vdfcg_ctx* ctx, const CellsDev& c, const CellBinsDev& out) {
  CellGeom g{};
  g.n_bins = c.n_bins;
  int64_t bins = 1;
  for (int a = 0; a < c.d; ++a) {
    g.lo[a] = c.lo[a];
    g.hi[a] = c.hi[a];
    g.inv[a] = c.n_bins / (c.hi[a] - c.lo[a]);
    bins *= c.n_bins;
  }
  const bool weighted = c.w != nullptr;
  int* err = arena<int>(ctx, 1);
  VDFCG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
  const int64_t maxc = c.max_cell >= 0 ? c.max_cell : max_cell_size(ctx, c.offsets, c.n_cells);
  const double avg = c.n_cells ? double(c.n) / c.n_cells : 0.0;
  const int binbits = bits_for(static_cast<uint64_t>(bins));  // SENT = 2^binbits - 1 > any bin
  // Sparse cells: unit weights use the occupancy bitmap (no sort); fractional weights
  // use the composite-key sort, which sums every bin in particle order (bit-exact).
  bool done = false;
  const bool sparse = avg * 4.0 < double(bins) || maxc <= 1024;
  const int64_t words = (bins + 31) / 32;
  const int64_t ccap = std::max<int64_t>(1, std::min<int64_t>(maxc, bins));  // >= every nnz
  const int64_t kcap = std::min<int64_t>(maxc, 4096);
  // TMA-staged variant: the staging window (largest cell + up to 16 bytes of widening at
  // each end per array) fits beside the bitmap. Bases need only element alignment: the
  // kernel carries each array's offset from a 16-byte boundary (Eigen N x 3 columns).
  using S = Stage<D>;
  const int64_t capp = ((maxc + 2 * (S::kA - 1) + S::kA - 1) / S::kA) * S::kA;
  const size_t tma_smem_pk = size_t(S::kArrays) * capp * S::kElem + size_t(words) * 8 +
                             size_t((ccap + 1) / 2) * 4 + size_t(ccap) * 4 + size_t(capp) * 4;
  size_t tma_smem = tma_smem_pk + size_t(ccap) * 4 - size_t((ccap + 1) / 2) * 4;
  bool aligned = true;
  StageShift shift{};
  for (int a = 0; a < S::kArrays; ++a) {
    const uintptr_t addr = D == 0 ? reinterpret_cast<uintptr_t>(c.keys) : reinterpret_cast<uintptr_t>(c.vel[a]);
    aligned = aligned && (addr % S::kElem) == 0;
    shift.sh[a] = static_cast<int>((addr % 16) / S::kElem);
  }
  static const int tma_env = [] {
    const char* e = getenv("VDFCG_HIST_TMA");  // 0: off, 1: 512-thread CTAs, 2: 256
    return e ? atoi(e) : 1;
  }();
  // path override for measurements: VDFCG_HIST_PATH = tma | bitmap | sort | dense
  static const int path_env = [] {
    const char* e = getenv("VDFCG_HIST_PATH");
    if (!e) return 0;
    const std::string v(e);
    return v == "tma" ? 1 : v == "bitmap" ? 2 : v == "sort" ? 3 : v == "dense" ? 4 : 0;
  }();
  const int tb = tma_env == 2 ? 256 : 512;
  const bool tma_fits = aligned && tma_env && tma_smem <= 220 * 1024 && words <= 16 * tb && maxc < 65536;
  // Unit weights, measured on 65536 cells (tools: exp-style sweeps recorded in DESIGN.md):
  // the TMA bitmap kernel whenever it fits two CTAs per SM (1907 particles/cell,
  // 16^3..48^3: 0.74-1.0 ms, 6x the dense path at 16^3), or one CTA per SM with a bitmap of
  // <= 4096 words (6000/cell, 16^3..32^3: 2.6-3.0 ms vs 6-18 ms dense); else the plain
  // bitmap kernel for bitmaps of <= 4096 words (6000/cell at 48^3: 4.5 ms vs 11.5 sort);
  // 64^3 (1907/cell): TMA with 4-word prefix groups at two CTAs/SM 1.44 ms vs 1.97 sort,
  // 2.4 one-CTA TMA, 7.6 bitmap; larger cells at 64^3 take the radix sort.
  const bool bitmap_fits = words * 8 + ccap * 4 + kcap * 4 <= 160 * 1024;
  // 4-word prefix groups when only they bring a large bitmap (64^3) to two CTAs per SM
  // (the swizzle permutes words within aligned 16-word blocks: the bitmap is padded to a
  // multiple of 16 words, the padding never set)
  const int64_t words16 = (words + 15) & ~int64_t(15);
  const size_t tma_smem_gw = tma_smem - size_t(words) * 8 + size_t(words16) * 4 + size_t(words16 / 4) * 4;
  const bool gw4 = tb == 512 && words16 > 8 * 512 && ((words16 + 511) / 512) % 4 == 0 &&
                   tma_smem > 110 * 1024 && tma_smem_gw <= 110 * 1024;
  int kwords = static_cast<int>(words);
  int choice = path_env;
  if (choice == 0 && !weighted) {
    if (tma_fits && (tma_smem <= 110 * 1024 || gw4)) choice = 1;
    else if (tma_fits && words <= 4096) choice = 1;
    else if (sparse && bitmap_fits && words <= 4096) choice = 2;
    else if (maxc <= 8192 && sparse) choice = 3;
  }
  if (!weighted && tma_fits && choice == 1) {
    const bool w8 = words <= 8 * tb;
    bool gen = false;
    for (int a = 0; a < S::kArrays; ++a) gen = gen || shift.sh[a] != 0;
    const bool three = tma_smem * 3 + 3 * 1024 <= 227 * 1024;
    const bool three_pk = !three && tma_smem_pk * 3 + 3 * 1024 <= 227 * 1024;
    if (three_pk) tma_smem = tma_smem_pk;
    using KFn = void (*)(VelPtrs, const int64_t*, int, CellGeom, int, int, int, StageShift, int32_t*,
                         uint32_t*, double*, double*, double*);
    KFn k;
#define VDFCG_TMA_PICK(B, WPT)                                                                     \
  k = gen ? (three ? cells_bitmap_tma_kernel<D, B, WPT, true, 3>                                  \
                   : three_pk ? cells_bitmap_tma_kernel<D, B, WPT, true, 3, true>                  \
                              : cells_bitmap_tma_kernel<D, B, WPT, true, 1>)                       \
          : (three ? cells_bitmap_tma_kernel<D, B, WPT, false, 3>                                 \
                   : three_pk ? cells_bitmap_tma_kernel<D, B, WPT, false, 3, true>                 \
                              : cells_bitmap_tma_kernel<D, B, WPT, false, 1>)
    if (gw4) {
      tma_smem = tma_smem_gw;
      kwords = static_cast<int>(words16);
      k = gen ? cells_bitmap_tma_kernel<D, 512, 16, true, 1, false, 4>
              : cells_bitmap_tma_kernel<D, 512, 16, false, 1, false, 4>;
    } else if (tb == 512) {
      if (w8) VDFCG_TMA_PICK(512, 8);
      else VDFCG_TMA_PICK(512, 16);
    } else {
      if (w8) VDFCG_TMA_PICK(256, 8);
      else VDFCG_TMA_PICK(256, 16);
    }
#undef VDFCG_TMA_PICK
    VDFCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tma_smem)));
    int occ = 0;
    VDFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, tb, tma_smem));
    const int grid = std::max(1, std::min(c.n_cells, ctx->sm_count * std::max(occ, 1)));
    VelPtrs vp{{c.vel[0], c.vel[1], c.vel[2]}, c.keys};
    VDFCG_LAUNCH(ctx, "cells_bitmap_tma",
                 k<<<grid, tb, tma_smem, ctx->stream>>>(vp, c.offsets, c.n_cells, g, kwords,
                                                        static_cast<int>(ccap), static_cast<int>(capp), shift,
                                                        out.nnz, out.keys, out.counts, out.oor, out.in_range));
    done = true;
  }
  if (!done && !weighted && bitmap_fits && (choice == 2 || (choice == 0 && sparse))) {
    const int cap = static_cast<int>(std::max<int64_t>(kcap, 1));
    const size_t smem = size_t(words) * 8 + size_t(ccap) * 4 + size_t(cap) * 4;
    auto k = cells_bitmap_kernel<D, 256>;
    VDFCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int occ = 0;
    VDFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, smem));
    const int grid = std::max(1, std::min(c.n_cells, ctx->sm_count * std::max(occ, 1)));
    VelPtrs vp{{c.vel[0], c.vel[1], c.vel[2]}, c.keys};
    VDFCG_LAUNCH(ctx, "cells_bitmap",
                 k<<<grid, 256, smem, ctx->stream>>>(vp, c.offsets, c.n_cells, g, static_cast<int>(words),
                                                     static_cast<int>(ccap), cap, out.nnz, out.keys, out.counts, out.oor,
                                                     out.in_range));
    done = true;
  }
  if (!done && maxc <= 8192 && (weighted || choice == 3 || (choice == 0 && sparse))) {
    done = weighted ? try_sort_path<D, true>(ctx, c, out, g, binbits, maxc, err)
                    : try_sort_path<D, false>(ctx, c, out, g, binbits, maxc, err);
  }
  if (!done) {
    // Dense per-cell grids (global scratch), shared-memory privatised when they fit.
    unsigned* dense = nullptr;
    double* densew = nullptr;
    unsigned long long* oor_cnt = nullptr;
    double* oorw = nullptr;
    const int64_t total_bins = bins * c.n_cells;
    if (weighted) {
      densew = arena<double>(ctx, total_bins);
      oorw = arena<double>(ctx, c.n_cells);
      VDFCG_CUDA(cudaMemsetAsync(densew, 0, total_bins * 8, ctx->stream));
      VDFCG_CUDA(cudaMemsetAsync(oorw, 0, c.n_cells * 8, ctx->stream));
    } else {
      dense = arena<unsigned>(ctx, total_bins);
      oor_cnt = arena<unsigned long long>(ctx, c.n_cells);
      VDFCG_CUDA(cudaMemsetAsync(dense, 0, total_bins * 4, ctx->stream));
      VDFCG_CUDA(cudaMemsetAsync(oor_cnt, 0, c.n_cells * 8, ctx->stream));
    }
    const bool ordered = weighted && int64_t(c.n_cells) * (bins + 1) + 1 < (int64_t(1) << 31) &&
                         c.n < (int64_t(1) << 32);
    if (ordered) {  // reference summation order (bit-exact), see cells_weighted_ordered
      cells_weighted_ordered<D>(ctx, c, g, bins, densew, oorw, err);
    } else {
    const bool smem_ok = !weighted && bins * 4 <= 160 * 1024;
    const int block = 1024;
    // chunk: enough items to fill every SM several times, >= 16K particles each
    int64_t chunk = std::max<int64_t>(16384, (c.n + int64_t(ctx->sm_count) * 4 - 1) /
                                                 (int64_t(ctx->sm_count) * 4));
    if (smem_ok) chunk = std::max<int64_t>(chunk, bins * 2);
    int64_t* cpc = arena<int64_t>(ctx, c.n_cells);
    int64_t* item_off = arena<int64_t>(ctx, c.n_cells + 1);
    VDFCG_LAUNCH(ctx, "cells_items",
                 chunks_per_cell_kernel<<<std::max(1, std::min((c.n_cells + 255) / 256, 1024)), 256, 0,
                                          ctx->stream>>>(c.offsets, c.n_cells, chunk, cpc));
    launch_scan_i64(ctx, cpc, item_off, c.n_cells);
    const int64_t est_items = (c.n + chunk - 1) / chunk + c.n_cells;
    VelPtrs vp{{c.vel[0], c.vel[1], c.vel[2]}, c.keys};
    if (smem_ok) {
      const size_t smem = static_cast<size_t>(bins) * 4;
      auto k = cells_dense_kernel<D, true>;
      VDFCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      int occ = 0;
      VDFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, block, smem));
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(est_items, int64_t(ctx->sm_count) * std::max(occ, 1))));
      VDFCG_LAUNCH(ctx, "cells_dense",
                   k<<<grid, block, smem, ctx->stream>>>(vp, c.w, c.offsets, c.n_cells, item_off,
                                                         chunk, g, bins, dense, densew, oor_cnt,
                                                         oorw, err));
    } else {
      auto k = cells_dense_kernel<D, false>;
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(est_items, int64_t(ctx->sm_count) * 2)));
      VDFCG_LAUNCH(ctx, "cells_dense",
                   k<<<grid, block, 0, ctx->stream>>>(vp, c.w, c.offsets, c.n_cells, item_off,
                                                      chunk, g, bins, dense, densew, oor_cnt, oorw,
                                                      err));
    }
    }
    const int grid = std::max(1, std::min(c.n_cells, ctx->sm_count * 4));
    if (weighted)
      VDFCG_LAUNCH(ctx, "cells_compact",
                   cells_compact_kernel<true><<<grid, 512, 0, ctx->stream>>>(
                       c.n_cells, bins, dense, densew, oor_cnt, oorw, c.offsets, out.nnz, out.keys,
                       out.counts, out.oor, out.in_range));
    else
      VDFCG_LAUNCH(ctx, "cells_compact",
                   cells_compact_kernel<false><<<grid, 512, 0, ctx->stream>>>(
                       c.n_cells, bins, dense, densew, oor_cnt, oorw, c.offsets, out.nnz, out.keys,
                       out.counts, out.oor, out.in_range));
  }
  if (weighted) {
    int* h = static_cast<int*>(ctx->pinned);
    VDFCG_CUDA(cudaMemcpyAsync(h, err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (*h) throw InvalidArgument("particle weights must all be > 0");
  }
}

void launch_bin_cells(vdfcg_ctx* ctx, const CellsDev& c, const CellBinsDev& out) {
  if (c.n_cells == 0) return;
  if (c.keys) bin_cells_d<0>(ctx, c, out);
  else if (c.d == 2) bin_cells_d<2>(ctx, c, out);
  else bin_cells_d<3>(ctx, c, out);
}

}  // namespace vdfcg
