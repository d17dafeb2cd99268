// index.cu — per-particle cell-index input (sm_100a).
//
// BASELINE north_star: the histogrammer "streams particle (u,v,w) and cell-index arrays".
// Particles arrive in any order with an int32 cell id each (a PIC particle array); the
// reference's only fan-out of one particle set into parts is split_subdomains
// (pipeline.cpp:76-104), each part then binned and fitted on its own (fit_one_plane,
// pipeline.cpp:130-160, 340-345). Here the grouping is a STABLE least-significant-digit
// radix sort over the cell id whose first pass also computes every particle's bin key
// (histogram.cpp:36-41), so the velocities are read exactly once and only
// (cell u32, key u32 [, weight f64]) items move between passes:
//
//   pass p, digit = cell bits [p*RB, (p+1)*RB):
//     ix_upsweep    CTA q counts the digits of its contiguous particle range (SMEM
//                   privatised) -> hist[digit][q]
//     scan          exclusive scan of hist in digit-major order = the first output slot of
//                   every (digit, CTA) pair
//     ix_downsweep  CTA q walks its range tile by tile (8192 items, warp-striped loads);
//                   a block match-rank (warp match.any + per-warp SMEM digit counters, one
//                   scan over (digit, warp)) gives every item its stable rank inside the
//                   tile; items are exchanged through shared memory into rank order and
//                   written out in contiguous runs per digit (u64 (cell, key) items)
//   ix_offsets      cell boundaries of the final cell array -> CSR offsets[n_cells+1]
//
// Stability keeps each cell's particles in input order, so fractional weights are summed in
// the order of the reference's sequential `counts(i,j) += w` (histogram.cpp:66-74) by the
// per-cell sort path. The grouped keys then go through the same per-cell kernels as the
// pre-grouped path (hist.cu, D == 0: keys instead of velocities).
//
// Algorithmic bytes per particle: d*8 + 4 (+8 weight) read. Moved bytes: pass 1
// reads 4 (upsweep) + d*8 + 4 (+8) and writes 8 (+8); every later pass reads 4 + 8 (+8) and
// writes 8 (+8); the offsets kernel reads 4; the per-cell binning reads 4 (+8).
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "common.cuh"
#include "hist.cuh"

namespace vdfcg {
namespace {

constexpr int kIxBlock = 512;
constexpr int kIxIpt = 8;
constexpr int kIxTile = kIxBlock * kIxIpt;  // 4096 items, two CTAs per SM
constexpr int kIxWarps = kIxBlock / 32;

struct IxGeom {
  int n_bins;
  double lo[3], hi[3], inv[3];
};

// Item sources / destinations. Between passes an item is one u64 (cell << 32 | key), so a
// digit run is one contiguous stream; the last pass writes keys and cells as u32 arrays.
struct IxSrc {
  const double* v[3];
  const double* w;
  const int32_t* cell_in;      // first pass: the caller's int32 cell ids
  const uint64_t* items;       // later passes: the previous pass's output
  const double* ws;
};

struct IxDst {
  uint64_t* items;  // non-last passes
  uint32_t* cells;  // last pass
  uint32_t* keys;   // last pass
  double* w;
};

// err bits: 1 = cell id outside [0, n_cells), 2 = weight not > 0
template <int D>
VDFCG_DEV uint32_t particle_key(const IxSrc& s, int64_t i, const IxGeom& g) {
  uint32_t key = 0;
  bool out = false;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int b = bin_index(__ldg(s.v[a] + i), g.lo[a], g.hi[a], g.n_bins, g.inv[a]);
    out |= b < 0;
    key = key * static_cast<uint32_t>(g.n_bins) + static_cast<uint32_t>(b);
  }
  return out ? 0xffffffffu : key;
}

VDFCG_DEV uint32_t checked_cell(int32_t c, int n_cells, bool& bad) {
  const bool ok = c >= 0 && c < n_cells;
  bad |= !ok;
  return ok ? static_cast<uint32_t>(c) : 0u;  // invalid ids are reported, and kept in range
}

constexpr int kUpBlock = 512;

constexpr int kUpSplit = 4;  // upsweep CTAs per downsweep CTA range (the ranges are long)

// hist must be zeroed: CTA (q, s) counts quarter s of CTA q's range and adds into hist[d][q].
template <int RB, bool FIRST>
__global__ void __launch_bounds__(kUpBlock) ix_upsweep(IxSrc s, int64_t n, int64_t per, int n_cells,
                                                        int shift, uint32_t* __restrict__ hist, int* err) {
  constexpr int DIG = 1 << RB;
  __shared__ uint32_t h[DIG];
  for (int t = threadIdx.x; t < DIG; t += kUpBlock) h[t] = 0u;
  __syncthreads();
  const int q = blockIdx.x / kUpSplit, part = blockIdx.x % kUpSplit;
  const int nq = gridDim.x / kUpSplit;
  const int64_t sub = per / kUpSplit;
  const int64_t b = static_cast<int64_t>(q) * per + part * sub;
  const int64_t e = min(n, min(static_cast<int64_t>(q) * per + per, b + sub + (part == kUpSplit - 1 ? per - kUpSplit * sub : 0)));
  bool bad = false;
  constexpr int U = 8;
  for (int64_t i0 = b + threadIdx.x; i0 < e; i0 += int64_t(U) * kUpBlock) {
    uint32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + int64_t(u) * kUpBlock;
      c[u] = 0xffffffffu;
      if (i < e)
        c[u] = FIRST ? checked_cell(__ldg(s.cell_in + i), n_cells, bad)
                     : static_cast<uint32_t>(__ldg(s.items + i) >> 32);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] != 0xffffffffu) atomicAdd(&h[(c[u] >> shift) & (DIG - 1)], 1u);
  }
  if (FIRST && bad) atomicOr(err, 1);
  __syncthreads();
  for (int t = threadIdx.x; t < DIG; t += kUpBlock)
    if (h[t]) atomicAdd(hist + static_cast<int64_t>(t) * nq + q, h[t]);
}

VDFCG_DEV uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Stable rank of every tile item by digit. Tile order is warp-striped (item i of lane l in
// warp w is element w*32*IPT + i*32 + l), ranks are digit-major, then that order: each warp
// ranks its 512 items against per-warp SMEM digit counters with match.any (one counter
// update per distinct digit per 32 items), then one scan over (digit, warp) turns the
// per-warp counts into tile positions. tstart[d] = first tile position of digit d.
template <int RB>
VDFCG_DEV void tile_rank(const uint32_t (&cell)[kIxIpt], int shift, uint32_t (&rank)[kIxIpt],
                         uint32_t* wcnt /*[WARPS][DIG]*/, uint32_t* tstart /*[DIG+1]*/,
                         uint32_t* s_tot /*[BLOCK/32 + 1]*/) {
  constexpr int DIG = 1 << RB;
  constexpr int DPT = DIG >= kIxBlock ? DIG / kIxBlock : 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    uint4* w4 = reinterpret_cast<uint4*>(wcnt);
    for (int t = threadIdx.x; t < kIxWarps * DIG / 4; t += kIxBlock) w4[t] = make_uint4(0u, 0u, 0u, 0u);
  }
  __syncthreads();
  uint32_t* my = wcnt + warp * DIG;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kIxIpt; ++i) {
    const uint32_t d = (cell[i] >> shift) & (DIG - 1);
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = my[d];
    __syncwarp();
    if ((peers & lt) == 0) my[d] = before + __popc(peers);
    __syncwarp();
    rank[i] = before + __popc(peers & lt);
  }
  __syncthreads();
  // exclusive scan over (digit, warp): thread t owns digits [t*DPT, t*DPT + DPT)
  uint32_t tot = 0;
  const bool owns = threadIdx.x * DPT < DIG;
  if (owns) {
#pragma unroll
    for (int k = 0; k < DPT; ++k) {
      const int d = threadIdx.x * DPT + k;
#pragma unroll
      for (int w = 0; w < kIxWarps; ++w) {
        const uint32_t c = wcnt[w * DIG + d];
        wcnt[w * DIG + d] = tot;
        tot += c;
      }
    }
  }
  // block exclusive scan of the per-thread totals (warp shuffles + one SMEM pass)
  uint32_t incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t x = lane < kIxWarps ? s_tot[lane] : 0u;
    uint32_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    if (lane < kIxWarps) s_tot[lane] = xi - x;  // exclusive warp offsets
  }
  __syncthreads();
  const uint32_t base = s_tot[warp] + incl - tot;  // exclusive prefix of this thread's digits
  if (owns) {
#pragma unroll
    for (int k = 0; k < DPT; ++k) {
      const int d = threadIdx.x * DPT + k;
      // wcnt holds the exclusive prefix within this thread's digits: rebase it; warp 0's
      // entry is the digit's first tile position
      tstart[d] = base + wcnt[d];
#pragma unroll
      for (int w = 0; w < kIxWarps; ++w) wcnt[w * DIG + d] += base;
    }
  }
  if (threadIdx.x == 0) tstart[DIG] = kIxTile;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kIxIpt; ++i) {
    const uint32_t d = (cell[i] >> shift) & (DIG - 1);
    rank[i] += wcnt[warp * DIG + d];
  }
}

template <int D, int RB, bool FIRST, bool LAST, bool W>
__global__ void __launch_bounds__(kIxBlock, 2) ix_downsweep(IxSrc s, int64_t n, int64_t per, int n_cells,
                                                                     IxGeom g, int shift,
                                                                     const uint32_t* __restrict__ base, IxDst dst,
                                                                     int* err) {
  constexpr int DIG = 1 << RB;
  __shared__ uint32_t run[DIG];
  __shared__ uint32_t tstart[DIG + 1];
  __shared__ uint32_t s_tot[kIxWarps + 1];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* s_item = reinterpret_cast<uint64_t*>(smem_raw);            // [TILE]
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(s_item + kIxTile);      // [WARPS * DIG]
  double* s_w = reinterpret_cast<double*>(wcnt + kIxWarps * DIG);      // [W ? TILE : 0]
  for (int t = threadIdx.x; t < DIG; t += kIxBlock) run[t] = base[static_cast<int64_t>(t) * gridDim.x + blockIdx.x];
  const int64_t b = static_cast<int64_t>(blockIdx.x) * per;
  const int64_t e = min(n, b + per);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int bad = 0;
  for (int64_t t0 = b; t0 < e; t0 += kIxTile) {
    const int valid = static_cast<int>(e - t0 < kIxTile ? e - t0 : int64_t(kIxTile));
    uint32_t cell[kIxIpt], key[kIxIpt];
    double wt[W ? kIxIpt : 1];
#pragma unroll
    for (int i = 0; i < kIxIpt; ++i) {
      const int j = warp * 32 * kIxIpt + i * 32 + lane;
      cell[i] = 0xffffffffu;  // padding: digit DIG-1, ranks after every real item
      key[i] = 0xffffffffu;
      if (W) wt[i] = 0.0;
      if (j < valid) {
        const int64_t x = t0 + j;
        if (FIRST) {
          bool bc = false;
          cell[i] = checked_cell(__ldg(s.cell_in + x), n_cells, bc);
          bad |= bc ? 1 : 0;
          key[i] = particle_key<D>(s, x, g);
          if (W) {
            wt[i] = __ldg(s.w + x);
            if (!(wt[i] > 0.0)) bad |= 2;
          }
        } else {
          const uint64_t it = __ldg(s.items + x);
          cell[i] = static_cast<uint32_t>(it >> 32);
          key[i] = static_cast<uint32_t>(it);
          if (W) wt[i] = __ldg(s.ws + x);
        }
      }
    }
    uint32_t rank[kIxIpt];
    __syncthreads();  // previous tile: shared buffers and run[] are free
    tile_rank<RB>(cell, shift, rank, wcnt, tstart, s_tot);
#pragma unroll
    for (int i = 0; i < kIxIpt; ++i) {
      if (rank[i] < static_cast<uint32_t>(valid)) {
        s_item[rank[i]] = (static_cast<uint64_t>(cell[i]) << 32) | key[i];
        if (W) s_w[rank[i]] = wt[i];
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < valid; r += kIxBlock) {
      const uint64_t it = s_item[r];
      const uint32_t c = static_cast<uint32_t>(it >> 32);
      const uint32_t d = (c >> shift) & (DIG - 1);
      const uint32_t pos = run[d] + static_cast<uint32_t>(r) - tstart[d];
      if (LAST) {
        dst.cells[pos] = c;
        dst.keys[pos] = static_cast<uint32_t>(it);
      } else {
        dst.items[pos] = it;
      }
      if (W) dst.w[pos] = s_w[r];
    }
    __syncthreads();
    for (int d = threadIdx.x; d < DIG; d += kIxBlock)
      run[d] += min(tstart[d + 1], static_cast<uint32_t>(valid)) - min(tstart[d], static_cast<uint32_t>(valid));
  }
  if (FIRST && bad) atomicOr(err, bad);
}

// Exclusive scan of n u32 values in place (n = digits x CTAs, a few 100K): one CTA, tiles of
// 4096 with a running prefix.
__global__ void __launch_bounds__(1024) ix_scan_u32(uint32_t* v, int64_t n) {
  using Scan = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename Scan::TempStorage ss;
  __shared__ uint32_t s_run;
  if (threadIdx.x == 0) s_run = 0u;
  __syncthreads();
  for (int64_t t0 = 0; t0 < n; t0 += 4096) {
    uint32_t x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t k = t0 + threadIdx.x * 4 + i;
      x[i] = k < n ? v[k] : 0u;
    }
    uint32_t tot;
    Scan(ss).ExclusiveSum(x, x, tot);
    const uint32_t r = s_run;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t k = t0 + threadIdx.x * 4 + i;
      if (k < n) v[k] = x[i] + r;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_run = r + tot;
    __syncthreads();
  }
}

// CSR offsets from the cell-sorted ids: the cells in (cells[p-1], cells[p]] start at p.
// Four consecutive positions per thread (one 16-byte load when aligned).
__global__ void ix_offsets(const uint32_t* __restrict__ cells, int64_t n, int n_cells, int64_t* off) {
  const int64_t groups = n / 4 + 1;  // group g covers positions 4g .. 4g+3 (and p = n)
  for (int64_t gi = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; gi < groups;
       gi += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p0 = gi * 4;
    int64_t v[5];
    v[0] = p0 > 0 ? static_cast<int64_t>(__ldg(cells + p0 - 1)) : -1;
    if (p0 + 4 <= n) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(cells + p0));
      v[1] = q.x;
      v[2] = q.y;
      v[3] = q.z;
      v[4] = q.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k + 1] = p0 + k < n ? static_cast<int64_t>(__ldg(cells + p0 + k)) : n_cells;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (p0 + k > n) break;
      for (int64_t x = v[k] + 1; x <= v[k + 1]; ++x) off[x] = p0 + k;
    }
  }
}

template <int D, int RB, bool FIRST, bool LAST, bool W>
size_t downsweep_smem() {
  return size_t(kIxTile) * 8 + size_t(kIxWarps) * (1 << RB) * 4 + (W ? size_t(kIxTile) * 8 : 0);
}

template <int D, int RB, bool FIRST, bool LAST, bool W>
void run_pass(vdfcg_ctx* ctx, const IxSrc& src, const IxDst& dst, int64_t n, int grid, int64_t per,
              int n_cells, const IxGeom& g, int shift, uint32_t* hist, int* err) {
  constexpr int DIG = 1 << RB;
  VDFCG_CUDA(cudaMemsetAsync(hist, 0, size_t(DIG) * grid * sizeof(uint32_t), ctx->stream));
  VDFCG_LAUNCH(ctx, "group_upsweep",
               (ix_upsweep<RB, FIRST><<<grid * kUpSplit, kUpBlock, 0, ctx->stream>>>(src, n, per, n_cells, shift,
                                                                                       hist, err)));
  VDFCG_LAUNCH(ctx, "group_scan", ix_scan_u32<<<1, 1024, 0, ctx->stream>>>(hist, int64_t(DIG) * grid));
  const size_t smem = downsweep_smem<D, RB, FIRST, LAST, W>();
  auto k = ix_downsweep<FIRST ? D : 0, RB, FIRST, LAST, W>;
  VDFCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  VDFCG_LAUNCH(ctx, "group_downsweep",
               k<<<grid, kIxBlock, smem, ctx->stream>>>(src, n, per, n_cells, g, shift, hist, dst, err));
}

template <int D, int RB, bool W>
void group_impl(vdfcg_ctx* ctx, const IndexedDev& in, int passes, const GroupedDev& out, int* err) {
  constexpr int DIG = 1 << RB;
  const int64_t n = in.n;
  IxGeom g{};
  g.n_bins = in.n_bins;
  for (int a = 0; a < D; ++a) {
    g.lo[a] = in.lo[a];
    g.hi[a] = in.hi[a];
    g.inv[a] = in.n_bins / (in.hi[a] - in.lo[a]);  // histogram.cpp:64-65
  }
  const size_t smem = downsweep_smem<D, RB, true, false, W>();
  auto k0 = ix_downsweep<D, RB, true, false, W>;
  int occ = 0;
  VDFCG_CUDA(cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  VDFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k0, kIxBlock, smem));
  const int64_t tiles = (n + kIxTile - 1) / kIxTile;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(ctx->sm_count) * std::max(occ, 1))));
  const int64_t per = ((tiles + grid - 1) / grid) * kIxTile;
  uint32_t* hist = arena<uint32_t>(ctx, size_t(DIG) * grid);
  // ping-pong u64 item buffers between passes; the last pass writes the caller's grouped
  // keys / weights and the cell ids the offsets are read from
  uint64_t* items[2] = {passes > 1 ? arena<uint64_t>(ctx, size_t(n)) : nullptr,
                        passes > 2 ? arena<uint64_t>(ctx, size_t(n)) : nullptr};
  double* ws[2] = {W && passes > 1 ? arena<double>(ctx, size_t(n)) : nullptr,
                   W && passes > 2 ? arena<double>(ctx, size_t(n)) : nullptr};
  uint32_t* cells = arena<uint32_t>(ctx, size_t(n));
  IxSrc src{{in.vel[0], in.vel[1], in.vel[2]}, in.w, in.cell, nullptr, nullptr};
  for (int p = 0; p < passes; ++p) {
    const bool first = p == 0, last = p == passes - 1;
    IxDst dst{last ? nullptr : items[p & 1], cells, out.keys, last ? out.w : ws[p & 1]};
    const int sh = p * RB;
    if (first && last) run_pass<D, RB, true, true, W>(ctx, src, dst, n, grid, per, in.n_cells, g, sh, hist, err);
    else if (first) run_pass<D, RB, true, false, W>(ctx, src, dst, n, grid, per, in.n_cells, g, sh, hist, err);
    else if (last) run_pass<D, RB, false, true, W>(ctx, src, dst, n, grid, per, in.n_cells, g, sh, hist, err);
    else run_pass<D, RB, false, false, W>(ctx, src, dst, n, grid, per, in.n_cells, g, sh, hist, err);
    src.items = dst.items;
    src.ws = dst.w;
  }
  const int og = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n / 4 + 256) / 256, int64_t(ctx->sm_count) * 8)));
  VDFCG_LAUNCH(ctx, "group_offsets", ix_offsets<<<og, 256, 0, ctx->stream>>>(cells, n, in.n_cells, out.offsets));
}

int bits_needed(int64_t v) {  // smallest b with 2^b > v
  int b = 0;
  while (b < 62 && (int64_t(1) << b) <= v) ++b;
  return b;
}

template <int D, bool W>
void group_d(vdfcg_ctx* ctx, const IndexedDev& in, const GroupedDev& out, int* err) {
  const int cbits = std::max(1, bits_needed(int64_t(in.n_cells) - 1));
  const int passes = (cbits + 8) / 9;  // <= 9 bits per pass
  if (cbits <= 8 * passes) group_impl<D, 8, W>(ctx, in, passes, out, err);
  else group_impl<D, 9, W>(ctx, in, passes, out, err);
}

}  // namespace

void launch_group_cells(vdfcg_ctx* ctx, const IndexedDev& in, const GroupedDev& out, int* err) {
  if (in.n == 0) {
    VDFCG_CUDA(cudaMemsetAsync(out.offsets, 0, (size_t(in.n_cells) + 1) * sizeof(int64_t), ctx->stream));
    return;
  }
  const bool w = in.w != nullptr;
  if (in.d == 2) {
    if (w) group_d<2, true>(ctx, in, out, err);
    else group_d<2, false>(ctx, in, out, err);
  } else {
    if (w) group_d<3, true>(ctx, in, out, err);
    else group_d<3, false>(ctx, in, out, err);
  }
}

}  // namespace vdfcg
