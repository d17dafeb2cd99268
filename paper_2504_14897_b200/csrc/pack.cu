// pack.cu — K6: .gmmc records for every fitted cell (FORMATS.md:7-50).
// Header: magic "GMMC", version 1, d, plane, reserved, u32 M, i64 cycle, d x (lo, hi) f64,
// u16 label length, label, u32 CRC-32 (zlib polynomial) of the header; payload per
// component: weight, mean[d], covariance upper triangle row-major, f64 little-endian.
// One warp per record: lane 0 assembles and checksums the header, the warp streams the
// payload bytes.
#include <algorithm>

#include "common.cuh"
#include "hist.cuh"
#include "pack.cuh"

namespace vdfcg {

int64_t header_bytes(int d, int label_len) { return 4 + 4 + 4 + 8 + 16 * d + 2 + label_len + 4; }
int64_t payload_bytes(int m, int d) { return int64_t(m) * (1 + d + d * (d + 1) / 2) * 8; }

VDFCG_DEV uint32_t crc32_update(uint32_t crc, uint8_t b) {
  crc ^= b;
#pragma unroll
  for (int k = 0; k < 8; ++k) crc = (crc >> 1) ^ (0xEDB88320u & (0u - (crc & 1u)));
  return crc;
}

__global__ void pack_sizes_kernel(PackIn in, PackMeta meta, int64_t* sizes) {
  const int64_t hb = 4 + 4 + 4 + 8 + 16 * meta.d + 2 + meta.label_len + 4;
  const int per = (1 + meta.d + meta.d * (meta.d + 1) / 2) * 8;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < in.n_cells; c += gridDim.x * blockDim.x) {
    const bool ok = (!in.status || in.status[c] == 0) && in.comps[c] > 0;
    sizes[c] = ok ? hb + int64_t(in.comps[c]) * per : 0;
  }
}

VDFCG_DEV void put_bytes(uint8_t* dst, int& pos, uint64_t v, int n, uint32_t& crc, bool do_crc) {
  for (int i = 0; i < n; ++i) {
    const uint8_t b = static_cast<uint8_t>(v >> (8 * i));
    dst[pos++] = b;
    if (do_crc) crc = crc32_update(crc, b);
  }
}

__global__ void __launch_bounds__(256) pack_kernel(PackIn in, PackMeta meta, const int64_t* offsets,
                                                   uint8_t* out) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int d = meta.d;
  const int per = 1 + d + d * (d + 1) / 2;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < in.n_cells; c += warps) {
    const int64_t o = offsets[c];
    if (offsets[c + 1] == o) continue;
    uint8_t* dst = out + o;
    const int m = in.comps[c];
    int hb = 0;
    if (lane == 0) {
      uint32_t crc = 0xFFFFFFFFu;
      int pos = 0;
      put_bytes(dst, pos, 0x434D4D47ull, 4, crc, true);  // "GMMC"
      put_bytes(dst, pos, 1, 1, crc, true);
      put_bytes(dst, pos, static_cast<uint64_t>(d), 1, crc, true);
      put_bytes(dst, pos, static_cast<uint64_t>(meta.plane), 1, crc, true);
      put_bytes(dst, pos, 0, 1, crc, true);
      put_bytes(dst, pos, static_cast<uint32_t>(m), 4, crc, true);
      put_bytes(dst, pos, static_cast<uint64_t>(meta.cycle), 8, crc, true);
      for (int a = 0; a < d; ++a) {
        put_bytes(dst, pos, static_cast<uint64_t>(__double_as_longlong(meta.lo[a])), 8, crc, true);
        put_bytes(dst, pos, static_cast<uint64_t>(__double_as_longlong(meta.hi[a])), 8, crc, true);
      }
      put_bytes(dst, pos, static_cast<uint64_t>(meta.label_len), 2, crc, true);
      for (int i = 0; i < meta.label_len; ++i) put_bytes(dst, pos, meta.label[i], 1, crc, true);
      crc ^= 0xFFFFFFFFu;
      put_bytes(dst, pos, crc, 4, crc, false);
      hb = pos;
    }
    hb = __shfl_sync(0xffffffffu, hb, 0);
    // payload: doubles, component-major: weight, mean, upper covariance
    const int nval = m * per;
    const int64_t kb = static_cast<int64_t>(c) * in.K;
    for (int v = lane; v < nval; v += 32) {
      const int i = v / per, r = v - i * per;
      double x;
      if (r == 0) {
        x = in.w[kb + i];
      } else if (r <= d) {
        x = in.mu[(kb + i) * d + (r - 1)];
      } else {
        int u = r - 1 - d, a = 0;
        while (u >= d - a) {
          u -= d - a;
          ++a;
        }
        const int b = a + u;
        x = in.cov[((kb + i) * d + a) * d + b];
      }
      const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(x));
      uint8_t* p = dst + hb + v * 8;
#pragma unroll
      for (int k = 0; k < 8; ++k) p[k] = static_cast<uint8_t>(bits >> (8 * k));
    }
  }
}

int64_t launch_pack_offsets(vdfcg_ctx* ctx, const PackIn& in, const PackMeta& meta,
                            int64_t* offsets) {
  int64_t* sizes = arena<int64_t>(ctx, in.n_cells);
  const int grid = std::max(1, std::min((in.n_cells + 255) / 256, ctx->sm_count * 8));
  VDFCG_LAUNCH(ctx, "pack_sizes", pack_sizes_kernel<<<grid, 256, 0, ctx->stream>>>(in, meta, sizes));
  launch_scan_i64(ctx, sizes, offsets, in.n_cells);
  int64_t* h = static_cast<int64_t*>(ctx->pinned);
  VDFCG_CUDA(cudaMemcpyAsync(h, offsets + in.n_cells, 8, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  return *h;
}

void launch_pack(vdfcg_ctx* ctx, const PackIn& in, const PackMeta& meta, const int64_t* offsets,
                 uint8_t* out) {
  const int grid = std::max(1, std::min((in.n_cells * 32 + 255) / 256, ctx->sm_count * 16));
  VDFCG_LAUNCH(ctx, "pack_gmmc", pack_kernel<<<grid, 256, 0, ctx->stream>>>(in, meta, offsets, out));
}

}  // namespace vdfcg
