// pack.cuh — .gmmc record packing (FORMATS.md, codec.cpp:103-136) on the device.
#pragma once

#include "ctx.cuh"

namespace vdfcg {

struct PackMeta {
  int d;
  int plane;        // 0,1,2 or 255
  int64_t cycle;
  double lo[3], hi[3];
  const uint8_t* label;  // device
  int label_len;
};

struct PackIn {
  int n_cells;
  int K;                  // stride
  const int32_t* status;  // may be null (all ok)
  const int32_t* comps;
  const double* w;
  const double* mu;
  const double* cov;      // [cells*K*d*d]
};

int64_t header_bytes(int d, int label_len);
int64_t payload_bytes(int m, int d);
// sizes -> offsets (device, n_cells+1), returns total bytes (synchronizes).
int64_t launch_pack_offsets(vdfcg_ctx* ctx, const PackIn& in, const PackMeta& meta,
                            int64_t* offsets);
void launch_pack(vdfcg_ctx* ctx, const PackIn& in, const PackMeta& meta, const int64_t* offsets,
                 uint8_t* out);

}  // namespace vdfcg
