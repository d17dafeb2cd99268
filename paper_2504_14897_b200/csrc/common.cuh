// common.cuh — shared device helpers for the vdfcg kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#define VDFCG_DEV __device__ __forceinline__
#define VDFCG_HD __host__ __device__ __forceinline__

namespace vdfcg {

constexpr int kWarp = 32;
constexpr int kMaxK = 16;   // VDFCG_MAX_COMPONENTS
constexpr int kMaxWarps = 32;

// log(2*pi) as a double (the reference computes std::log(2.0 * M_PI), gaussian.hpp:31).
constexpr double kLog2Pi = 1.8378770664093453;
constexpr double kMassFloorRel = 1e-250;  // wgmm.cpp:20

VDFCG_DEV double dinf() { return __longlong_as_double(0x7ff0000000000000ULL); }
VDFCG_DEV double dnan() { return __longlong_as_double(0x7ff8000000000000ULL); }

// histogram.cpp:36-41 bin_index. Left-closed right-open, top edge closed. NaN is out of
// range (the reference's x86 float->int conversion of floor(NaN) yields INT_MIN, which
// fails the range test at histogram.cpp:70). For in-range values t = (v - lo) * inv >= 0,
// so truncation equals floor: one F2I instead of FRND + F2I, and a select instead of a
// branch. (v - lo) * inv cannot contract into an FMA.
VDFCG_DEV int bin_index(double v, double lo, double hi, int n, double inv) {
  const int i = min(__double2int_rz((v - lo) * inv), n - 1);
  return (v >= lo && v <= hi) ? i : -1;
}

// GridSpec::center_x (types.hpp:48,51): lo + (i + 0.5) * ((hi - lo) / n), no FMA.
VDFCG_DEV double bin_center(double lo, double hi, int n, int i) {
  const double dx = (hi - lo) / static_cast<double>(n);
  return __dadd_rn(lo, __dmul_rn(static_cast<double>(i) + 0.5, dx));
}

template <class T>
VDFCG_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <class T>
VDFCG_DEV T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  return v;
}

template <class T>
VDFCG_DEV T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}

// Warp transpose-reduction of N per-lane values (reduce-scatter over xor butterflies):
// at offset o each lane keeps one half of its values, sends the other half to lane^o and
// adds what it receives, so the work halves every level (~N·7/... instructions instead of
// N·5 shuffles + adds). On return lane l holds the warp totals of global indices
// start + j for j < count (count <= HOUT), in a fixed summation order (deterministic).
template <int N>
struct WarpScatter {
  static constexpr int H1 = (N + 1) / 2, H2 = (H1 + 1) / 2, H3 = (H2 + 1) / 2, H4 = (H3 + 1) / 2,
                       H5 = (H4 + 1) / 2;
  static constexpr int HOUT = H5;
};

template <int N, int O, int NN>
VDFCG_DEV void scatter_level(double (&v)[NN], int lane, int& start, int& count) {
  constexpr int H = (N + 1) / 2;
  const bool up = (lane & O) != 0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const double lo = v[i];
    const double hi = (i + H < N) ? v[i + H] : 0.0;
    const double send = up ? lo : hi;
    const double keep = up ? hi : lo;
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
  }
  if (up) {
    start += H;
    count = count > H ? count - H : 0;
  } else {
    count = count < H ? count : H;
  }
}

template <int N>
VDFCG_DEV void warp_scatter_sum(double (&v)[N], int lane, int& start, int& count) {
  using WS = WarpScatter<N>;
  start = 0;
  count = N;
  scatter_level<N, 16>(v, lane, start, count);
  scatter_level<WS::H1, 8>(v, lane, start, count);
  scatter_level<WS::H2, 4>(v, lane, start, count);
  scatter_level<WS::H3, 2>(v, lane, start, count);
  scatter_level<WS::H4, 1>(v, lane, start, count);
}

// Kahan accumulator (gaussian.hpp:55-68). Explicit _rn intrinsics keep the
// compensation exact regardless of contraction.
struct Kahan {
  double s = 0.0, c = 0.0;
  VDFCG_DEV void add(double x) {
    const double y = __dsub_rn(x, c);
    const double t = __dadd_rn(s, y);
    c = __dsub_rn(__dsub_rn(t, s), y);
    s = t;
  }
  VDFCG_DEV double value() const { return __dsub_rn(s, c); }
};

}  // namespace vdfcg
