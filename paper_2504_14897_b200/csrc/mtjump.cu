// mtjump.cu — mt19937_64 jump-ahead for the device copy of the reference generator
// (rng.hpp:17-48, synthdata.cpp:54-86).
//
// The reference draws every particle from ONE sequential mt19937_64(seed) stream. Its raw
// (untempered) words y_0, y_1, ... obey y_{k+312} = y_{k+156} ^ twist(y_k, y_{k+1}), a linear
// recurrence over GF(2) whose state transition has minimal polynomial x * phi(x), phi of
// degree 19937 (the factor x is the 31 unused low bits of the seeded word 0). Hence for
// k >= 1 every bit lane satisfies phi, and so does the 64-bit word sequence:
//     y_{k+J} = XOR_{i : g_i = 1} y_{k+i},   g(x) = x^J mod phi(x),
// i.e. the 312-word window at any offset J is a correlation of the first 19937 + 312 words
// with the bits of g. The stream is cut into chunks of L raw words; chunk c's window at
// 1 + c L comes from g_c = x^{cL} mod phi (host, GF(2)[x] arithmetic with PCLMULQDQ + Barrett
// reduction, seed-independent and cached for the process), and each chunk then runs the
// ordinary 312-word twist from its window — one CTA per chunk, all SMs at once, instead of
// one CTA twisting the whole stream. phi itself is found once by Berlekamp-Massey on one bit
// lane of 2 * 19937 raw words. Every word equals the sequential stream's bit for bit.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include <immintrin.h>

#include "common.cuh"
#include "ctx.cuh"

namespace vdfcg {

constexpr int kMtN64 = 312, kMtM64 = 156;
constexpr int kPhiDeg = 19937;
constexpr int kPolyWords = (kPhiDeg + 63) / 64;          // 312 words hold a residue mod phi
constexpr int kBaseWords = 1 + kPhiDeg + kMtN64;          // y_0 .. y_{19937+312}

namespace {

using Poly = std::vector<uint64_t>;

// ---------------------------------------------------------------- host GF(2)[x]
__attribute__((target("pclmul,sse4.1"))) void clmul_pclmul(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
  const __m128i r = _mm_clmulepi64_si128(_mm_set_epi64x(0, static_cast<long long>(a)),
                                         _mm_set_epi64x(0, static_cast<long long>(b)), 0);
  lo = static_cast<uint64_t>(_mm_cvtsi128_si64(r));
  hi = static_cast<uint64_t>(_mm_extract_epi64(r, 1));
}

void clmul_soft(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
  lo = hi = 0;
  for (int i = 0; i < 64; ++i)
    if ((b >> i) & 1) {
      lo ^= a << i;
      if (i) hi ^= a >> (64 - i);
    }
}

const bool kHavePclmul = __builtin_cpu_supports("pclmul");

// r = a * b (carry-less), |r| = |a| + |b| words
__attribute__((target("pclmul,sse4.1"))) Poly pmul_fast(const Poly& a, const Poly& b) {
  Poly r(a.size() + b.size(), 0);
  for (size_t i = 0; i < a.size(); ++i) {
    if (!a[i]) continue;
    const __m128i ai = _mm_set_epi64x(0, static_cast<long long>(a[i]));
    for (size_t j = 0; j < b.size(); ++j) {
      const __m128i p = _mm_clmulepi64_si128(ai, _mm_set_epi64x(0, static_cast<long long>(b[j])), 0);
      r[i + j] ^= static_cast<uint64_t>(_mm_cvtsi128_si64(p));
      r[i + j + 1] ^= static_cast<uint64_t>(_mm_extract_epi64(p, 1));
    }
  }
  return r;
}

Poly pmul(const Poly& a, const Poly& b) {
  if (kHavePclmul) return pmul_fast(a, b);
  Poly r(a.size() + b.size(), 0);
  for (size_t i = 0; i < a.size(); ++i)
    for (size_t j = 0; j < b.size(); ++j) {
      uint64_t lo, hi;
      clmul_soft(a[i], b[j], lo, hi);
      r[i + j] ^= lo;
      r[i + j + 1] ^= hi;
    }
  return r;
}

inline int bit(const Poly& p, int64_t i) {
  return (i >> 6) < static_cast<int64_t>(p.size()) ? static_cast<int>((p[i >> 6] >> (i & 63)) & 1) : 0;
}

// bits [from, from + len) of p as a polynomial (p >> from, truncated)
Poly shr(const Poly& p, int64_t from, int64_t len) {
  Poly r((len + 63) / 64, 0);
  for (int64_t i = 0; i < len; ++i)
    if (bit(p, from + i)) r[i >> 6] |= uint64_t(1) << (i & 63);
  return r;
}

Poly low(const Poly& p, int64_t len) { return shr(p, 0, len); }

struct Jumper {
  std::mutex mu;
  bool ready = false;
  Poly phi;   // degree 19937, phi[19937] = 1
  Poly mu_;   // floor(x^(2 deg) / phi)
  int64_t L = 0;
  Poly h;     // x^L mod phi
  std::vector<Poly> g;  // g[c] = x^(c L) mod phi

  // a mod phi for deg(a) < 2 * deg(phi) (Barrett: q = ((a >> n) * mu) >> n, r = a - q phi)
  Poly mod(const Poly& a) const {
    const int64_t n = kPhiDeg;
    const Poly q = shr(pmul(shr(a, n, n), mu_), n, n + 1);
    const Poly qp = pmul(q, phi);
    Poly r = low(a, n);
    const Poly lq = low(qp, n);
    for (size_t i = 0; i < r.size(); ++i) r[i] ^= lq[i];
    return r;
  }
  Poly mulmod(const Poly& a, const Poly& b) const { return mod(pmul(a, b)); }

  // x^e mod phi by square-and-multiply from x^1
  Poly xpow(uint64_t e) const {
    Poly r(kPolyWords, 0);
    r[0] = 1;
    Poly base(kPolyWords, 0);
    base[0] = 2;  // x
    while (e) {
      if (e & 1) r = mulmod(r, base);
      e >>= 1;
      if (e) base = mulmod(base, base);
    }
    r.resize(kPolyWords);
    return r;
  }

  void init_phi() {
    // raw words of mt19937_64(5489): phi is seed-independent
    std::vector<uint64_t> mt(kMtN64);
    mt[0] = 5489;
    for (int i = 1; i < kMtN64; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    const int64_t N = 2 * int64_t(kPhiDeg) + 64;
    std::vector<uint8_t> s(N);
    int idx = kMtN64;
    int64_t k = -1;  // raw word index
    for (int64_t t = 0; t < N + 1; ++t) {
      if (idx >= kMtN64) {
        for (int i = 0; i < kMtN64; ++i) {
          const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % kMtN64] & 0x7FFFFFFFULL);
          mt[i] = mt[(i + kMtM64) % kMtN64] ^ (x >> 1) ^ ((x & 1) ? 0xB5026F5AA96619E9ULL : 0ULL);
        }
        idx = 0;
      }
      ++k;
      const uint64_t y = mt[idx++];
      if (k >= 1 && k - 1 < N) s[k - 1] = static_cast<uint8_t>(y & 1);  // bit lane 0 of y_1, y_2, ...
    }
    // Berlekamp-Massey over GF(2) on bit-packed polynomials: connection polynomial C
    // (C_0 = 1). R is s reversed, so sum_i C_i s_{nn-i} is a dot product of C with R read
    // from bit N-1-nn on.
    const int W = static_cast<int>((N + 64) / 64) + 2;
    std::vector<uint64_t> R(W + 2, 0);
    for (int64_t i = 0; i < N; ++i)
      if (s[i]) R[(N - 1 - i) >> 6] |= uint64_t(1) << ((N - 1 - i) & 63);
    auto rbits = [&](int64_t off) {  // 64 bits of R starting at bit off
      const int64_t w = off >> 6;
      const int b = static_cast<int>(off & 63);
      const uint64_t lo = R[w] >> b;
      return b ? (lo | (R[w + 1] << (64 - b))) : lo;
    };
    std::vector<uint64_t> C(W, 0), B(W, 0), T;
    C[0] = B[0] = 1;
    int Lc = 0, m = 1;
    auto add_shifted = [&](std::vector<uint64_t>& dst, const std::vector<uint64_t>& src, int sft) {
      const int ws = sft >> 6, bs = sft & 63;
      for (int i = W - 1; i >= 0; --i) {
        uint64_t v = 0;
        if (i - ws >= 0) v = src[i - ws] << bs;
        if (bs && i - ws - 1 >= 0) v |= src[i - ws - 1] >> (64 - bs);
        dst[i] ^= v;
      }
    };
    for (int64_t nn = 0; nn < N; ++nn) {
      // discrepancy: sum_{i=0..Lc} C_i s_{nn-i}, s_{nn-i} = R bit (N-1-nn+i)
      uint64_t acc = 0;
      const int words = Lc / 64 + 1;
      for (int w = 0; w < words; ++w) acc ^= C[w] & rbits(N - 1 - nn + 64 * int64_t(w));
      const int dsc = __builtin_popcountll(acc) & 1;
      if (!dsc) {
        ++m;
      } else if (2 * Lc <= nn) {
        T = C;
        add_shifted(C, B, m);
        Lc = static_cast<int>(nn + 1 - Lc);
        B = T;
        m = 1;
      } else {
        add_shifted(C, B, m);
        ++m;
      }
    }
    auto cbit = [&](int i) { return static_cast<int>((C[i >> 6] >> (i & 63)) & 1); };
    // phi(x) = x^L C(1/x): phi_j = C[L - j]
    phi.assign((kPhiDeg + 1 + 63) / 64, 0);
    for (int j = 0; j <= kPhiDeg; ++j)
      if (cbit(kPhiDeg - j)) phi[j >> 6] |= uint64_t(1) << (j & 63);
    // mu = floor(x^(2n) / phi) by long division
    const int64_t n = kPhiDeg;
    Poly rem((2 * n + 1 + 63) / 64 + 1, 0);
    rem[(2 * n) >> 6] |= uint64_t(1) << ((2 * n) & 63);
    mu_.assign((n + 1 + 63) / 64, 0);
    for (int64_t d = 2 * n; d >= n; --d) {
      if (!bit(rem, d)) continue;
      const int64_t sft = d - n;
      mu_[sft >> 6] |= uint64_t(1) << (sft & 63);
      // rem ^= phi << sft
      const int ws = static_cast<int>(sft >> 6), bs = static_cast<int>(sft & 63);
      for (size_t i = 0; i < phi.size(); ++i) {
        rem[i + ws] ^= phi[i] << bs;
        if (bs && i + ws + 1 < rem.size()) rem[i + ws + 1] ^= phi[i] >> (64 - bs);
      }
    }
    ready = true;
  }

  // g[0..count) for chunk stride L (grows the cache; L fixed per process)
  void chunks(int64_t stride, int count) {
    if (!ready) init_phi();
    if (stride != L) {
      L = stride;
      h = xpow(static_cast<uint64_t>(L));
      g.clear();
    }
    if (g.empty()) {
      Poly one(kPolyWords, 0);
      one[0] = 1;
      g.push_back(one);
    }
    while (static_cast<int>(g.size()) < count) {
      Poly nx = mulmod(g.back(), h);
      nx.resize(kPolyWords);
      g.push_back(nx);
    }
  }
};

Jumper& jumper() {
  static Jumper j;
  return j;
}

}  // namespace

// ---------------------------------------------------------------- device
VDFCG_DEV uint64_t jtwist(uint64_t upper_src, uint64_t lower_src) {
  const uint64_t xx = (upper_src & 0xFFFFFFFF80000000ULL) | (lower_src & 0x7FFFFFFFULL);
  return (xx >> 1) ^ ((xx & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
}

// Chunk c = blockIdx.x: raw words [1 + c L, 1 + (c + 1) L) (clipped to count). The base words
// y_0 .. y_{19937+312} are staged in shared memory; thread j (< 312) forms window word
// W[j] = y_{1 + cL + j} = XOR over the set bits i of g_c of y_{1 + i + j}; then 156 threads
// continue the twist from the window with the register-pair scheme of mt_stream_kernel.
__global__ void __launch_bounds__(kMtN64) mt_chunk_kernel(const uint64_t* __restrict__ base,
                                                         const uint64_t* __restrict__ gbits, int64_t L,
                                                         int64_t count, uint64_t* __restrict__ out) {
  extern __shared__ __align__(16) uint64_t sbase[];  // [kBaseWords] then u16 bit list [<= 19937]
  __shared__ uint64_t sh[2][2][kMtM64];
  __shared__ uint64_t win[kMtN64];
  __shared__ int wsum[kMtN64 / 32 + 1];
  const int t = threadIdx.x;
  const int c = blockIdx.x;
  const int64_t s0 = 1 + static_cast<int64_t>(c) * L;
  if (s0 >= count) return;
  const int64_t s1 = min(count, s0 + L);
  uint16_t* blist = reinterpret_cast<uint16_t*>(sbase + kBaseWords);
  for (int i = t; i < kBaseWords; i += blockDim.x) sbase[i] = __ldg(base + i);
  // the set bits of g_c as an index list: popcount per word, block exclusive scan, scatter
  const uint64_t gw = __ldg(gbits + static_cast<int64_t>(c) * kPolyWords + t);
  const int pc = __popcll(gw);
  int incl = pc;
  const int lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31 || t == kMtN64 - 1) wsum[warp] = incl;
  __syncthreads();
  int pre = incl - pc;
  for (int w = 0; w < warp; ++w) pre += wsum[w];
  int total = 0;
  for (int w = 0; w <= (kMtN64 - 1) / 32; ++w) total += wsum[w];
  for (uint64_t m = gw; m; m &= m - 1) blist[pre++] = static_cast<uint16_t>(t * 64 + __ffsll(static_cast<long long>(m)) - 1);
  __syncthreads();
  {
    // W[t] = XOR of y_{1 + i + t} over the list: four independent accumulators (the list reads
    // are broadcasts, the base reads consecutive across the warp)
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    const uint64_t* yb = sbase + 1 + t;
    int k = 0;
    for (; k + 4 <= total; k += 4) {
      a0 ^= yb[blist[k]];
      a1 ^= yb[blist[k + 1]];
      a2 ^= yb[blist[k + 2]];
      a3 ^= yb[blist[k + 3]];
    }
    for (; k < total; ++k) a0 ^= yb[blist[k]];
    const uint64_t acc = (a0 ^ a1) ^ (a2 ^ a3);
    win[t] = acc;
    if (s0 + t < s1) out[s0 + t] = acc;
  }
  __syncthreads();
  const bool tw = t < kMtM64;  // the twist runs on 156 threads; the rest only keep the barriers
  uint64_t A = tw ? win[t] : 0, B = tw ? win[t + kMtM64] : 0;
  int p = 0;
  for (int64_t b = s0 + kMtN64; b < s1; b += kMtN64) {
    if (tw) {
      sh[p][0][t] = A;
      sh[p][1][t] = B;
    }
    __syncthreads();
    if (!tw) {
      p ^= 1;
      continue;
    }
    uint64_t A1, B1;
    if (t + 1 < kMtM64) {
      A1 = sh[p][0][t + 1];
      B1 = sh[p][1][t + 1];
    } else {
      A1 = sh[p][1][0];
      B1 = sh[p][1][0] ^ jtwist(sh[p][0][0], sh[p][0][1]);
    }
    A = B ^ jtwist(A, A1);
    B = A ^ jtwist(B, B1);
    if (b + t < s1) out[b + t] = A;
    if (b + t + kMtM64 < s1) out[b + t + kMtM64] = B;
    p ^= 1;
  }
}

__global__ void mt_word0_kernel(const uint64_t* base, uint64_t* out) { out[0] = base[0]; }

void launch_mt_serial(vdfcg_ctx* ctx, uint64_t seed, int64_t count, uint64_t* out);  // synth.cu

// Raw words [0, count) of mt19937_64(seed): the serial single-CTA twist for short streams,
// else the base window + one CTA per chunk. Returns false when it left the work to the caller.
bool launch_mt_stream_jump(vdfcg_ctx* ctx, uint64_t seed, int64_t count, uint64_t* out) {
  constexpr int64_t kChunk = int64_t(1) << 18;  // raw words per chunk (cache key of g_c)
  if (count < 4 * kChunk) return false;
  const int chunks = static_cast<int>((count - 1 + kChunk - 1) / kChunk);
  Jumper& J = jumper();
  std::vector<uint64_t> host;
  {
    std::lock_guard<std::mutex> lk(J.mu);
    J.chunks(kChunk, chunks);
    host.resize(size_t(chunks) * kPolyWords);
    for (int c = 0; c < chunks; ++c) std::memcpy(&host[size_t(c) * kPolyWords], J.g[c].data(), kPolyWords * 8);
  }
  uint64_t* base = arena<uint64_t>(ctx, kBaseWords);
  uint64_t* gdev = arena<uint64_t>(ctx, host.size());
  VDFCG_CUDA(cudaMemcpyAsync(gdev, host.data(), host.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  launch_mt_serial(ctx, seed, kBaseWords, base);
  const size_t smem = size_t(kBaseWords) * 8 + size_t(kPhiDeg + 8) * 2;
  VDFCG_CUDA(cudaFuncSetAttribute(mt_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  VDFCG_LAUNCH(ctx, "mt19937_64_chunks",
               mt_chunk_kernel<<<chunks, kMtN64, smem, ctx->stream>>>(base, gdev, kChunk, count, out));
  VDFCG_LAUNCH(ctx, "mt19937_64_chunks", mt_word0_kernel<<<1, 1, 0, ctx->stream>>>(base, out));
  // the host copy of g must outlive the async H2D
  VDFCG_CUDA(cudaStreamSynchronize(ctx->stream));
  return true;
}

// ---------------------------------------------------------------- host check hook
// Window of 312 raw words at offset 1 + J, by the host correlation (tests: compares the
// jump machinery with a sequential host replay without a device).
void mt_window_host(uint64_t seed, uint64_t J, uint64_t* out) {
  Jumper& Jm = jumper();
  Poly g;
  {
    std::lock_guard<std::mutex> lk(Jm.mu);
    if (!Jm.ready) Jm.init_phi();
    g = Jm.xpow(J);
  }
  std::vector<uint64_t> mt(kMtN64), y(kBaseWords);
  mt[0] = seed;
  for (int i = 1; i < kMtN64; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
  int idx = kMtN64;
  for (int k = 0; k < kBaseWords; ++k) {
    if (idx >= kMtN64) {
      for (int i = 0; i < kMtN64; ++i) {
        const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % kMtN64] & 0x7FFFFFFFULL);
        mt[i] = mt[(i + kMtM64) % kMtN64] ^ (x >> 1) ^ ((x & 1) ? 0xB5026F5AA96619E9ULL : 0ULL);
      }
      idx = 0;
    }
    y[k] = mt[idx++];
  }
  for (int j = 0; j < kMtN64; ++j) {
    uint64_t acc = 0;
    for (int i = 0; i < kPhiDeg; ++i)
      if (bit(g, i)) acc ^= y[1 + i + j];
    out[j] = acc;
  }
}

}  // namespace vdfcg

extern "C" int vdfcg_debug_mt_window(uint64_t seed, uint64_t offset, uint64_t* out) {
  return vdfcg::guard_impl([&] {
    if (!out || offset < 1) throw vdfcg::InvalidArgument("offset >= 1 and an output buffer required");
    vdfcg::mt_window_host(seed, offset - 1, out);
  });
}
