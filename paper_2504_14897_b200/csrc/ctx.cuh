// ctx.cuh — context, workspace arena, host/device staging, per-kernel timing, errors.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vdfcg.h"

namespace vdfcg {

// Exceptions carried to the C-ABI boundary and mapped to return codes.
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RepairFailed : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);
#define VDFCG_CUDA(x) ::vdfcg::cuda_check((x), #x)

bool is_device_pointer(const void* p);
// Device memory of ANOTHER GPU than the context's cannot be read by its kernels (no peer
// mapping is set up): such pointers are rejected with the reference's invalid_argument.
void check_pointer_device(const vdfcg_ctx* ctx, const void* p);

// Runs f, mapping the exceptions above to VDFCG_* codes + the thread-local message.
int guard_impl(const std::function<void()>& f);

}  // namespace vdfcg

struct vdfcg_ctx {
  int device = 0;
  int sm_count = 148;
  size_t smem_optin = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // H2D of later cell chunks overlaps compute
  cudaStream_t aux_stream = nullptr;   // second compute stream: chunk kernels overlap tails
  cudaEvent_t handoff = nullptr;       // orders the arena's last user before a new stream
  // grow-only arena, reset at the start of every API call
  struct Chunk {
    char* base;
    size_t size;
    size_t used;
  };
  std::vector<Chunk> chunks;
  // pinned scalar readback slot
  void* pinned = nullptr;
  // pinned staging ring for pageable host inputs (allocated on first use)
  void* ring = nullptr;
  size_t ring_slot = 0;
  int ring_slots = 0;
  std::vector<cudaEvent_t> ring_ev;
  // device diagnostics counters: [0] exact second EM passes run
  unsigned long long* diag = nullptr;
  // timing
  bool timing = false;
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  std::map<std::string, std::pair<double, long long>> times;
  long long launches = 0;
};

namespace vdfcg {

void arena_reset(vdfcg_ctx* ctx);
void* arena_alloc(vdfcg_ctx* ctx, size_t bytes);
template <class T>
T* arena(vdfcg_ctx* ctx, size_t count) {
  return static_cast<T*>(arena_alloc(ctx, (count ? count : 1) * sizeof(T)));
}

// Device view of a caller buffer: the pointer itself when it is device memory,
// otherwise a staged copy (H2D at construction for inputs, D2H on finish() for outputs).
template <class T>
struct Staged {
  T* dev = nullptr;
  T* host = nullptr;
  size_t count = 0;
  bool staged = false;
};

template <class T>
Staged<T> stage_in(vdfcg_ctx* ctx, const T* p, size_t count) {
  Staged<T> s;
  s.count = count;
  if (!p) return s;
  if (is_device_pointer(p)) {
    check_pointer_device(ctx, p);
    s.dev = const_cast<T*>(p);
    return s;
  }
  s.dev = arena<T>(ctx, count);
  s.host = const_cast<T*>(p);
  s.staged = true;
  if (count)
    VDFCG_CUDA(cudaMemcpyAsync(s.dev, p, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return s;
}

template <class T>
Staged<T> stage_out(vdfcg_ctx* ctx, T* p, size_t count) {
  Staged<T> s;
  s.count = count;
  if (!p) return s;
  if (is_device_pointer(p)) {
    check_pointer_device(ctx, p);
    s.dev = p;
    return s;
  }
  s.dev = arena<T>(ctx, count);
  s.host = p;
  s.staged = true;
  return s;
}

template <class T>
void finish(vdfcg_ctx* ctx, const Staged<T>& s, size_t count = size_t(-1)) {
  if (!s.staged || !s.host) return;
  const size_t n = count == size_t(-1) ? s.count : count;
  if (n)
    VDFCG_CUDA(cudaMemcpyAsync(s.host, s.dev, n * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
}

void sync(vdfcg_ctx* ctx);

// Kernel launch bracket: records CUDA events around the launch when timing is on.
struct LaunchScope {
  vdfcg_ctx* ctx;
  const char* name;
  cudaEvent_t a = nullptr, b = nullptr;
  LaunchScope(vdfcg_ctx* c, const char* n);
  ~LaunchScope() noexcept(false);
};
#define VDFCG_LAUNCH(ctx, name, ...)          \
  do {                                        \
    ::vdfcg::LaunchScope _ls((ctx), (name));  \
    __VA_ARGS__;                              \
    VDFCG_CUDA(cudaGetLastError());           \
  } while (0)

}  // namespace vdfcg
