// ctx.cu — context lifecycle, arena, staging, timing, error plumbing of the C-ABI.
#include <cstring>
#include <functional>
#include <string>

#include "ctx.cuh"

namespace vdfcg {

thread_local std::string g_last_error;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")");
  }
}

bool is_device_pointer(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void check_pointer_device(const vdfcg_ctx* ctx, const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  if (a.type == cudaMemoryTypeDevice && a.device != ctx->device)
    throw InvalidArgument("device pointer on cuda:" + std::to_string(a.device) +
                          " passed to a context on cuda:" + std::to_string(ctx->device));
}

void arena_reset(vdfcg_ctx* ctx) {
  for (auto& c : ctx->chunks) c.used = 0;
}

void* arena_alloc(vdfcg_ctx* ctx, size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  for (auto& c : ctx->chunks) {
    if (c.size - c.used >= bytes) {
      void* p = c.base + c.used;
      c.used += bytes;
      return p;
    }
  }
  size_t sz = bytes;
  if (!ctx->chunks.empty()) sz = std::max(sz, ctx->chunks.back().size * 2);
  sz = std::max(sz, size_t(64) << 20);
  char* base = nullptr;
  VDFCG_CUDA(cudaMalloc(&base, sz));
  ctx->chunks.push_back({base, sz, bytes});
  return base;
}

void sync(vdfcg_ctx* ctx) { VDFCG_CUDA(cudaStreamSynchronize(ctx->stream)); }

static cudaEvent_t take_event(vdfcg_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  VDFCG_CUDA(cudaEventCreate(&e));
  return e;
}

LaunchScope::LaunchScope(vdfcg_ctx* c, const char* n) : ctx(c), name(n) {
  ++ctx->launches;
  if (ctx->timing) {
    a = take_event(ctx);
    b = take_event(ctx);
    VDFCG_CUDA(cudaEventRecord(a, ctx->stream));
  }
}

LaunchScope::~LaunchScope() noexcept(false) {
  if (ctx->timing && a) {
    cudaEventRecord(b, ctx->stream);
    ctx->pending.push_back({name, a, b});
  }
}

static void resolve_timing(vdfcg_ctx* ctx) {
  if (ctx->pending.empty()) return;
  sync(ctx);
  for (auto& p : ctx->pending) {
    float ms = 0.f;
    VDFCG_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    auto& t = ctx->times[p.name];
    t.first += ms;
    t.second += 1;
    ctx->event_pool.push_back(p.a);
    ctx->event_pool.push_back(p.b);
  }
  ctx->pending.clear();
}

}  // namespace vdfcg

namespace vdfcg {
int guard_impl(const std::function<void()>& f) {
  try {
    f();
    return VDFCG_OK;
  } catch (const InvalidArgument& e) {
    g_last_error = e.what();
    return VDFCG_INVALID_ARGUMENT;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return VDFCG_INVALID_ARGUMENT;
  } catch (const RepairFailed& e) {
    g_last_error = e.what();
    return VDFCG_REPAIR_FAILED;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return VDFCG_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return VDFCG_RUNTIME_ERROR;
  } catch (...) {
    g_last_error = "unknown error";
    return VDFCG_RUNTIME_ERROR;
  }
}
}  // namespace vdfcg

using namespace vdfcg;

extern "C" {

const char* vdfcg_last_error(void) { return g_last_error.c_str(); }

int vdfcg_abi_version(void) { return VDFCG_ABI_VERSION; }

int vdfcg_ctx_create(int device, vdfcg_ctx** out) {
  return guard_impl([&] {
    if (!out) throw InvalidArgument("null output pointer");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw CudaError("no CUDA device available (vdfcg has no CPU fallback)");
    }
    if (device < 0 || device >= n) throw InvalidArgument("device index out of range");
    VDFCG_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    VDFCG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      throw CudaError(std::string("vdfcg kernels are built for sm_100a; device is ") + prop.name);
    auto* c = new vdfcg_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    VDFCG_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    VDFCG_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    VDFCG_CUDA(cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    VDFCG_CUDA(cudaHostAlloc(&c->pinned, 4096, cudaHostAllocDefault));
    VDFCG_CUDA(cudaMalloc(&c->diag, 8 * sizeof(unsigned long long)));
    VDFCG_CUDA(cudaMemset(c->diag, 0, 8 * sizeof(unsigned long long)));
    *out = c;
  });
}

int vdfcg_ctx_destroy(vdfcg_ctx* ctx) {
  return guard_impl([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& c : ctx->chunks) cudaFree(c.base);
    for (auto& p : ctx->pending) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->diag) cudaFree(ctx->diag);
    if (ctx->aux_stream) {
      cudaStreamSynchronize(ctx->aux_stream);
      cudaStreamDestroy(ctx->aux_stream);
    }
    if (ctx->copy_stream) {
      cudaStreamSynchronize(ctx->copy_stream);
      cudaStreamDestroy(ctx->copy_stream);
    }
    for (auto e : ctx->ring_ev) cudaEventDestroy(e);
    if (ctx->ring) cudaFreeHost(ctx->ring);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    if (ctx->handoff) cudaEventDestroy(ctx->handoff);
    delete ctx;
  });
}

int vdfcg_ctx_set_stream(vdfcg_ctx* ctx, void* s) {
  return guard_impl([&] {
    if (!ctx) throw InvalidArgument("null context");
    cudaStream_t next = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
    if (next != ctx->stream) {
      // Every call resets the shared arena; asynchronous work still queued on the old
      // stream may be using it, so the new stream waits for everything enqueued so far.
      VDFCG_CUDA(cudaSetDevice(ctx->device));
      if (!ctx->handoff) VDFCG_CUDA(cudaEventCreateWithFlags(&ctx->handoff, cudaEventDisableTiming));
      VDFCG_CUDA(cudaEventRecord(ctx->handoff, ctx->stream));
      VDFCG_CUDA(cudaStreamWaitEvent(next, ctx->handoff, 0));
      ctx->stream = next;
    }
  });
}

int vdfcg_ctx_synchronize(vdfcg_ctx* ctx) {
  return guard_impl([&] {
    if (!ctx) throw InvalidArgument("null context");
    VDFCG_CUDA(cudaSetDevice(ctx->device));
    sync(ctx);
  });
}

int vdfcg_ctx_enable_timing(vdfcg_ctx* ctx, int enable) {
  return guard_impl([&] {
    if (!ctx) throw InvalidArgument("null context");
    ctx->timing = enable != 0;
  });
}

int vdfcg_ctx_reset_timing(vdfcg_ctx* ctx) {
  return guard_impl([&] {
    if (!ctx) throw InvalidArgument("null context");
    resolve_timing(ctx);
    ctx->times.clear();
  });
}

int vdfcg_ctx_kernel_times(vdfcg_ctx* ctx, int32_t max_entries, char* names, double* ms,
                           int64_t* launches, int32_t* n_entries) {
  return guard_impl([&] {
    if (!ctx) throw InvalidArgument("null context");
    VDFCG_CUDA(cudaSetDevice(ctx->device));
    resolve_timing(ctx);
    int i = 0;
    for (auto& kv : ctx->times) {
      if (i >= max_entries) break;
      std::memset(names + 32 * i, 0, 32);
      std::strncpy(names + 32 * i, kv.first.c_str(), 31);
      ms[i] = kv.second.first;
      launches[i] = kv.second.second;
      ++i;
    }
    *n_entries = i;
  });
}

int64_t vdfcg_ctx_launch_count(vdfcg_ctx* ctx) { return ctx ? ctx->launches : -1; }

int vdfcg_ctx_diagnostics(vdfcg_ctx* ctx, int64_t* exact_passes, int reset) {
  return guard_impl([&] {
    if (!ctx) throw InvalidArgument("null context");
    VDFCG_CUDA(cudaSetDevice(ctx->device));
    unsigned long long h[8];
    VDFCG_CUDA(cudaMemcpyAsync(h, ctx->diag, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (exact_passes) *exact_passes = static_cast<int64_t>(h[0]);
    if (reset) VDFCG_CUDA(cudaMemsetAsync(ctx->diag, 0, sizeof(h), ctx->stream));
  });
}

}  // extern "C"
