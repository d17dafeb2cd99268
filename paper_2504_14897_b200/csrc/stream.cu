// stream.cu — asynchronous record streams: the wire/disk step after
// the per-cell pack. A stream file is a concatenation of standard FORMATS.md payloads
// (.gmmc records or .h2d histogram payloads) plus a binary index `<path>.idx`; see the
// format comment in include/vdfcg.h.
//
// Data path: append() copies the batch D2H into a pinned staging buffer on the context
// stream and records an event; the stream's IO thread waits on that event, CRCs each
// record and fwrite()s the batch. The caller's next kernels overlap the file write; the
// pinned buffers are recycled through a small pool.
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ctx.cuh"

struct vdfcg_stream;

namespace vdfcg {
namespace {

// zlib CRC-32 (reflected 0xEDB88320), slicing-by-8.
struct Crc32 {
  uint32_t t[8][256];
  Crc32() {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      t[0][i] = c;
    }
    for (int s = 1; s < 8; ++s)
      for (int i = 0; i < 256; ++i) t[s][i] = (t[s - 1][i] >> 8) ^ t[0][t[s - 1][i] & 0xff];
  }
  uint32_t operator()(const uint8_t* p, size_t n) const {
    uint32_t c = 0xFFFFFFFFu;
    while (n >= 8) {
      uint32_t a, b;
      std::memcpy(&a, p, 4);
      std::memcpy(&b, p + 4, 4);
      a ^= c;
      c = t[7][a & 0xff] ^ t[6][(a >> 8) & 0xff] ^ t[5][(a >> 16) & 0xff] ^ t[4][a >> 24] ^
          t[3][b & 0xff] ^ t[2][(b >> 8) & 0xff] ^ t[1][(b >> 16) & 0xff] ^ t[0][b >> 24];
      p += 8;
      n -= 8;
    }
    while (n--) c = t[0][(c ^ *p++) & 0xff] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
  }
};
const Crc32& crc_table() {
  static const Crc32 t;
  return t;
}

struct IndexEntry {
  int64_t cell;
  uint64_t offset;
  uint32_t length;
  uint32_t crc;
  double aux;
};
static_assert(sizeof(IndexEntry) == 32, "index entry layout");

struct Job {
  int device = 0;
  cudaEvent_t ready = nullptr;      // null: data already in `buf`
  uint8_t* buf = nullptr;
  size_t cap = 0;
  std::vector<uint32_t> len;        // per record
  std::vector<int64_t> cell;
  std::vector<double> aux;
};

__global__ void densify_kernel(const int64_t* offsets, const int32_t* nnz, const uint32_t* keys,
                               const double* counts, int c0, int n_cells, int64_t bins2,
                               double* dense) {
  for (int c = c0 + blockIdx.x; c < c0 + n_cells; c += gridDim.x) {
    const int64_t off = offsets[c];
    double* out = dense + int64_t(c - c0) * bins2;
    for (int r = threadIdx.x; r < nnz[c]; r += blockDim.x) out[keys[off + r]] = counts[off + r];
  }
}

}  // namespace
}  // namespace vdfcg

using namespace vdfcg;

struct vdfcg_stream {
  std::string path;
  int kind = 0;
  FILE* data = nullptr;
  uint64_t bytes = 0;
  std::vector<IndexEntry> index;
  std::string error;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<Job> queue;
  std::vector<std::pair<uint8_t*, size_t>> pool;
  bool closing = false;
  std::thread io;

  uint8_t* get_buffer(size_t need, size_t* cap) {
    {
      std::lock_guard<std::mutex> g(mu);
      for (size_t i = 0; i < pool.size(); ++i)
        if (pool[i].second >= need) {
          uint8_t* b = pool[i].first;
          *cap = pool[i].second;
          pool.erase(pool.begin() + i);
          return b;
        }
    }
    void* p = nullptr;
    *cap = std::max<size_t>(need, 1 << 20);
    VDFCG_CUDA(cudaMallocHost(&p, *cap));
    return static_cast<uint8_t*>(p);
  }

  void run() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] { return closing || !queue.empty(); });
        if (queue.empty()) return;
        j = std::move(queue.front());
        queue.pop_front();
      }
      if (j.ready) {
        cudaSetDevice(j.device);
        const cudaError_t e = cudaEventSynchronize(j.ready);
        cudaEventDestroy(j.ready);
        if (e != cudaSuccess && error.empty()) error = cudaGetErrorString(e);
      }
      size_t pos = 0;
      for (size_t r = 0; r < j.len.size(); ++r) {
        IndexEntry ie{j.cell[r], bytes + pos, j.len[r], j.len[r] ? crc_table()(j.buf + pos, j.len[r]) : 0u,
                      j.aux[r]};
        index.push_back(ie);
        pos += j.len[r];
      }
      if (pos && error.empty() && std::fwrite(j.buf, 1, pos, data) != pos) error = "stream write failed: " + path;
      bytes += pos;
      std::lock_guard<std::mutex> g(mu);
      pool.emplace_back(j.buf, j.cap);
    }
  }

  void submit(Job&& j) {
    {
      std::lock_guard<std::mutex> g(mu);
      queue.push_back(std::move(j));
    }
    cv.notify_one();
  }
};

namespace {

void begin_ctx(vdfcg_ctx* ctx) {
  if (!ctx) throw InvalidArgument("null vdfcg context");
  VDFCG_CUDA(cudaSetDevice(ctx->device));
  arena_reset(ctx);
}

void put_index(FILE* f, const vdfcg_stream& s) {
  uint8_t head[16] = {'G', 'M', 'I', 'X', 1, static_cast<uint8_t>(s.kind), 0, 0};
  const uint64_t n = s.index.size();
  std::memcpy(head + 8, &n, 8);  // little-endian host (x86-64 / aarch64)
  std::fwrite(head, 1, 16, f);
  std::fwrite(s.index.data(), sizeof(IndexEntry), s.index.size(), f);
}

}  // namespace

extern "C" {

int vdfcg_stream_open(const char* path, int32_t kind, vdfcg_stream** out) {
  return guard_impl([&] {
    if (!path || !out) throw InvalidArgument("null argument");
    if (kind != VDFCG_STREAM_GMMC && kind != VDFCG_STREAM_H2D) throw InvalidArgument("unknown stream kind");
    auto* s = new vdfcg_stream();
    s->path = path;
    s->kind = kind;
    s->data = std::fopen(path, "wb");
    if (!s->data) {
      delete s;
      throw RuntimeError(std::string("cannot open stream file ") + path);
    }
    s->io = std::thread([s] { s->run(); });
    *out = s;
  });
}

int vdfcg_stream_append_records(vdfcg_stream* s, vdfcg_ctx* ctx, const uint8_t* records,
                                const int64_t* record_offsets, int32_t n_cells,
                                int64_t cell_base) {
  return guard_impl([&] {
    begin_ctx(ctx);
    if (!s || !record_offsets || n_cells < 0) throw InvalidArgument("null argument");
    if (s->kind != VDFCG_STREAM_GMMC) throw InvalidArgument("not a .gmmc record stream");
    std::vector<int64_t> off(size_t(n_cells) + 1);
    VDFCG_CUDA(cudaMemcpyAsync(off.data(), record_offsets, off.size() * 8, cudaMemcpyDefault, ctx->stream));
    sync(ctx);
    for (int c = 0; c < n_cells; ++c)
      if (off[c + 1] < off[c]) throw InvalidArgument("record offsets must be non-decreasing");
    const size_t total = size_t(off[n_cells] - off[0]);
    if (total && !records) throw InvalidArgument("null records");
    Job j;
    j.device = ctx->device;
    j.buf = s->get_buffer(total, &j.cap);
    if (total) {
      VDFCG_CUDA(cudaMemcpyAsync(j.buf, records + off[0], total, cudaMemcpyDefault, ctx->stream));
      VDFCG_CUDA(cudaEventCreateWithFlags(&j.ready, cudaEventDisableTiming));
      VDFCG_CUDA(cudaEventRecord(j.ready, ctx->stream));
    }
    for (int c = 0; c < n_cells; ++c) {
      j.len.push_back(static_cast<uint32_t>(off[c + 1] - off[c]));
      j.cell.push_back(cell_base + c);
      j.aux.push_back(0.0);
    }
    s->submit(std::move(j));
  });
}

int vdfcg_stream_append_h2d(vdfcg_stream* s, vdfcg_ctx* ctx, const vdfcg_cells* cells,
                            const vdfcg_cell_bins* bins, int64_t cell_base) {
  return guard_impl([&] {
    begin_ctx(ctx);
    if (!s || !cells || !bins) throw InvalidArgument("null argument");
    if (s->kind != VDFCG_STREAM_H2D) throw InvalidArgument("not an .h2d stream");
    if (cells->dimension != 2) throw InvalidArgument(".h2d payloads are 2D: cells must be 2V");
    if (cells->n_bins < 1 || cells->n_cells < 0 || !cells->cell_offsets)
      throw InvalidArgument("invalid cells");
    if (!bins->nnz || !bins->keys || !bins->counts || !bins->out_of_range)
      throw InvalidArgument("cell bins: nnz, keys, counts, out_of_range are required");
    const int nc = cells->n_cells;
    const int64_t bins2 = int64_t(cells->n_bins) * cells->n_bins;
    const int64_t n = cells->n_particles;
    const int64_t* offs = stage_in(ctx, cells->cell_offsets, size_t(nc) + 1).dev;
    const int32_t* nnz = stage_in(ctx, bins->nnz, size_t(nc)).dev;
    const uint32_t* keys = stage_in(ctx, bins->keys, size_t(n)).dev;
    const double* counts = stage_in(ctx, bins->counts, size_t(n)).dev;
    std::vector<double> oor(nc);
    VDFCG_CUDA(cudaMemcpyAsync(oor.data(), bins->out_of_range, size_t(nc) * 8, cudaMemcpyDefault, ctx->stream));
    // chunks of <= 256 MB of dense payload
    const int chunk = static_cast<int>(std::max<int64_t>(1, (int64_t(256) << 20) / (bins2 * 8)));
    double* dense = arena<double>(ctx, size_t(std::min(chunk, std::max(nc, 1))) * bins2);
    for (int c0 = 0; c0 < nc; c0 += chunk) {
      const int m = std::min(chunk, nc - c0);
      const size_t bytes = size_t(m) * bins2 * 8;
      VDFCG_CUDA(cudaMemsetAsync(dense, 0, bytes, ctx->stream));
      VDFCG_LAUNCH(ctx, "densify_h2d",
                   densify_kernel<<<std::min(m, ctx->sm_count * 8), 256, 0, ctx->stream>>>(
                       offs, nnz, keys, counts, c0, m, bins2, dense));
      Job j;
      j.device = ctx->device;
      j.buf = s->get_buffer(bytes, &j.cap);
      VDFCG_CUDA(cudaMemcpyAsync(j.buf, dense, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      VDFCG_CUDA(cudaEventCreateWithFlags(&j.ready, cudaEventDisableTiming));
      VDFCG_CUDA(cudaEventRecord(j.ready, ctx->stream));
      sync(ctx);  // the next chunk reuses `dense`; oor is final
      for (int c = c0; c < c0 + m; ++c) {
        j.len.push_back(static_cast<uint32_t>(bins2 * 8));
        j.cell.push_back(cell_base + c);
        j.aux.push_back(oor[c]);
      }
      s->submit(std::move(j));
    }
  });
}

int vdfcg_stream_close(vdfcg_stream* s, int64_t* n_records, int64_t* n_bytes) {
  return guard_impl([&] {
    if (!s) throw InvalidArgument("null stream");
    {
      std::lock_guard<std::mutex> g(s->mu);
      s->closing = true;
    }
    s->cv.notify_one();
    if (s->io.joinable()) s->io.join();
    std::string err = s->error;
    if (s->data) std::fclose(s->data);
    if (err.empty()) {
      FILE* f = std::fopen((s->path + ".idx").c_str(), "wb");
      if (!f) err = "cannot write stream index " + s->path + ".idx";
      else {
        put_index(f, *s);
        std::fclose(f);
      }
    }
    if (n_records) *n_records = static_cast<int64_t>(s->index.size());
    if (n_bytes) *n_bytes = static_cast<int64_t>(s->bytes);
    for (auto& b : s->pool) cudaFreeHost(b.first);
    delete s;
    if (!err.empty()) throw RuntimeError(err);
  });
}

}  // extern "C"
