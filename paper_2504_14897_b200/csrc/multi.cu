// multi.cu — one host process driving several B200s.
//
// Spatial cells are independent fits (run_pipeline fans the parts out with
// no coordination, pipeline.cpp:340-345), so the cells of one species are split into
// contiguous ranges balanced by PARTICLE count (prefix sum of the per-cell counts), and each
// device runs bin -> fit -> pack on its range with its own context, stream set and host
// thread — no collective on the data path. The only cross-device step is the final gather
// (pipeline.cpp:349-353 gathers every part and writes the artifacts): each device's .gmmc
// records land in a per-device host buffer (the D2H the single-device call already does,
// from pinned staging), then are concatenated in cell order into the caller's record buffer
// with global record offsets, so the result is byte-identical to a one-device call.
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "api.cuh"
#include "ctx.cuh"

struct vdfcg_multi {
  std::vector<int> devices;
  std::vector<vdfcg_ctx*> ctx;  // one per device, each used by one worker thread at a time
};

namespace vdfcg {
namespace {

// Cell ranges [cb[r], cb[r+1]) with about total/n_parts particles each: cb[r] is the cell
// boundary whose particle prefix is nearest to r * total / n_parts (ties: the lower one).
void partition(const int64_t* off, int n_cells, int n_parts, int32_t* cb) {
  const int64_t base = off[0], total = off[n_cells] - off[0];
  cb[0] = 0;
  for (int r = 1; r < n_parts; ++r) {
    const int64_t target = base + (total * r) / n_parts;
    int c = static_cast<int>(std::lower_bound(off, off + n_cells + 1, target) - off);
    if (c > 0 && (c > n_cells || target - off[c - 1] <= off[c] - target)) --c;
    c = std::min(std::max(c, static_cast<int>(cb[r - 1])), n_cells);
    cb[r] = c;
  }
  cb[n_parts] = n_cells;
}

struct WorkerResult {
  int rc = VDFCG_OK;
  std::string msg;
  std::vector<uint8_t> records;
  std::vector<int64_t> offsets;
};

void rethrow(int rc, const std::string& msg) {
  if (rc == VDFCG_INVALID_ARGUMENT) throw InvalidArgument(msg);
  if (rc == VDFCG_REPAIR_FAILED) throw RepairFailed(msg);
  if (rc == VDFCG_CUDA_ERROR) throw CudaError(msg);
  throw RuntimeError(msg);
}

}  // namespace
}  // namespace vdfcg

using namespace vdfcg;

extern "C" {

int vdfcg_partition_cells(const int64_t* cell_offsets, int32_t n_cells, int32_t n_parts,
                          int32_t* cell_begin) {
  return guard_impl([&] {
    if (!cell_offsets || !cell_begin) throw InvalidArgument("null argument");
    if (n_cells < 0 || n_parts < 1) throw InvalidArgument("partition: n_cells >= 0 and n_parts >= 1 required");
    for (int c = 0; c < n_cells; ++c)
      if (cell_offsets[c + 1] < cell_offsets[c]) throw InvalidArgument("cell_offsets must be non-decreasing");
    partition(cell_offsets, n_cells, n_parts, cell_begin);
  });
}

int vdfcg_multi_create(const int32_t* devices, int32_t n_devices, vdfcg_multi** out) {
  return guard_impl([&] {
    if (!out || (!devices && n_devices > 0)) throw InvalidArgument("null argument");
    if (n_devices < 1) throw InvalidArgument("at least one device is required");
    auto* m = new vdfcg_multi();
    for (int i = 0; i < n_devices; ++i) {
      vdfcg_ctx* c = nullptr;
      const int rc = vdfcg_ctx_create(devices[i], &c);
      if (rc != VDFCG_OK) {
        const std::string msg = vdfcg_last_error();
        for (auto* x : m->ctx) vdfcg_ctx_destroy(x);
        delete m;
        rethrow(rc, msg);
      }
      m->devices.push_back(devices[i]);
      m->ctx.push_back(c);
    }
    *out = m;
  });
}

int vdfcg_multi_destroy(vdfcg_multi* m) {
  return guard_impl([&] {
    if (!m) return;
    for (auto* c : m->ctx) vdfcg_ctx_destroy(c);
    delete m;
  });
}

int32_t vdfcg_multi_device_count(const vdfcg_multi* m) { return m ? static_cast<int32_t>(m->ctx.size()) : 0; }

int vdfcg_multi_context(vdfcg_multi* m, int32_t index, vdfcg_ctx** out) {
  return guard_impl([&] {
    if (!m || !out) throw InvalidArgument("null argument");
    if (index < 0 || index >= static_cast<int>(m->ctx.size())) throw InvalidArgument("device index out of range");
    *out = m->ctx[index];
  });
}

int vdfcg_multi_compress_cells(vdfcg_multi* m, const vdfcg_cells* cells, const vdfcg_fit_config* cfg,
                               vdfcg_cell_bins* bins, vdfcg_cell_results* out,
                               const vdfcg_model_meta* meta, uint8_t* records, int64_t capacity,
                               int64_t* record_offsets, int32_t* cell_begin) {
  return guard_impl([&] {
    if (!m || !cells || !cfg || !out) throw InvalidArgument("null argument");
    if (!cells->cell_offsets || is_device_pointer(cells->cell_offsets))
      throw InvalidArgument("multi-device compress_cells takes host cell_offsets");
    const int n_dev = static_cast<int>(m->ctx.size());
    const int nc = cells->n_cells;
    const int d = cells->dimension;
    if (nc < 0) throw InvalidArgument("negative sizes");
    const int64_t* off = cells->cell_offsets;
    if (nc > 0 && (off[0] < 0 || off[nc] > cells->n_particles)) throw InvalidArgument("cell_offsets out of range");
    for (int c = 0; c < nc; ++c)
      if (off[c + 1] < off[c]) throw InvalidArgument("cell_offsets must be non-decreasing");
    std::vector<int32_t> cb(n_dev + 1);
    partition(off, nc, n_dev, cb.data());
    const int K = out->capacity_components;
    const bool pack = records || record_offsets;
    if (pack && (!meta || !record_offsets)) throw InvalidArgument("packing needs meta and record_offsets");
    // largest record: header (26 + 16 d + label) + K components of 1 + d + d(d+1)/2 doubles
    const int64_t max_rec = 26 + 16 * int64_t(d) + (meta ? meta->label_len : 0) +
                            int64_t(K) * (1 + d + d * (d + 1) / 2) * 8;
    // every device runs the EM launch shape of the whole batch: fits bitwise-identical to a
    // one-device call
    EmShape shape;
    shape.cells = nc;
    shape.avg = nc ? double(off[nc] - off[0]) / nc : 0.0;
    std::vector<WorkerResult> res(n_dev);
    std::vector<std::thread> th;
    for (int r = 0; r < n_dev; ++r) {
      th.emplace_back([&, r] {
        const int c0 = cb[r], c1 = cb[r + 1];
        WorkerResult& R = res[r];
        if (c1 <= c0) return;
        // the device's cell range as a self-contained batch (offsets rebased to 0)
        const int64_t p0 = off[c0];
        std::vector<int64_t> lo(size_t(c1 - c0) + 1);
        for (int c = c0; c <= c1; ++c) lo[c - c0] = off[c] - p0;
        vdfcg_cells sub = *cells;
        sub.n_cells = c1 - c0;
        sub.n_particles = off[c1] - p0;
        sub.cell_offsets = lo.data();
        for (int a = 0; a < d; ++a) sub.velocity[a] = cells->velocity[a] ? cells->velocity[a] + p0 : nullptr;
        sub.weights = cells->weights ? cells->weights + p0 : nullptr;
        vdfcg_cell_bins sb{}, *sbp = nullptr;
        if (bins && bins->nnz) {
          sb.nnz = bins->nnz + c0;
          sb.keys = bins->keys + p0;
          sb.counts = bins->counts + p0;
          sb.out_of_range = bins->out_of_range + c0;
          sb.in_range = bins->in_range + c0;
          sbp = &sb;
        }
        vdfcg_cell_results so = *out;
        const int64_t Kc = K;
        so.status = out->status + c0;
        so.components = out->components + c0;
        so.iterations = out->iterations + c0;
        so.converged = out->converged + c0;
        so.weights = out->weights + c0 * Kc;
        so.means = out->means + c0 * Kc * d;
        so.covariances = out->covariances + c0 * Kc * d * d;
        so.final_loglik = out->final_loglik + c0;
        if (out->loglik_trace) so.loglik_trace = out->loglik_trace + int64_t(c0) * out->capacity_trace;
        if (out->n_events) so.n_events = out->n_events + c0;
        if (out->event_iteration) so.event_iteration = out->event_iteration + c0 * Kc;
        if (out->event_component) so.event_component = out->event_component + c0 * Kc;
        if (out->event_weight) so.event_weight = out->event_weight + c0 * Kc;
        int64_t cap = 0;
        if (pack) {
          cap = max_rec * (c1 - c0);
          R.records.resize(size_t(cap));
          R.offsets.resize(size_t(c1 - c0) + 1);
        }
        R.rc = compress_cells_shaped(m->ctx[r], &sub, cfg, nullptr, sbp, &so, pack ? meta : nullptr,
                                     pack ? R.records.data() : nullptr, cap,
                                     pack ? R.offsets.data() : nullptr, shape);
        if (R.rc != VDFCG_OK) R.msg = vdfcg_last_error();
      });
    }
    for (auto& t : th) t.join();
    for (int r = 0; r < n_dev; ++r)
      if (res[r].rc != VDFCG_OK) rethrow(res[r].rc, res[r].msg);
    if (cell_begin) std::copy(cb.begin(), cb.end(), cell_begin);
    if (!pack) return;
    // gather: device ranges in cell order -> one record buffer, global offsets
    int64_t pos = 0;
    record_offsets[0] = 0;
    for (int r = 0; r < n_dev; ++r) {
      const int c0 = cb[r], c1 = cb[r + 1];
      if (c1 <= c0) continue;
      const int64_t bytes = res[r].offsets[size_t(c1 - c0)];
      if (pos + bytes > capacity) throw InvalidArgument("compress_cells: record capacity too small");
      if (records && bytes) std::memcpy(records + pos, res[r].records.data(), size_t(bytes));
      for (int c = c0; c < c1; ++c) record_offsets[c + 1] = pos + res[r].offsets[size_t(c - c0) + 1];
      pos += bytes;
    }
  });
}

}  // extern "C"
