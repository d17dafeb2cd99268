"""Cell-batched compression: the GPU generalisation of the reference's per-part fan-out
(pipeline.cpp:76-104, 130-160, 340-349): every spatial cell of a species is binned into
its own velocity histogram (2V or 3V) and fitted with the same
FitConfig (pipeline.cpp:144), all on the device.

Arrays may be numpy (host; the library stages them through the context stream — the
end-to-end path) or torch CUDA tensors (device-resident; no copies).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _abi, _marshal
from .types import AffineMap, FitConfig, GaussianComponent, GmmModel, ModelMeta


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        return x.data_ptr()
    return x.ctypes.data


def _empty(like, shape, kind: str):
    """numpy on host / torch on the device of `like`."""
    if _is_torch(like):
        import torch
        dt = {"f64": torch.float64, "i32": torch.int32, "u32": torch.int32, "i64": torch.int64,
              "u8": torch.uint8}[kind]
        # host outputs follow the input's pinnedness (pinned D2H is asynchronous + faster)
        pin = like.device.type == "cpu" and like.is_pinned()
        return torch.empty(shape, dtype=dt, device=like.device, pin_memory=pin)
    dt = {"f64": np.float64, "i32": np.int32, "u32": np.uint32, "i64": np.int64, "u8": np.uint8}[kind]
    return np.empty(shape, dtype=dt)


def _ctx(*arrays):
    """The calling thread's library context, ordered with torch: when any argument is a
    CUDA tensor the context runs on that device's *current torch stream*, so the
    library's kernels follow the ops that produced the inputs and precede the ops that
    consume the outputs (no host synchronisation needed). Host (numpy) calls are
    synchronous."""
    api = _api()
    for a in arrays:
        if _is_torch(a) and a.is_cuda:
            import torch
            ctx = api.context(a.device.index)
            ctx.set_stream(torch.cuda.current_stream(a.device).cuda_stream)
            return ctx
    return api.context()


def _api():
    from . import api
    return api


class CellBatch:
    """Particles of one species grouped by spatial cell (vdfcg_cells).

    velocity: sequence of d axis arrays (u, v[, w]), each n_particles long, or an
    (n, d) array; cell_offsets: n_cells+1 int64 (cell c owns [off[c], off[c+1]))."""

    def __init__(self, velocity, cell_offsets, n_bins: int, lo, hi, weights=None):
        if not isinstance(velocity, (list, tuple)):
            if _is_torch(velocity):
                velocity = [velocity[:, a].contiguous() for a in range(velocity.shape[1])]
            else:
                v = np.asarray(velocity, dtype=np.float64)
                velocity = [np.ascontiguousarray(v[:, a]) for a in range(v.shape[1])]
        self.axes = list(velocity)
        self.d = len(self.axes)
        self.offsets = cell_offsets
        self.weights = weights
        self.n_bins = int(n_bins)
        self.lo = [float(x) for x in lo]
        self.hi = [float(x) for x in hi]
        self.n = int(self.axes[0].shape[0])
        self.n_cells = int(cell_offsets.shape[0]) - 1
        s = _abi.Cells()
        s.dimension = self.d
        s.n_particles = self.n
        for a in range(self.d):
            s.velocity[a] = _ptr(self.axes[a])
        s.weights = _ptr(weights)
        s.n_cells = self.n_cells
        s.cell_offsets = _ptr(cell_offsets)
        s.n_bins = self.n_bins
        for a in range(self.d):
            s.lo[a] = self.lo[a]
            s.hi[a] = self.hi[a]
        self.struct = s

    @property
    def on_device(self) -> bool:
        return _is_torch(self.axes[0]) and self.axes[0].is_cuda


@dataclass
class CellBins:
    nnz: object
    keys: object
    counts: object
    out_of_range: object
    in_range: object

    def struct(self) -> _abi.CellBins:
        return _abi.CellBins(_ptr(self.nnz), _ptr(self.keys), _ptr(self.counts),
                             _ptr(self.out_of_range), _ptr(self.in_range))

    @staticmethod
    def alloc(batch: CellBatch) -> "CellBins":
        like = batch.axes[0]
        return CellBins(_empty(like, (batch.n_cells,), "i32"), _empty(like, (max(batch.n, 1),), "u32"),
                        _empty(like, (max(batch.n, 1),), "f64"), _empty(like, (batch.n_cells,), "f64"),
                        _empty(like, (batch.n_cells,), "f64"))


class CellResults:
    """Per-cell fit results (vdfcg_cell_results), capacity K components."""

    FIELDS = ("status", "components", "iterations", "converged", "weights", "means",
              "covariances", "final_loglik", "loglik_trace", "n_events", "event_iteration",
              "event_component", "event_weight")

    def __init__(self, like, n_cells: int, d: int, k: int, trace: int = 0, events: bool = True):
        self.n_cells, self.d, self.k, self.trace_cap = n_cells, d, k, trace
        self.status = _empty(like, (n_cells,), "i32")
        self.components = _empty(like, (n_cells,), "i32")
        self.iterations = _empty(like, (n_cells,), "i32")
        self.converged = _empty(like, (n_cells,), "i32")
        self.weights = _empty(like, (n_cells * k,), "f64")
        self.means = _empty(like, (n_cells * k * d,), "f64")
        self.covariances = _empty(like, (n_cells * k * d * d,), "f64")
        self.final_loglik = _empty(like, (n_cells,), "f64")
        self.loglik_trace = _empty(like, (max(n_cells * trace, 1),), "f64") if trace else None
        self.n_events = _empty(like, (n_cells,), "i32") if events else None
        self.event_iteration = _empty(like, (n_cells * k,), "i32") if events else None
        self.event_component = _empty(like, (n_cells * k,), "i32") if events else None
        self.event_weight = _empty(like, (n_cells * k,), "f64") if events else None

    def struct(self) -> _abi.CellResults:
        s = _abi.CellResults()
        s.capacity_components = self.k
        s.capacity_trace = self.trace_cap
        for f in self.FIELDS:
            setattr(s, f, _ptr(getattr(self, f)))
        return s

    def numpy(self) -> "CellResults":
        """Host copy (numpy) of device results."""
        out = CellResults.__new__(CellResults)
        out.n_cells, out.d, out.k, out.trace_cap = self.n_cells, self.d, self.k, self.trace_cap
        for f in self.FIELDS:
            v = getattr(self, f)
            if v is not None and _is_torch(v):
                v = v.cpu().numpy()
            setattr(out, f, v)
        return out

    def model(self, c: int) -> GmmModel:
        """Cell c's fitted model (canonical, data space)."""
        r = self if not _is_torch(self.weights) else self.numpy()
        d, k = r.d, r.k
        m = int(r.components[c])
        comps = []
        for i in range(m):
            j = c * k + i
            comps.append(GaussianComponent(float(r.weights[j]), np.array(r.means[j * d:(j + 1) * d]),
                                           np.array(r.covariances[j * d * d:(j + 1) * d * d]).reshape(d, d)))
        return GmmModel(comps, AffineMap.identity(d), d)


def _check(rc):
    _marshal.check(rc, _api().last_error)


def bin_cells(batch: CellBatch, out: Optional[CellBins] = None) -> CellBins:
    api = _api()
    out = out or CellBins.alloc(batch)
    bs = out.struct()
    _check(api.lib().vdfcg_bin_cells(_ctx(batch.axes[0]).handle, C.byref(batch.struct), C.byref(bs)))
    return out


def fit_cells(batch: CellBatch, bins: CellBins, config: FitConfig, trace: bool = False,
              out: Optional[CellResults] = None,
              warm: Optional[CellResults] = None) -> CellResults:
    """Fit every cell (same FitConfig, pipeline.cpp:144). `warm`: the previous cycle's
    results — each cell restarts from its own model (time series, pipeline.cpp:482-564)."""
    api = _api()
    d = batch.d
    wm = _abi.ModelBuffers.from_model(config.warm_start) if config.warm_start is not None else None
    cfg = _abi.fit_config_struct(config, d, wm)
    k = max(config.initial_components, wm.k if wm else 0, warm.k if warm is not None else 0)
    out = out or CellResults(batch.axes[0], batch.n_cells, d, k,
                             config.max_em_iterations if trace else 0)
    bs = bins.struct()
    rs = out.struct()
    ws = warm.struct() if warm is not None else None
    _check(api.lib().vdfcg_fit_cells_warm(_ctx(batch.axes[0], out.weights).handle, C.byref(batch.struct), C.byref(bs),
                                          C.byref(cfg), C.byref(ws) if ws is not None else None,
                                          C.byref(rs)))
    return out


def pack_cells(results: CellResults, meta: ModelMeta):
    """.gmmc record per cell (FORMATS.md) -> (records, offsets[n_cells+1])."""
    api = _api()
    like = results.weights
    ms, _keep = _abi.meta_struct(meta, results.d)
    per = 26 + 16 * results.d + ms.label_len + results.k * (1 + results.d + results.d * (results.d + 1) // 2) * 8
    cap = results.n_cells * per
    rec = _empty(like, (max(cap, 1),), "u8")
    offs = _empty(like, (results.n_cells + 1,), "i64")
    rs = results.struct()
    _check(api.lib().vdfcg_pack_cells(_ctx(results.weights).handle, results.n_cells, results.d,
                                      C.byref(rs), C.byref(ms), _ptr(rec), cap, _ptr(offs)))
    total = int(offs[-1])
    return rec[:total], offs


def compress_cells(batch: CellBatch, config: FitConfig, meta: Optional[ModelMeta] = None,
                   trace: bool = False, bins: Optional[CellBins] = None,
                   results: Optional[CellResults] = None, keep_bins: bool = True,
                   warm: Optional[CellResults] = None):
    """bin -> fit (-> pack) in one device pass. Returns (bins, results, records, offsets).
    `warm`: per-cell warm start from the previous cycle's results (see fit_cells)."""
    api = _api()
    d = batch.d
    wm = _abi.ModelBuffers.from_model(config.warm_start) if config.warm_start is not None else None
    cfg = _abi.fit_config_struct(config, d, wm)
    k = max(config.initial_components, wm.k if wm else 0, warm.k if warm is not None else 0)
    like = batch.axes[0]
    if keep_bins and bins is None:
        bins = CellBins.alloc(batch)
    results = results or CellResults(like, batch.n_cells, d, k, config.max_em_iterations if trace else 0)
    bs = bins.struct() if bins is not None else _abi.CellBins()
    rs = results.struct()
    rec = offs = None
    cap = 0
    ms = None
    if meta is not None:
        ms, _keep = _abi.meta_struct(meta, d)
        per = 26 + 16 * d + ms.label_len + k * (1 + d + d * (d + 1) // 2) * 8
        cap = batch.n_cells * per
        rec = _empty(like, (max(cap, 1),), "u8")
        offs = _empty(like, (batch.n_cells + 1,), "i64")
    ws = warm.struct() if warm is not None else None
    _check(api.lib().vdfcg_compress_cells_warm(
        _ctx(batch.axes[0], results.weights).handle, C.byref(batch.struct), C.byref(cfg),
        C.byref(ws) if ws is not None else None, C.byref(bs) if bins is not None else None,
        C.byref(rs), C.byref(ms) if ms is not None else None, _ptr(rec), cap, _ptr(offs)))
    if rec is not None:
        rec = rec[:int(offs[-1])]
    return bins, results, rec, offs


class ParticleBatch:
    """Particles of one species in ANY order with an int32 cell id each (vdfcg_particles):
    the per-particle cell-index input of a PIC code. velocity: d axis arrays (or an (n, d)
    array), cell: n int32 ids in [0, n_cells)."""

    def __init__(self, velocity, cell, n_cells: int, n_bins: int, lo, hi, weights=None):
        if not isinstance(velocity, (list, tuple)):
            if _is_torch(velocity):
                velocity = [velocity[:, a].contiguous() for a in range(velocity.shape[1])]
            else:
                v = np.asarray(velocity, dtype=np.float64)
                velocity = [np.ascontiguousarray(v[:, a]) for a in range(v.shape[1])]
        self.axes = list(velocity)
        self.d = len(self.axes)
        self.cell = cell
        self.weights = weights
        self.n_cells = int(n_cells)
        self.n_bins = int(n_bins)
        self.lo = [float(x) for x in lo]
        self.hi = [float(x) for x in hi]
        self.n = int(self.axes[0].shape[0])
        s = _abi.Particles()
        s.dimension = self.d
        s.n_particles = self.n
        for a in range(self.d):
            s.velocity[a] = _ptr(self.axes[a])
        s.weights = _ptr(weights)
        s.cell = _ptr(cell)
        s.n_cells = self.n_cells
        s.n_bins = self.n_bins
        for a in range(self.d):
            s.lo[a] = self.lo[a]
            s.hi[a] = self.hi[a]
        self.struct = s

    def grouped(self, cell_offsets) -> CellBatch:
        """The cell-grouped view for fit_cells / cell_metrics (which read only the geometry
        and cell_offsets, never the velocities — these stay in the caller's order)."""
        return CellBatch(self.axes, cell_offsets, self.n_bins, self.lo, self.hi, self.weights)


def bin_cells_indexed(batch: ParticleBatch, out: Optional[CellBins] = None):
    """Histogram every cell of an unsorted particle array. Returns (cell_offsets, bins);
    bins are indexed by cell_offsets exactly like bin_cells' output."""
    api = _api()
    like = batch.axes[0]
    offs = _empty(like, (batch.n_cells + 1,), "i64")
    if out is None:
        out = CellBins(_empty(like, (batch.n_cells,), "i32"), _empty(like, (max(batch.n, 1),), "u32"),
                       _empty(like, (max(batch.n, 1),), "f64"), _empty(like, (batch.n_cells,), "f64"),
                       _empty(like, (batch.n_cells,), "f64"))
    bs = out.struct()
    _check(api.lib().vdfcg_bin_cells_indexed(_ctx(like).handle, C.byref(batch.struct), _ptr(offs),
                                             C.byref(bs)))
    return offs, out


def compress_cells_indexed(batch: ParticleBatch, config: FitConfig,
                           meta: Optional[ModelMeta] = None, trace: bool = False,
                           keep_bins: bool = True, warm: Optional[CellResults] = None):
    """group by cell -> bin -> fit (-> pack) on the device. Returns
    (cell_offsets, bins, results, records, record_offsets); cell c is cell id c.
    `warm`: the previous cycle's results — cell c restarts from its own model."""
    api = _api()
    d = batch.d
    wm = _abi.ModelBuffers.from_model(config.warm_start) if config.warm_start is not None else None
    cfg = _abi.fit_config_struct(config, d, wm)
    k = max(config.initial_components, wm.k if wm else 0, warm.k if warm is not None else 0)
    like = batch.axes[0]
    offs = _empty(like, (batch.n_cells + 1,), "i64")
    bins = None
    if keep_bins:
        bins = CellBins(_empty(like, (batch.n_cells,), "i32"), _empty(like, (max(batch.n, 1),), "u32"),
                        _empty(like, (max(batch.n, 1),), "f64"), _empty(like, (batch.n_cells,), "f64"),
                        _empty(like, (batch.n_cells,), "f64"))
    results = CellResults(like, batch.n_cells, d, k, config.max_em_iterations if trace else 0)
    bs = bins.struct() if bins is not None else None
    rs = results.struct()
    rec = roffs = None
    cap = 0
    ms = None
    if meta is not None:
        ms, _keep = _abi.meta_struct(meta, d)
        per = 26 + 16 * d + ms.label_len + k * (1 + d + d * (d + 1) // 2) * 8
        cap = batch.n_cells * per
        rec = _empty(like, (max(cap, 1),), "u8")
        roffs = _empty(like, (batch.n_cells + 1,), "i64")
    ws = warm.struct() if warm is not None else None
    _check(api.lib().vdfcg_compress_cells_indexed_warm(
        _ctx(like, results.weights).handle, C.byref(batch.struct), C.byref(cfg),
        C.byref(ws) if ws is not None else None, _ptr(offs),
        C.byref(bs) if bs is not None else None, C.byref(rs),
        C.byref(ms) if ms is not None else None, _ptr(rec), cap, _ptr(roffs)))
    if rec is not None:
        rec = rec[:int(roffs[-1])]
    return offs, bins, results, rec, roffs


def partition_cells(cell_offsets, n_parts: int) -> np.ndarray:
    """Contiguous cell ranges balanced by particle count (vdfcg_partition_cells, host only):
    part r owns cells [b[r], b[r+1])."""
    off = np.ascontiguousarray(np.asarray(cell_offsets, dtype=np.int64))
    out = np.zeros(n_parts + 1, dtype=np.int32)
    _check(_api().lib().vdfcg_partition_cells(off.ctypes.data, len(off) - 1, int(n_parts), out.ctypes.data))
    return out


class MultiDevice:
    """Several devices driven from this process (vdfcg_multi): one context, stream set and
    host thread per device; cells split by particle count; records gathered in cell order."""

    def __init__(self, devices):
        api = _api()
        self.devices = [int(x) for x in devices]
        arr = (C.c_int32 * len(self.devices))(*self.devices)
        h = C.c_void_p()
        _check(api.lib().vdfcg_multi_create(arr, len(self.devices), C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            _api().lib().vdfcg_multi_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def compress_cells(self, batch: CellBatch, config: FitConfig, meta: Optional[ModelMeta] = None,
                       trace: bool = False, keep_bins: bool = False):
        """compress_cells over every device (host numpy inputs). Returns
        (bins or None, results, records, record_offsets, cell_begin)."""
        d = batch.d
        wm = _abi.ModelBuffers.from_model(config.warm_start) if config.warm_start is not None else None
        cfg = _abi.fit_config_struct(config, d, wm)
        k = max(config.initial_components, wm.k if wm else 0)
        like = batch.axes[0]
        bins = CellBins.alloc(batch) if keep_bins else None
        results = CellResults(like, batch.n_cells, d, k, config.max_em_iterations if trace else 0)
        rec = offs = None
        cap = 0
        ms = None
        if meta is not None:
            ms, _keep = _abi.meta_struct(meta, d)
            per = 26 + 16 * d + ms.label_len + k * (1 + d + d * (d + 1) // 2) * 8
            cap = batch.n_cells * per
            rec = _empty(like, (max(cap, 1),), "u8")
            offs = _empty(like, (batch.n_cells + 1,), "i64")
        cb = np.zeros(len(self.devices) + 1, dtype=np.int32)
        bs = bins.struct() if bins is not None else None
        rs = results.struct()
        _check(_api().lib().vdfcg_multi_compress_cells(
            self.handle, C.byref(batch.struct), C.byref(cfg), C.byref(bs) if bs is not None else None,
            C.byref(rs), C.byref(ms) if ms is not None else None, _ptr(rec), cap, _ptr(offs),
            cb.ctypes.data))
        if rec is not None:
            rec = rec[:int(offs[-1])]
        return bins, results, rec, offs, cb


class CellMetrics:
    """Per-cell MetricsReport fields (vdfcg_cell_metrics), one array per field."""

    FIELDS = _abi.METRIC_FIELDS

    def __init__(self, like, n_cells: int):
        self.n_cells = n_cells
        for f in self.FIELDS:
            setattr(self, f, _empty(like, (n_cells,), "f64"))

    def struct(self) -> _abi.CellMetrics:
        return _abi.CellMetrics(*[_ptr(getattr(self, f)) for f in self.FIELDS])

    def report(self, c: int):
        """Cell c as a MetricsReport (metrics.hpp:39-54)."""
        from ._metrics import MetricsReport
        vals = {f: float(getattr(self, f)[c]) for f in MetricsReport.FIELDS}
        return MetricsReport(**vals)


def cell_metrics(batch: CellBatch, bins: CellBins, results: CellResults,
                 out: Optional[CellMetrics] = None) -> CellMetrics:
    """assemble_metrics (pipeline.cpp:106-128) for every cell, on the device: JSD and both
    KL divergences between the cell histogram and the model pdf on the bins^d grid,
    weighted log-likelihood, BIC (both n's), moment errors, compression ratios."""
    api = _api()
    out = out or CellMetrics(batch.axes[0], batch.n_cells)
    bs, rs, ms = bins.struct(), results.struct(), out.struct()
    _check(api.lib().vdfcg_metrics_cells(_ctx(batch.axes[0], results.weights).handle, C.byref(batch.struct), C.byref(bs),
                                         C.byref(rs), C.byref(ms)))
    return out


def synth_cells(d: int, cell_offsets, seed: int, species: int, u, v, w=None,
                cell_base: int = 0) -> None:
    """Deterministic synthetic plasma cells into device tensors (tests/bench data).
    cell_offsets: GLOBAL particle offsets of cells [cell_base, cell_base + n)."""
    api = _api()
    _check(api.lib().vdfcg_synth_cells(_ctx(u).handle, d, int(cell_offsets.shape[0]) - 1,
                                       _ptr(cell_offsets), int(cell_base),
                                       seed & 0xFFFFFFFFFFFFFFFF, species, _ptr(u), _ptr(v),
                                       _ptr(w)))
