"""ctypes mirror of include/vdfcg.h (structs and converters only — no compute).

Shared by the product wrapper (``api.py``, which loads libvdfcg.so) and by the
test-only oracle wrapper (``oracle/oracle.py``), so both sides are fed identical
buffers.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

from .types import GaussianComponent, GmmModel, AffineMap

VDFCG_OK = 0
VDFCG_INVALID_ARGUMENT = 1
VDFCG_RUNTIME_ERROR = 2
VDFCG_REPAIR_FAILED = 3
VDFCG_CUDA_ERROR = 4
VDFCG_CODEC_ERROR = 5
MAX_COMPONENTS = 16

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "vdfcg.h")

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int32)
lp = C.POINTER(C.c_int64)
up = C.POINTER(C.c_uint32)
bp = C.POINTER(C.c_uint8)


class Model(C.Structure):
    _fields_ = [("dimension", C.c_int32), ("components", C.c_int32), ("weights", dp),
                ("means", dp), ("covariances", dp), ("scale", dp), ("offset", dp)]


class FitConfig(C.Structure):
    _fields_ = [("initial_components", C.c_int32), ("max_em_iterations", C.c_int32),
                ("prune_threshold", C.c_double), ("prune_check_interval", C.c_int32),
                ("loglik_rel_tolerance", C.c_double), ("seed", C.c_uint64),
                ("has_temperature", C.c_int32), ("temperature", C.c_double * 3),
                ("warm_start", C.POINTER(Model)), ("estep_fp32", C.c_int32)]


class FitResult(C.Structure):
    _fields_ = [("capacity_components", C.c_int32), ("capacity_trace", C.c_int32),
                ("model", Model), ("loglik_trace", dp), ("trace_len", C.c_int32),
                ("iterations_used", C.c_int32), ("converged", C.c_int32),
                ("n_events", C.c_int32), ("event_iteration", ip), ("event_component", ip),
                ("event_weight", dp)]


class ModelMeta(C.Structure):
    _fields_ = [("species_label", C.c_char_p), ("label_len", C.c_int32), ("plane", C.c_int32),
                ("cycle", C.c_int64), ("range_lo", C.c_double * 3),
                ("range_hi", C.c_double * 3)]


class Cells(C.Structure):
    _fields_ = [("dimension", C.c_int32), ("n_particles", C.c_int64),
                ("velocity", C.c_void_p * 3), ("weights", C.c_void_p), ("n_cells", C.c_int32),
                ("cell_offsets", C.c_void_p), ("n_bins", C.c_int32), ("lo", C.c_double * 3),
                ("hi", C.c_double * 3)]


class Particles(C.Structure):
    _fields_ = [("dimension", C.c_int32), ("n_particles", C.c_int64),
                ("velocity", C.c_void_p * 3), ("weights", C.c_void_p), ("cell", C.c_void_p),
                ("n_cells", C.c_int32), ("n_bins", C.c_int32), ("lo", C.c_double * 3),
                ("hi", C.c_double * 3)]


class CellBins(C.Structure):
    _fields_ = [("nnz", C.c_void_p), ("keys", C.c_void_p), ("counts", C.c_void_p),
                ("out_of_range", C.c_void_p), ("in_range", C.c_void_p)]


class CellResults(C.Structure):
    _fields_ = [("capacity_components", C.c_int32), ("capacity_trace", C.c_int32),
                ("status", C.c_void_p), ("components", C.c_void_p), ("iterations", C.c_void_p),
                ("converged", C.c_void_p), ("weights", C.c_void_p), ("means", C.c_void_p),
                ("covariances", C.c_void_p), ("final_loglik", C.c_void_p),
                ("loglik_trace", C.c_void_p), ("n_events", C.c_void_p),
                ("event_iteration", C.c_void_p), ("event_component", C.c_void_p),
                ("event_weight", C.c_void_p)]


METRIC_FIELDS = ("jsd", "kl_pq", "kl_qp", "loglik", "bic", "bic_bin_count", "mean_moment_error",
                 "second_moment_error", "compression_ratio_vs_histogram",
                 "compression_ratio_vs_raw")


class CellMetrics(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in METRIC_FIELDS]


def header_functions(path: str = HEADER) -> list[str]:
    """Names of every function the C-ABI header declares."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vdfcg_[a-z0-9_]+)\s*\(", text)))


def ptr(a: np.ndarray, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


class ModelBuffers:
    """Owns numpy arrays backing a ``Model`` struct of capacity K."""

    def __init__(self, d: int, k: int, with_map: bool = False):
        self.d, self.k = d, k
        self.weights = np.zeros(max(k, 1))
        self.means = np.zeros(max(k, 1) * d)
        self.covs = np.zeros(max(k, 1) * d * d)
        self.scale = np.ones(d) if with_map else None
        self.offset = np.zeros(d) if with_map else None
        self.struct = Model(d, k, ptr(self.weights), ptr(self.means), ptr(self.covs),
                            ptr(self.scale) if with_map else None,
                            ptr(self.offset) if with_map else None)

    @classmethod
    def from_model(cls, m: GmmModel, capacity: int | None = None) -> "ModelBuffers":
        d = m.dimension
        k = m.size()
        has_map = not m.normalization.is_identity()
        b = cls(d, capacity or k, with_map=has_map)
        for i, c in enumerate(m.components):
            b.weights[i] = c.weight
            b.means[i * d:(i + 1) * d] = c.mean
            b.covs[i * d * d:(i + 1) * d * d] = np.asarray(c.covariance, dtype=float).reshape(-1)
        if has_map:
            b.scale[:] = m.normalization.scale
            b.offset[:] = m.normalization.offset
        b.struct.components = k
        return b

    def to_model(self) -> GmmModel:
        d = self.d
        k = self.struct.components
        comps = []
        for i in range(k):
            comps.append(GaussianComponent(
                weight=float(self.weights[i]),
                mean=self.means[i * d:(i + 1) * d].copy(),
                covariance=self.covs[i * d * d:(i + 1) * d * d].reshape(d, d).copy()))
        norm = (AffineMap(self.scale.copy(), self.offset.copy()) if self.scale is not None
                else AffineMap.identity(d))
        return GmmModel(components=comps, normalization=norm, dimension=d)


def fit_config_struct(cfg, d: int, warm: ModelBuffers | None = None) -> FitConfig:
    s = FitConfig()
    s.initial_components = int(cfg.initial_components)
    s.max_em_iterations = int(cfg.max_em_iterations)
    s.prune_threshold = float(cfg.prune_threshold)
    s.prune_check_interval = int(cfg.prune_check_interval)
    s.loglik_rel_tolerance = float(cfg.loglik_rel_tolerance)
    s.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
    if cfg.temperature is not None:
        t = np.asarray(cfg.temperature, dtype=float).reshape(-1)
        s.has_temperature = 1
        for a in range(min(len(t), 3)):
            s.temperature[a] = float(t[a])
    else:
        s.has_temperature = 0
    s.warm_start = C.pointer(warm.struct) if warm is not None else None
    s.estep_fp32 = 1 if getattr(cfg, "estep_fp32", False) else 0
    return s


def meta_struct(meta, d: int) -> tuple[ModelMeta, bytes]:
    label = meta.species_label.encode("utf-8")
    s = ModelMeta()
    s.species_label = label
    s.label_len = len(label)
    s.plane = 255 if meta.plane is None else int(meta.plane)
    s.cycle = int(meta.cycle)
    if len(meta.axis_ranges) != d:
        raise ValueError("model meta must carry one axis range per dimension")
    for a, r in enumerate(meta.axis_ranges):
        s.range_lo[a] = float(r.lo)
        s.range_hi[a] = float(r.hi)
    return s, label
