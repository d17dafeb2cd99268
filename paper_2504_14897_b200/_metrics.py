"""Fit-quality mirror of the reference (metrics.hpp, pdf_grid.hpp, wgmm.hpp:128-136,
histogram.hpp:57-63) — SURVEY.md 8(f) row 1.

Like ``_marshal``, every function that computes over a grid or a point set takes
``call(name, *args)`` and ``errmsg()``: ``api`` binds them to libvdfcg.so (sm_100a
kernels), ``oracle/oracle.py`` to the CPU restatement. Scalar formulas the reference
evaluates on a handful of numbers (bic, compression_ratio, the mixture moments of a
model) are plain host arithmetic here too.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._marshal import Call, check
from .types import GmmModel, GridSpec, Histogram2D, InvalidArgument, WeightedPoints


@dataclass
class PdfGrid:
    """pdf_grid.hpp:9-23: density values on a GridSpec; values[i, j] = bin (i, j)."""
    spec: GridSpec
    values: np.ndarray

    def bin_area(self) -> float:
        return self.spec.dx() * self.spec.dy()

    def mass(self, i: int, j: int) -> float:
        return float(self.values[i, j]) * self.bin_area()

    def aligned_with(self, other: "PdfGrid") -> bool:
        a, b = self.spec, other.spec
        return (a.n_bins == b.n_bins and a.x.lo == b.x.lo and a.x.hi == b.x.hi and
                a.y.lo == b.y.lo and a.y.hi == b.y.hi)

    @staticmethod
    def normalized(spec: GridSpec, raw) -> "PdfGrid":
        """pdf_grid.cpp:5-19."""
        if not (spec.n_bins >= 1 and spec.x.valid() and spec.y.valid()):
            raise InvalidArgument("invalid grid spec")
        raw = np.array(raw, dtype=np.float64)
        if raw.shape != (spec.n_bins, spec.n_bins):
            raise InvalidArgument("pdf grid shape does not match spec")
        if np.any(raw < 0.0):
            raise InvalidArgument("pdf grid values must be non-negative")
        total = float(raw.sum()) * (spec.dx() * spec.dy())
        if not (total > 0.0) or not math.isfinite(total):
            raise InvalidArgument("degenerate pdf grid: total mass is zero or non-finite")
        return PdfGrid(spec, raw / total)


def to_pdf(hist: Histogram2D) -> PdfGrid:
    """histogram.cpp:111-115."""
    if hist.degenerate():
        raise InvalidArgument("degenerate histogram: no in-range weight")
    return PdfGrid.normalized(hist.grid(), hist.counts)


def evaluate_pdf(call: Call, errmsg, model: GmmModel, grid: GridSpec) -> np.ndarray:
    """wgmm.cpp:425-453: the mixture density at every bin centre (n x n)."""
    mb = _abi.ModelBuffers.from_model(model)
    out = np.zeros((max(grid.n_bins, 1), max(grid.n_bins, 1)), order="F")
    check(call("evaluate_pdf", C.byref(mb.struct), int(grid.n_bins), float(grid.x.lo),
               float(grid.x.hi), float(grid.y.lo), float(grid.y.hi), out.ctypes.data), errmsg)
    return out


def weighted_loglik(call: Call, errmsg, model: GmmModel, points: WeightedPoints) -> float:
    """wgmm.cpp:257-267 (covariances repaired on a copy; the caller's model is untouched)."""
    mb = _abi.ModelBuffers.from_model(model)
    x = np.asfortranarray(points.points, dtype=np.float64)
    w = np.ascontiguousarray(points.weights, dtype=np.float64)
    out = C.c_double()
    check(call("weighted_loglik", C.byref(mb.struct), x.ctypes.data, w.ctypes.data, len(w),
               C.byref(out)), errmsg)
    return out.value


def _divergences(call: Call, errmsg, p: PdfGrid, q: PdfGrid, what: str):
    if not p.aligned_with(q):
        raise InvalidArgument(f"{what}: grids are not aligned")
    a = np.ascontiguousarray(p.values, dtype=np.float64).ravel(order="F")
    b = np.ascontiguousarray(q.values, dtype=np.float64).ravel(order="F")
    j, kpq, kqp = C.c_double(), C.c_double(), C.c_double()
    check(call("pdf_divergences", a.ctypes.data, b.ctypes.data, a.size, p.bin_area(),
               C.byref(j) if what == "jsd" else None, C.byref(kpq), C.byref(kqp)), errmsg)
    return j.value, kpq.value, kqp.value


def kl_divergence(call: Call, errmsg, p: PdfGrid, q: PdfGrid) -> float:
    """metrics.cpp:12-26: sum p_n log(p_n / q_n); +inf where Q vanishes under P."""
    return _divergences(call, errmsg, p, q, "kl_divergence")[1]


def jsd(call: Call, errmsg, p: PdfGrid, q: PdfGrid) -> float:
    """metrics.cpp:28-46."""
    return _divergences(call, errmsg, p, q, "jsd")[0]


def bic_parameter_count(components: int, dimension: int) -> int:
    """metrics.cpp:48-50."""
    return components * (1 + dimension * (dimension + 3) // 2)


def bic(loglik: float, model: GmmModel, n_observed: float) -> float:
    """metrics.cpp:52-56."""
    if not (n_observed > 0.0):
        raise InvalidArgument("bic: n_observed must be > 0")
    return -2.0 * loglik + bic_parameter_count(model.size(), model.dimension) * math.log(n_observed)


def mixture_moments(model: GmmModel):
    """wgmm.cpp:455-471: (mean, second moment) of the mixture in data space."""
    d = model.dimension
    mean = np.zeros(d)
    m2 = np.zeros((d, d))
    for c in model.components:
        mu = np.asarray(c.mean, float)
        mean += c.weight * mu
        m2 += c.weight * (np.asarray(c.covariance, float) + np.outer(mu, mu))
    if model.normalization.is_identity():
        return mean, m2
    s = np.diag(model.normalization.scale)
    b = np.asarray(model.normalization.offset, float)
    mean_x = model.normalization.inverse(mean)
    m2_x = s @ m2 @ s + np.outer(s @ mean, b) + np.outer(b, s @ mean) + np.outer(b, b)
    return mean_x, m2_x


def weighted_data_moments(points: WeightedPoints):
    """wgmm.cpp:473-480."""
    total = float(np.sum(points.weights))
    if not (total > 0.0):
        raise InvalidArgument("weighted moments: zero total weight")
    x = np.asarray(points.points, float)
    w = np.asarray(points.weights, float)
    return x.T @ w / total, (x.T * w) @ x / total


def moment_errors(model: GmmModel, points: WeightedPoints):
    """metrics.cpp:58-65."""
    mm, m2 = mixture_moments(model)
    dm, d2 = weighted_data_moments(points)
    return (float(np.linalg.norm(mm - dm) / math.sqrt(np.trace(d2))),
            float(np.linalg.norm(m2 - d2) / np.linalg.norm(d2)))


def compression_ratio(original_bytes: int, compressed_bytes: int) -> float:
    """metrics.cpp:67-72."""
    if original_bytes == 0:
        raise InvalidArgument("compression_ratio: zero original size")
    if compressed_bytes == 0:
        raise InvalidArgument("compression_ratio: zero compressed size")
    return float(original_bytes) / float(compressed_bytes)


@dataclass
class MetricsReport:
    """metrics.hpp:39-54 (+ the JSON / CSV forms of metrics.cpp:74-119)."""
    jsd: float = 0.0
    kl_pq: float = 0.0
    kl_qp: float = 0.0
    bic: float = 0.0
    bic_bin_count: float = 0.0
    mean_moment_error: float = 0.0
    second_moment_error: float = 0.0
    compression_ratio_vs_histogram: float = 0.0
    compression_ratio_vs_raw: float = 0.0

    FIELDS = ("jsd", "kl_pq", "kl_qp", "bic", "bic_bin_count", "mean_moment_error",
              "second_moment_error", "compression_ratio_vs_histogram", "compression_ratio_vs_raw")

    def to_json(self) -> dict:
        """JSON has no infinities: divergent values serialise as null."""
        return {f: (None if math.isinf(getattr(self, f)) else getattr(self, f)) for f in self.FIELDS}

    @staticmethod
    def from_json(j: dict) -> "MetricsReport":
        return MetricsReport(**{f: (math.inf if j[f] is None else float(j[f])) for f in MetricsReport.FIELDS})

    @staticmethod
    def csv_header() -> str:
        return ",".join(MetricsReport.FIELDS)

    def csv_row(self) -> str:
        def g(v):  # printf %.17g
            if math.isinf(v):
                return "inf" if v > 0 else "-inf"
            if math.isnan(v):
                return "nan"
            return "%.17g" % v
        return ",".join(g(getattr(self, f)) for f in self.FIELDS)


def assemble_metrics(call: Call, errmsg, model: GmmModel, hist: Histogram2D,
                     points: WeightedPoints, raw_particle_count: int,
                     raw_dimension: int) -> MetricsReport:
    """pipeline.cpp:106-128."""
    from ._marshal import model_payload_bytes
    hist_pdf = to_pdf(hist)
    model_pdf = PdfGrid.normalized(hist.grid(), evaluate_pdf(call, errmsg, model, hist.grid()))
    r = MetricsReport()
    r.jsd = jsd(call, errmsg, hist_pdf, model_pdf)
    r.kl_pq = kl_divergence(call, errmsg, hist_pdf, model_pdf)
    r.kl_qp = kl_divergence(call, errmsg, model_pdf, hist_pdf)
    ll = weighted_loglik(call, errmsg, model, points)
    r.bic = bic(ll, model, points.total_weight)
    r.bic_bin_count = bic(ll, model, float(hist.n_bins) * hist.n_bins)
    r.mean_moment_error, r.second_moment_error = moment_errors(model, points)
    mb = model_payload_bytes(model.size(), model.dimension)
    r.compression_ratio_vs_histogram = compression_ratio(hist.n_bins * hist.n_bins * 8, mb)
    r.compression_ratio_vs_raw = compression_ratio(raw_particle_count * raw_dimension * 8, mb)
    return r
