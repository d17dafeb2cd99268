"""CPU oracle (TEST INFRASTRUCTURE ONLY).

ctypes wrapper around oracle/liboracle.so, the plain-C++ restatement of the reference
hot path (see vdfc_oracle.h for what pins it). Exposes the same Python-level functions
as the product package (``paper_2504_14897_b200``) so tests feed both the same inputs.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
from functools import partial

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))

from paper_2504_14897_b200 import _abi, _marshal, _metrics  # noqa: E402
from paper_2504_14897_b200.types import (AxisRange, FitConfig, ParticleSet,  # noqa: E402,F401
                                         WeightedPoints)

LIB_PATH = os.path.join(_HERE, "liboracle.so")
REFEM_PATH = os.path.join(_HERE, "_ref", "librefem.so")


def build(force: bool = False) -> None:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(os.path.join(_HERE, f)) for f in ("vdfc_oracle.cpp", "vdfc_oracle.h")):
        subprocess.run(["make", "-s", "-C", _HERE, os.path.join(_HERE, "liboracle.so")], check=True)


def _load():
    build()
    return C.CDLL(LIB_PATH)


_lib = _load()
_lib.oracle_last_error.restype = C.c_char_p
_lib.oracle_model_payload_bytes.restype = C.c_int64
for _n in ("oracle_bin_particles", "oracle_all_planes", "oracle_to_weighted_points"):
    getattr(_lib, _n).restype = C.c_int
_lib.oracle_bin_particles.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32,
                                      C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_void_p, C.c_void_p]
_lib.oracle_all_planes.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32,
                                   C.c_double, C.c_double, C.c_void_p, C.c_void_p]
_lib.oracle_to_weighted_points.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_double,
                                           C.c_double, C.c_double, C.c_int32, C.c_int64,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
_lib.oracle_normalize.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                  C.c_void_p, C.c_void_p]
_lib.oracle_init_model.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]
_lib.oracle_e_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_void_p]
_lib.oracle_m_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
_lib.oracle_prune_one.argtypes = [C.c_void_p, C.c_double, C.c_int32, C.c_void_p, C.c_void_p,
                                  C.c_void_p]
_lib.oracle_repair_covariance.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
_lib.oracle_fit.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_void_p,
                            C.c_void_p]
_lib.oracle_encode_model.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
_lib.oracle_generate.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p]
_lib.oracle_uniforms.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
_lib.oracle_validate_fit_config.argtypes = [C.c_void_p, C.c_int32]
_lib.oracle_mixture_moments.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
_lib.oracle_weighted_data_moments.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                              C.c_void_p, C.c_void_p]
_lib.oracle_bin_cells.argtypes = [C.c_void_p, C.c_void_p]
_lib.oracle_bin_cells_indexed.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
_lib.oracle_compress_cells.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_void_p, C.c_void_p]
_lib.oracle_evaluate_pdf.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_void_p]
_lib.oracle_weighted_loglik.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
_lib.oracle_pdf_divergences.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
_lib.oracle_cell_metrics.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_void_p]
_lib.oracle_pack_cells.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int64, C.c_void_p]


def _call(name, *args):
    return getattr(_lib, "oracle_" + name)(*args)


def _err():
    return _lib.oracle_last_error().decode()


bin_particles = partial(_marshal.bin_particles, _call, _err)
all_planes = partial(_marshal.all_planes, _call, _err)
to_weighted_points = partial(_marshal.to_weighted_points, _call, _err)
normalize = partial(_marshal.normalize, _call, _err)
denormalize_model = partial(_marshal.denormalize_model, _call, _err)
init_model = partial(_marshal.init_model, _call, _err)
e_step = partial(_marshal.e_step, _call, _err)
m_step = partial(_marshal.m_step, _call, _err)
prune_one = partial(_marshal.prune_one, _call, _err)
prune = partial(_marshal.prune, _call, _err)
repair_covariance = partial(_marshal.repair_covariance, _call, _err)
fit = partial(_marshal.fit, _call, _err)
encode_model = partial(_marshal.encode_model, _call, _err)
model_payload_bytes = _marshal.model_payload_bytes


def validate_fit_config(config: FitConfig, d: int) -> None:
    cfg = _abi.fit_config_struct(config, d)
    _marshal.check(_lib.oracle_validate_fit_config(C.byref(cfg), d), _err)


def uniforms(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    _lib.oracle_uniforms(seed & 0xFFFFFFFFFFFFFFFF, n, out.ctypes.data)
    return out


def mixture_moments(model):
    mb = _abi.ModelBuffers.from_model(model)
    d = model.dimension
    mean, m2 = np.zeros(d), np.zeros(d * d)
    _marshal.check(_lib.oracle_mixture_moments(C.byref(mb.struct), mean.ctypes.data,
                                               m2.ctypes.data), _err)
    return mean, m2.reshape(d, d)


def weighted_data_moments(points: WeightedPoints):
    x = np.asfortranarray(points.points, dtype=np.float64)
    n, d = x.shape
    w = np.ascontiguousarray(points.weights, dtype=np.float64)
    mean, m2 = np.zeros(d), np.zeros(d * d)
    _marshal.check(_lib.oracle_weighted_data_moments(x.ctypes.data, w.ctypes.data, n, d,
                                                     mean.ctypes.data, m2.ctypes.data), _err)
    return mean, m2.reshape(d, d)


# ----------------------------------------------------------------- synthetic data
PRESETS = {  # docs/presets.md / synthdata.cpp:109-134: (fraction, mean, variance)
    "maxwellian": [(1.0, (0, 0, 0), (1, 1, 1))],
    "drifting-beam": [(0.8, (0, 0, 0), (1, 1, 1)), (0.2, (3, 0, 0), (0.25, 0.25, 0.25))],
    "counter-streaming": [(0.5, (-3, 0, 0), (1, 1, 1)), (0.5, (3, 0, 0), (1, 1, 1))],
    "bump-on-tail": [(0.9, (0, 0, 0), (1, 1, 1)), (0.1, (4, 0, 0), (0.25, 0.25, 0.25))],
    "hot-core-cold-halo": [(0.5, (0, 0, 0), (2.25, 2.25, 2.25)),
                           (0.5, (0, 0, 0), (0.25, 0.25, 0.25))],
}


def generate(fractions, means, covs, n: int, seed: int, label: str = "synthetic") -> ParticleSet:
    """synthdata.cpp:54-86 restated (mt19937_64, Box-Muller, Cholesky)."""
    means = np.asarray(means, dtype=np.float64)
    covs = np.asarray(covs, dtype=np.float64)
    m, d = means.shape
    fr = np.ascontiguousarray(fractions, dtype=np.float64)
    mu = np.ascontiguousarray(means.reshape(-1))
    cv = np.ascontiguousarray(covs.reshape(-1))
    vel = np.zeros((n, d), order="F")
    temp = np.zeros(d)
    _marshal.check(_lib.oracle_generate(d, m, fr.ctypes.data, mu.ctypes.data, cv.ctypes.data, n,
                                        seed & 0xFFFFFFFFFFFFFFFF, vel.ctypes.data,
                                        temp.ctypes.data), _err)
    return ParticleSet(velocities=vel, species_label=label, nominal_temperature=temp)


def preset(name: str, n: int, seed: int) -> ParticleSet:
    comps = PRESETS[name]
    fr = [c[0] for c in comps]
    mu = [c[1] for c in comps]
    cv = [np.diag(c[2]).astype(float) for c in comps]
    return generate(fr, mu, cv, n, seed, label=name)


def gaussian_2d(n: int, seed: int, mean=(0.0, 0.0), cov=((1.0, 0.0), (0.0, 1.0))) -> ParticleSet:
    return generate([1.0], [mean], [cov], n, seed)


# ----------------------------------------------------------------- cells
class CellsHost:
    """Host arrays of a cell batch + the vdfcg_cells struct that views them."""

    def __init__(self, velocity: np.ndarray, cell_offsets: np.ndarray, n_bins: int, lo, hi,
                 weights: np.ndarray | None = None):
        self.velocity = np.asfortranarray(velocity, dtype=np.float64)  # N x d
        self.offsets = np.ascontiguousarray(cell_offsets, dtype=np.int64)
        self.weights = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        n, d = self.velocity.shape
        self.n, self.d, self.n_cells = n, d, len(self.offsets) - 1
        s = _abi.Cells()
        s.dimension = d
        s.n_particles = n
        base = self.velocity.ctypes.data
        for a in range(d):
            s.velocity[a] = base + a * n * 8
        s.weights = self.weights.ctypes.data if self.weights is not None else None
        s.n_cells = self.n_cells
        s.cell_offsets = self.offsets.ctypes.data
        s.n_bins = n_bins
        for a in range(d):
            s.lo[a] = float(lo[a])
            s.hi[a] = float(hi[a])
        self.struct = s


class CellBinsHost:
    def __init__(self, n: int, n_cells: int):
        self.nnz = np.zeros(n_cells, dtype=np.int32)
        self.keys = np.zeros(max(n, 1), dtype=np.uint32)
        self.counts = np.zeros(max(n, 1))
        self.out_of_range = np.zeros(n_cells)
        self.in_range = np.zeros(n_cells)
        self.struct = _abi.CellBins(self.nnz.ctypes.data, self.keys.ctypes.data,
                                    self.counts.ctypes.data, self.out_of_range.ctypes.data,
                                    self.in_range.ctypes.data)


class CellResultsHost:
    def __init__(self, n_cells: int, d: int, k: int, trace: int = 0):
        self.k, self.d, self.trace_cap = k, d, trace
        self.status = np.zeros(n_cells, dtype=np.int32)
        self.components = np.zeros(n_cells, dtype=np.int32)
        self.iterations = np.zeros(n_cells, dtype=np.int32)
        self.converged = np.zeros(n_cells, dtype=np.int32)
        self.weights = np.zeros(n_cells * k)
        self.means = np.zeros(n_cells * k * d)
        self.covariances = np.zeros(n_cells * k * d * d)
        self.final_loglik = np.zeros(n_cells)
        self.loglik_trace = np.zeros(max(n_cells * trace, 1))
        self.n_events = np.zeros(n_cells, dtype=np.int32)
        self.event_iteration = np.zeros(n_cells * k, dtype=np.int32)
        self.event_component = np.zeros(n_cells * k, dtype=np.int32)
        self.event_weight = np.zeros(n_cells * k)
        s = _abi.CellResults()
        s.capacity_components = k
        s.capacity_trace = trace
        for f in ("status", "components", "iterations", "converged", "weights", "means",
                  "covariances", "final_loglik", "n_events", "event_iteration",
                  "event_component", "event_weight"):
            setattr(s, f, getattr(self, f).ctypes.data)
        s.loglik_trace = self.loglik_trace.ctypes.data if trace > 0 else None
        self.struct = s


def bin_cells(cells: CellsHost) -> CellBinsHost:
    out = CellBinsHost(cells.n, cells.n_cells)
    _marshal.check(_lib.oracle_bin_cells(C.byref(cells.struct), C.byref(out.struct)), _err)
    return out


class ParticlesHost:
    """Host arrays of an unsorted particle set with a per-particle cell id (vdfcg_particles)."""

    def __init__(self, velocity: np.ndarray, cell: np.ndarray, n_cells: int, n_bins: int, lo, hi,
                 weights: np.ndarray | None = None):
        self.velocity = np.asfortranarray(velocity, dtype=np.float64)  # N x d
        self.cell = np.ascontiguousarray(cell, dtype=np.int32)
        self.weights = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        n, d = self.velocity.shape
        self.n, self.d, self.n_cells = n, d, int(n_cells)
        s = _abi.Particles()
        s.dimension = d
        s.n_particles = n
        base = self.velocity.ctypes.data
        for a in range(d):
            s.velocity[a] = base + a * n * 8
        s.weights = self.weights.ctypes.data if self.weights is not None else None
        s.cell = self.cell.ctypes.data
        s.n_cells = self.n_cells
        s.n_bins = n_bins
        for a in range(d):
            s.lo[a] = float(lo[a])
            s.hi[a] = float(hi[a])
        self.struct = s


def bin_cells_indexed(particles: ParticlesHost) -> tuple[np.ndarray, CellBinsHost]:
    """Stable group-by-cell + per-cell binning; returns (cell_offsets, bins)."""
    out = CellBinsHost(particles.n, particles.n_cells)
    offsets = np.zeros(particles.n_cells + 1, dtype=np.int64)
    _marshal.check(_lib.oracle_bin_cells_indexed(C.byref(particles.struct), offsets.ctypes.data,
                                                 C.byref(out.struct)), _err)
    return offsets, out


def compress_cells(cells: CellsHost, config: FitConfig, cell_begin: int = 0,
                   cell_end: int | None = None, threads: int = 0, trace: int = 0):
    d = cells.d
    k = max(config.initial_components, 1)
    cfg = _abi.fit_config_struct(config, d)
    bins = CellBinsHost(cells.n, cells.n_cells)
    res = CellResultsHost(cells.n_cells, d, k, trace)
    end = cells.n_cells if cell_end is None else cell_end
    _marshal.check(_lib.oracle_compress_cells(C.byref(cells.struct), C.byref(cfg), cell_begin, end,
                                              threads, C.byref(bins.struct), C.byref(res.struct)),
                   _err)
    return bins, res


def pack_cells(res: CellResultsHost, n_cells: int, meta) -> tuple[bytes, np.ndarray]:
    ms, _keep = _abi.meta_struct(meta, res.d)
    cap = int(n_cells * (26 + 16 * res.d + ms.label_len + res.k * (1 + res.d + res.d * (res.d + 1) // 2) * 8))
    buf = np.zeros(max(cap, 1), dtype=np.uint8)
    offs = np.zeros(n_cells + 1, dtype=np.int64)
    _marshal.check(_lib.oracle_pack_cells(n_cells, res.d, C.byref(res.struct), C.byref(ms),
                                          buf.ctypes.data, cap, offs.ctypes.data), _err)
    return buf[:offs[-1]].tobytes(), offs


# ----------------------------------------------------------------- fit quality
evaluate_pdf = partial(_metrics.evaluate_pdf, _call, _err)
weighted_loglik = partial(_metrics.weighted_loglik, _call, _err)
kl_divergence = partial(_metrics.kl_divergence, _call, _err)
jsd = partial(_metrics.jsd, _call, _err)
assemble_metrics = partial(_metrics.assemble_metrics, _call, _err)
from paper_2504_14897_b200._metrics import (MetricsReport, PdfGrid, bic,  # noqa: E402,F401
                                            bic_parameter_count, compression_ratio,
                                            moment_errors, to_pdf)


class CellMetricsHost:
    def __init__(self, n_cells: int):
        for f in _abi.METRIC_FIELDS:
            setattr(self, f, np.zeros(n_cells))
        self.struct = _abi.CellMetrics(*[getattr(self, f).ctypes.data for f in _abi.METRIC_FIELDS])


def cell_metrics(cells: CellsHost, bins: CellBinsHost, res: CellResultsHost, cell_begin: int = 0,
                 cell_end: int | None = None, threads: int = 0) -> CellMetricsHost:
    """pipeline.cpp:106-128 assemble_metrics for every cell."""
    out = CellMetricsHost(cells.n_cells)
    end = cells.n_cells if cell_end is None else cell_end
    _marshal.check(_lib.oracle_cell_metrics(C.byref(cells.struct), C.byref(bins.struct),
                                            C.byref(res.struct), cell_begin, end, threads,
                                            C.byref(out.struct)), _err)
    return out


# ----------------------------------------------------------------- reference refem
def refem_available() -> bool:
    return os.path.exists(REFEM_PATH)


def refem_fit(xs, ys, m=4, max_iterations=100, prune_threshold=0.005, prune_interval=10,
              tolerance=1e-6, seed=0, temperature=(1.0, 1.0)):
    """proj/tests/support/reference_em.cpp:26-157, compiled from /root/reference."""
    lib = C.CDLL(REFEM_PATH)
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    ys = np.ascontiguousarray(ys, dtype=np.float64)
    cap_t = max(max_iterations, 1)
    alpha, means, covs = np.zeros(m), np.zeros(2 * m), np.zeros(4 * m)
    trace = np.zeros(cap_t)
    nc, tl, its, conv = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    f = lib.refem_fit_c
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                  C.c_double, C.c_uint64, C.c_double, C.c_double, C.c_int32, C.c_int32,
                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                  C.c_void_p, C.c_void_p]
    rc = f(xs.ctypes.data, ys.ctypes.data, len(xs), m, max_iterations, prune_threshold,
           prune_interval, tolerance, seed, temperature[0], temperature[1], m, cap_t,
           alpha.ctypes.data, means.ctypes.data, covs.ctypes.data, trace.ctypes.data,
           C.byref(nc), C.byref(tl), C.byref(its), C.byref(conv))
    if rc != 0:
        raise RuntimeError("refem failed")
    k = nc.value
    return dict(alpha=alpha[:k], means=means[:2 * k].reshape(k, 2),
                covs=covs[:4 * k].reshape(k, 2, 2), trace=trace[:tl.value],
                iterations=its.value, converged=bool(conv.value))
