"""Marshalling between the Python mirror types and the C-ABI (include/vdfcg.h).

Every function takes ``call(name, *args) -> int`` (one C entry point, already bound to
its library) and ``errmsg() -> str``. The product module (``api.py``) binds them to
libvdfcg.so; the test-only oracle wrapper (``oracle/oracle.py``) binds them to the CPU
restatement, so parity tests push identical buffers through both. Argument meaning and
error behaviour follow the reference functions cited on each wrapper.
"""
from __future__ import annotations

import copy
import ctypes as C
from typing import Callable, Optional

import numpy as np

from . import _abi
from .types import (AxisRange, CodecError, CovarianceRepairError, EStep, FitConfig, FitResult,
                    GaussianComponent, GmmModel, Histogram2D, InvalidArgument, ModelMeta,
                    ParticleSet, Plane, PruneEvent, WeightedPoints, plane_axes)

Call = Callable[..., int]


def check(rc: int, errmsg: Callable[[], str]) -> None:
    if rc == _abi.VDFCG_OK:
        return
    msg = errmsg()
    if rc == _abi.VDFCG_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == _abi.VDFCG_REPAIR_FAILED:
        raise CovarianceRepairError(msg)
    if rc == _abi.VDFCG_CODEC_ERROR:
        raise CodecError(msg)
    raise RuntimeError(msg)


def _fortran(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _pd(a):
    return _abi.ptr(a) if a is not None else None


# --------------------------------------------------------------------------- histogram
def bin_particles(call: Call, errmsg, particles: ParticleSet, plane: Plane, n_bins: int,
                  range_x: AxisRange, range_y: AxisRange) -> Histogram2D:
    """histogram.cpp:45-76."""
    particles.validate()
    v = _fortran(particles.velocities)
    n, d = v.shape
    w = np.ascontiguousarray(particles.weights, dtype=np.float64) if particles.has_weights() else None
    counts = np.zeros((max(n_bins, 0), max(n_bins, 0)), order="F")
    oor = C.c_double(0.0)
    rc = call("bin_particles", _pd(v), n, d, _pd(w), int(plane), int(n_bins), float(range_x.lo),
              float(range_x.hi), float(range_y.lo), float(range_y.hi), _pd(counts), C.byref(oor))
    check(rc, errmsg)
    return Histogram2D(counts=counts, range_x=range_x, range_y=range_y, plane=Plane(plane),
                       n_bins=n_bins, out_of_range_count=oor.value,
                       species_label=particles.species_label)


def all_planes(call: Call, errmsg, particles: ParticleSet, n_bins: int,
               rng: AxisRange) -> list[Histogram2D]:
    """histogram.cpp:78-84 (one fused pass on the device)."""
    if particles.dimension() != 3:
        raise InvalidArgument("all_planes requires d=3 particles; use bin_particles for d=2")
    particles.validate()
    v = _fortran(particles.velocities)
    n, d = v.shape
    w = np.ascontiguousarray(particles.weights, dtype=np.float64) if particles.has_weights() else None
    counts = np.zeros(3 * n_bins * n_bins)
    oor = np.zeros(3)
    rc = call("all_planes", _pd(v), n, d, _pd(w), int(n_bins), float(rng.lo), float(rng.hi),
              _pd(counts), _pd(oor))
    check(rc, errmsg)
    out = []
    for p in range(3):
        c = counts[p * n_bins * n_bins:(p + 1) * n_bins * n_bins].reshape(n_bins, n_bins, order="F")
        out.append(Histogram2D(counts=np.asfortranarray(c), range_x=rng, range_y=rng,
                               plane=Plane(p), n_bins=n_bins, out_of_range_count=float(oor[p]),
                               species_label=particles.species_label))
    return out


def to_weighted_points(call: Call, errmsg, hist: Histogram2D,
                       drop_empty: bool = True) -> WeightedPoints:
    """histogram.cpp:86-109."""
    nb = hist.n_bins
    counts = _fortran(hist.counts)
    cap = nb * nb
    buf = np.zeros(2 * max(cap, 1))
    w = np.zeros(max(cap, 1))
    count = C.c_int64(0)
    tot = C.c_double(0.0)
    rc = call("to_weighted_points", _pd(counts), nb, float(hist.range_x.lo), float(hist.range_x.hi),
              float(hist.range_y.lo), float(hist.range_y.hi), 1 if drop_empty else 0, cap,
              _pd(buf), _pd(w), C.byref(count), C.byref(tot))
    check(rc, errmsg)
    k = count.value
    pts = np.asfortranarray(buf[:2 * k].reshape(2, k).T)
    return WeightedPoints(points=pts, weights=w[:k].copy(), total_weight=tot.value)


# --------------------------------------------------------------------------- wgmm
def normalize(call: Call, errmsg, points: WeightedPoints):
    """wgmm.cpp:78-100 -> (WeightedPoints, AffineMap)."""
    from .types import AffineMap
    x = _fortran(points.points)
    n, d = x.shape
    w = np.ascontiguousarray(points.weights, dtype=np.float64)
    if len(w) != n:
        raise InvalidArgument("weighted points: weight count does not match point count")
    out = np.zeros((n, d), order="F")
    scale = np.zeros(d)
    offset = np.zeros(d)
    rc = call("normalize", _pd(x), _pd(w), n, d, _pd(out), _pd(scale), _pd(offset))
    check(rc, errmsg)
    return (WeightedPoints(points=out, weights=w.copy(), total_weight=points.total_weight),
            AffineMap(scale, offset))


def denormalize_model(call: Call, errmsg, model: GmmModel) -> GmmModel:
    """wgmm.cpp:102-120."""
    src = _abi.ModelBuffers.from_model(model)
    dst = _abi.ModelBuffers(model.dimension, model.size())
    rc = call("denormalize_model", C.byref(src.struct), C.byref(dst.struct))
    check(rc, errmsg)
    return dst.to_model()


def _warm(cfg: FitConfig):
    return _abi.ModelBuffers.from_model(cfg.warm_start) if cfg.warm_start is not None else None


def _check_temperature_size(cfg: FitConfig, d: int) -> None:
    if cfg.temperature is not None and len(np.asarray(cfg.temperature).reshape(-1)) != d:
        raise InvalidArgument("temperature must be a positive per-axis variance")


def init_model(call: Call, errmsg, normalized_points: WeightedPoints, config: FitConfig,
               temperature, amap) -> GmmModel:
    """wgmm.cpp:136-191."""
    x = _fortran(normalized_points.points)
    n, d = x.shape
    t = np.asarray(temperature, dtype=np.float64).reshape(-1)
    if config.warm_start is None and len(t) != d:
        raise InvalidArgument("temperature must be a positive per-axis variance")
    if amap.dim() != d:
        raise InvalidArgument("normalization map dimension mismatch")
    t3 = np.zeros(3)
    t3[:min(3, len(t))] = t[:3]
    warm = _warm(config)
    cfg = _abi.fit_config_struct(config, d, warm)
    k = max(config.initial_components, warm.k if warm else 0, 1)
    out = _abi.ModelBuffers(d, k, with_map=True)
    scale = np.ascontiguousarray(amap.scale, dtype=np.float64)
    offset = np.ascontiguousarray(amap.offset, dtype=np.float64)
    rc = call("init_model", _pd(x), n, d, C.byref(cfg), _pd(t3), _pd(scale), _pd(offset),
              C.byref(out.struct))
    check(rc, errmsg)
    return out.to_model()


def e_step(call: Call, errmsg, model: GmmModel, points: WeightedPoints) -> EStep:
    """wgmm.cpp:233-255; repairs ``model`` covariances in place like the reference."""
    if model.dimension != points.dimension():
        raise InvalidArgument("model and points dimension mismatch")
    x = _fortran(points.points)
    n, d = x.shape
    w = np.ascontiguousarray(points.weights, dtype=np.float64)
    mb = _abi.ModelBuffers.from_model(model)
    m = model.size()
    resp = np.zeros(max(m * n, 1))
    ll = C.c_double(0.0)
    unrep = np.zeros(max(m, 1), dtype=np.int32)
    nun = C.c_int32(0)
    rc = call("e_step", C.byref(mb.struct), _pd(x), _pd(w), n, _pd(resp), C.byref(ll),
              _abi.ptr(unrep, C.c_int32), C.byref(nun))
    check(rc, errmsg)
    back = mb.to_model()
    for i, c in enumerate(model.components):
        c.covariance = back.components[i].covariance
    return EStep(responsibilities=resp[:m * n].reshape(m, n, order="F"), loglik=ll.value,
                 unrepairable=[int(u) for u in unrep[:nun.value]])


def m_step(call: Call, errmsg, points: WeightedPoints, responsibilities, previous: GmmModel,
           degenerate: Optional[list] = None) -> GmmModel:
    """wgmm.cpp:269-318."""
    x = _fortran(points.points)
    n, d = x.shape
    m = previous.size()
    r = np.asfortranarray(np.asarray(responsibilities, dtype=np.float64))
    if r.shape != (m, n):
        raise InvalidArgument("responsibility matrix shape mismatch")
    w = np.ascontiguousarray(points.weights, dtype=np.float64)
    prev = _abi.ModelBuffers.from_model(previous)
    out = _abi.ModelBuffers(d, m, with_map=prev.scale is not None)
    dg = np.zeros(max(m, 1), dtype=np.int32)
    ndg = C.c_int32(0)
    rc = call("m_step", _pd(x), _pd(w), n, float(points.total_weight), _pd(r),
              C.byref(prev.struct), C.byref(out.struct), _abi.ptr(dg, C.c_int32), C.byref(ndg))
    check(rc, errmsg)
    res = out.to_model()
    res.normalization = copy.deepcopy(previous.normalization)
    if degenerate is not None:
        degenerate.extend(int(i) for i in dg[:ndg.value])
    return res


def prune_one(call: Call, errmsg, model: GmmModel, threshold: float,
              iteration: int = 0) -> Optional[PruneEvent]:
    """wgmm.cpp:320-333 (mutates ``model``)."""
    mb = _abi.ModelBuffers.from_model(model)
    pruned = C.c_int32(0)
    comp = C.c_int32(-1)
    wt = C.c_double(0.0)
    rc = call("prune_one", C.byref(mb.struct), float(threshold), int(iteration), C.byref(pruned),
              C.byref(comp), C.byref(wt))
    check(rc, errmsg)
    if not pruned.value:
        return None
    back = mb.to_model()
    model.components = back.components
    return PruneEvent(iteration=iteration, component=comp.value, weight=wt.value)


def prune(call: Call, errmsg, model: GmmModel, threshold: float) -> GmmModel:
    """wgmm.cpp:335-338."""
    m = copy.deepcopy(model)
    prune_one(call, errmsg, m, threshold)
    return m


def repair_covariance(call: Call, errmsg, sigma, return_doublings: bool = False):
    """wgmm.cpp:340-362."""
    s = np.asarray(sigma, dtype=np.float64)
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        raise InvalidArgument("covariance must be square")
    d = s.shape[0]
    src = np.ascontiguousarray(s)
    out = np.zeros((d, d))
    db = C.c_int32(-1)
    rc = call("repair_covariance", _pd(src), d, _pd(out), C.byref(db))
    check(rc, errmsg)
    return (out, db.value) if return_doublings else out


def fit(call: Call, errmsg, points: WeightedPoints, config: FitConfig) -> FitResult:
    """wgmm.cpp:364-423."""
    x = _fortran(points.points)
    n, d = x.shape
    w = np.ascontiguousarray(points.weights, dtype=np.float64)
    if len(w) != n:
        raise InvalidArgument("weighted points: weight count does not match point count")
    _check_temperature_size(config, d)
    warm = _warm(config)
    cfg = _abi.fit_config_struct(config, d, warm)
    k = max(config.initial_components, warm.k if warm else 0, 1)
    t_cap = max(config.max_em_iterations, 1)
    mb = _abi.ModelBuffers(d, k)
    trace = np.zeros(t_cap)
    ev_it = np.zeros(k, dtype=np.int32)
    ev_c = np.zeros(k, dtype=np.int32)
    ev_w = np.zeros(k)
    res = _abi.FitResult()
    res.capacity_components = k
    res.capacity_trace = t_cap
    res.model = mb.struct
    res.loglik_trace = _pd(trace)
    res.event_iteration = _abi.ptr(ev_it, C.c_int32)
    res.event_component = _abi.ptr(ev_c, C.c_int32)
    res.event_weight = _pd(ev_w)
    rc = call("fit", _pd(x), _pd(w), n, d, float(points.total_weight), C.byref(cfg), C.byref(res))
    check(rc, errmsg)
    mb.struct.components = res.model.components
    model = mb.to_model()
    events = [PruneEvent(int(ev_it[e]), int(ev_c[e]), float(ev_w[e]))
              for e in range(min(res.n_events, k))]
    return FitResult(model=model, loglik_trace=[float(v) for v in trace[:res.trace_len]],
                     iterations_used=res.iterations_used, pruning_events=events,
                     converged=bool(res.converged))


# --------------------------------------------------------------------------- codec
def model_payload_bytes(components: int, dimension: int) -> int:
    """codec.cpp:86-89."""
    return components * (1 + dimension + dimension * (dimension + 1) // 2) * 8


def encode_model(call: Call, errmsg, model: GmmModel, meta: ModelMeta) -> bytes:
    """codec.cpp:103-136."""
    model.validate()
    d = model.dimension
    if len(meta.axis_ranges) != d:
        raise InvalidArgument("model meta must carry one axis range per dimension")
    label = meta.species_label.encode("utf-8")
    if len(label) > 0xFFFF:
        raise InvalidArgument("species label too long")
    ms, _keep = _abi.meta_struct(meta, d)
    mb = _abi.ModelBuffers.from_model(model)
    cap = 26 + 16 * d + len(label) + model_payload_bytes(model.size(), d) + 16
    out = np.zeros(cap, dtype=np.uint8)
    length = C.c_int64(0)
    rc = call("encode_model", C.byref(mb.struct), C.byref(ms), _abi.ptr(out, C.c_uint8), cap,
              C.byref(length))
    check(rc, errmsg)
    return out[:length.value].tobytes()
