"""Product API: the reference's hot-path entry points, computed by libvdfcg.so.

Function names, argument meaning and exceptions follow the reference
(proj/include/vdfc/histogram.hpp, wgmm.hpp, codec.hpp). Every compute call goes
through the C-ABI in include/vdfcg.h into sm_100a kernels; there is no CPU fallback —
if the library cannot be loaded or no CUDA device exists, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from functools import partial

import numpy as np

from . import _abi, _marshal, _metrics
from .types import (AxisRange, FitConfig, GmmModel, InvalidArgument, ModelMeta,  # noqa: F401
                    ParticleSet, WeightedPoints)

LIB_PATH = os.environ.get("VDFCG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libvdfcg.so")

_lib = None
_lib_lock = threading.Lock()


def _bind(lib) -> None:
    vp, i32, i64, f64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint64
    sig = {
        "vdfcg_last_error": (C.c_char_p, []),
        "vdfcg_abi_version": (C.c_int, []),
        "vdfcg_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "vdfcg_ctx_destroy": (C.c_int, [vp]),
        "vdfcg_ctx_set_stream": (C.c_int, [vp, vp]),
        "vdfcg_ctx_synchronize": (C.c_int, [vp]),
        "vdfcg_ctx_enable_timing": (C.c_int, [vp, C.c_int]),
        "vdfcg_ctx_reset_timing": (C.c_int, [vp]),
        "vdfcg_ctx_kernel_times": (C.c_int, [vp, i32, vp, vp, vp, vp]),
        "vdfcg_ctx_launch_count": (i64, [vp]),
        "vdfcg_ctx_diagnostics": (C.c_int, [vp, vp, C.c_int]),
        "vdfcg_bin_particles": (C.c_int, [vp, vp, i64, i32, vp, i32, i32, f64, f64, f64, f64, vp, vp]),
        "vdfcg_all_planes": (C.c_int, [vp, vp, i64, i32, vp, i32, f64, f64, vp, vp]),
        "vdfcg_to_weighted_points": (C.c_int, [vp, vp, i32, f64, f64, f64, f64, i32, i64, vp, vp, vp, vp]),
        "vdfcg_validate_fit_config": (C.c_int, [vp, i32]),
        "vdfcg_normalize": (C.c_int, [vp, vp, vp, i64, i32, vp, vp, vp]),
        "vdfcg_denormalize_model": (C.c_int, [vp, vp, vp]),
        "vdfcg_init_model": (C.c_int, [vp, vp, i64, i32, vp, vp, vp, vp, vp]),
        "vdfcg_e_step": (C.c_int, [vp, vp, vp, vp, i64, vp, vp, vp, vp]),
        "vdfcg_m_step": (C.c_int, [vp, vp, vp, i64, f64, vp, vp, vp, vp, vp]),
        "vdfcg_prune_one": (C.c_int, [vp, vp, f64, i32, vp, vp, vp]),
        "vdfcg_repair_covariance": (C.c_int, [vp, vp, i32, vp, vp]),
        "vdfcg_fit": (C.c_int, [vp, vp, vp, i64, i32, f64, vp, vp]),
        "vdfcg_model_payload_bytes": (i64, [i32, i32]),
        "vdfcg_model_header_bytes": (i64, [i32, i32]),
        "vdfcg_encode_model": (C.c_int, [vp, vp, vp, vp, i64, vp]),
        "vdfcg_bin_cells": (C.c_int, [vp, vp, vp]),
        "vdfcg_fit_cells": (C.c_int, [vp, vp, vp, vp, vp]),
        "vdfcg_pack_cells": (C.c_int, [vp, i32, i32, vp, vp, vp, i64, vp]),
        "vdfcg_compress_cells": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, i64, vp]),
        "vdfcg_fit_cells_warm": (C.c_int, [vp, vp, vp, vp, vp, vp]),
        "vdfcg_compress_cells_warm": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, i64, vp]),
        "vdfcg_bin_cells_indexed": (C.c_int, [vp, vp, vp, vp]),
        "vdfcg_compress_cells_indexed": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, i64, vp]),
        "vdfcg_compress_cells_indexed_warm": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, vp]),
        "vdfcg_partition_cells": (C.c_int, [vp, i32, i32, vp]),
        "vdfcg_multi_create": (C.c_int, [vp, i32, C.POINTER(vp)]),
        "vdfcg_multi_destroy": (C.c_int, [vp]),
        "vdfcg_multi_device_count": (i32, [vp]),
        "vdfcg_multi_context": (C.c_int, [vp, i32, C.POINTER(vp)]),
        "vdfcg_multi_compress_cells": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, i64, vp, vp]),
        "vdfcg_synth_cells": (C.c_int, [vp, i32, i32, vp, i64, u64, i32, vp, vp, vp]),
        "vdfcg_probe_peaks": (C.c_int, [vp, vp, vp]),
        "vdfcg_generate": (C.c_int, [vp, i32, i32, vp, vp, vp, i64, u64, vp, vp]),
        "vdfcg_metrics_cells": (C.c_int, [vp, vp, vp, vp, vp]),
        "vdfcg_evaluate_pdf": (C.c_int, [vp, vp, i32, f64, f64, f64, f64, vp]),
        "vdfcg_weighted_loglik": (C.c_int, [vp, vp, vp, vp, i64, vp]),
        "vdfcg_pdf_divergences": (C.c_int, [vp, vp, vp, i64, f64, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args


def lib():
    """The loaded CUDA library; raises (loudly) when it is missing."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"libvdfcg.so not built ({LIB_PATH}); run "
                        "`python -m paper_2504_14897_b200.build` (there is no CPU fallback)")
                lb = C.CDLL(LIB_PATH)
                _bind(lb)
                _lib = lb
    return _lib


def last_error() -> str:
    return lib().vdfcg_last_error().decode()


class Context:
    """One CUDA stream + workspace on one device (vdfcg_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _marshal.check(lib().vdfcg_ctx_create(device, C.byref(h)), last_error)
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            lib().vdfcg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None) -> None:
        _marshal.check(lib().vdfcg_ctx_set_stream(self.handle, stream_ptr), last_error)

    def synchronize(self) -> None:
        _marshal.check(lib().vdfcg_ctx_synchronize(self.handle), last_error)

    def enable_timing(self, on: bool = True) -> None:
        _marshal.check(lib().vdfcg_ctx_enable_timing(self.handle, 1 if on else 0), last_error)

    def reset_timing(self) -> None:
        _marshal.check(lib().vdfcg_ctx_reset_timing(self.handle), last_error)

    def kernel_times(self) -> dict:
        """{kernel family: (total ms, launches)} from CUDA events on the context stream."""
        n = 64
        names = C.create_string_buffer(32 * n)
        ms = np.zeros(n)
        cnt = np.zeros(n, dtype=np.int64)
        k = C.c_int32(0)
        _marshal.check(lib().vdfcg_ctx_kernel_times(self.handle, n, names, ms.ctypes.data,
                                                    cnt.ctypes.data, C.byref(k)), last_error)
        out = {}
        for i in range(k.value):
            nm = names.raw[32 * i:32 * (i + 1)].split(b"\0", 1)[0].decode()
            out[nm] = (float(ms[i]), int(cnt[i]))
        return out

    def launch_count(self) -> int:
        return int(lib().vdfcg_ctx_launch_count(self.handle))

    def exact_passes(self, reset: bool = False) -> int:
        """(fit, iteration) pairs that ran the exact second M-step pass."""
        v = C.c_int64(0)
        _marshal.check(lib().vdfcg_ctx_diagnostics(self.handle, C.byref(v), 1 if reset else 0),
                       last_error)
        return int(v.value)


_tls = threading.local()


def context(device: int | None = None) -> Context:
    """Per-thread, per-device default context (the reference API is reentrant)."""
    if device is None:
        device = int(os.environ.get("VDFCG_DEVICE", getattr(_tls, "device", 0)))
    cache = getattr(_tls, "ctxs", None)
    if cache is None:
        cache = _tls.ctxs = {}
    if device not in cache:
        cache[device] = Context(device)
    return cache[device]


def _call(name, *args):
    return getattr(lib(), "vdfcg_" + name)(context().handle, *args)


def _err():
    return last_error()


# ---------------------------------------------------------------------------- API
bin_particles = partial(_marshal.bin_particles, _call, _err)
bin_particles.__doc__ = "histogram.hpp:48-49 bin_particles(particles, plane, n_bins, range_x, range_y)"
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

# fit quality (metrics.hpp, wgmm.hpp:128-136)
evaluate_pdf = partial(_metrics.evaluate_pdf, _call, _err)
weighted_loglik = partial(_metrics.weighted_loglik, _call, _err)
kl_divergence = partial(_metrics.kl_divergence, _call, _err)
jsd = partial(_metrics.jsd, _call, _err)
assemble_metrics = partial(_metrics.assemble_metrics, _call, _err)
from ._metrics import (MetricsReport, PdfGrid, bic, bic_parameter_count,  # noqa: E402,F401
                       compression_ratio, mixture_moments, moment_errors, to_pdf,
                       weighted_data_moments)


def default_axis_range(particles: ParticleSet, axis: int) -> AxisRange:
    """histogram.cpp:27-30: +/- 5 nominal thermal speeds."""
    vth = float(np.sqrt(particles.nominal_temperature[axis]))
    return AxisRange(-5.0 * vth, 5.0 * vth)


def probe_peaks() -> tuple[float, float]:
    """Measured (FP64, FP32) FMA TFLOP/s of the current device (roofline denominators)."""
    f64, f32 = C.c_double(0.0), C.c_double(0.0)
    _marshal.check(lib().vdfcg_probe_peaks(context().handle, C.byref(f64), C.byref(f32)), last_error)
    return f64.value, f32.value


def generate(fractions, means, covs, n: int, seed: int, label: str = "synthetic",
             out=None) -> ParticleSet:
    """synthdata.cpp:54-86 generate(ScenarioSpec) on the device: the reference's mixture
    generator on its own mt19937_64(seed) stream. ``out`` may be a CUDA tensor of n*d
    float64 (column-major velocities are written there and the returned ParticleSet holds
    a host copy only when ``out`` is None)."""
    means = np.asarray(means, dtype=np.float64)
    covs = np.asarray(covs, dtype=np.float64)
    m, d = means.shape
    fr = np.ascontiguousarray(fractions, dtype=np.float64)
    if fr.shape != (m,) or covs.shape != (m, d, d):
        raise InvalidArgument("generate: fractions/means/covariances shape mismatch")
    mu = np.ascontiguousarray(means.reshape(-1))
    cv = np.ascontiguousarray(covs.reshape(-1))
    temp = np.zeros(d)
    if out is None:
        vel = np.zeros((n, d), order="F")
        ptr = vel.ctypes.data
        ctx = context()
    else:
        import torch
        from .cells import _ctx
        # column-major n x d: a flat tensor of n*d values, or an (n, d) view with stride (1, n)
        ok = (isinstance(out, torch.Tensor) and out.dtype == torch.float64 and out.is_cuda
              and ((out.dim() == 1 and out.numel() == n * d and out.stride(0) == 1)
                   or (out.dim() == 2 and tuple(out.shape) == (n, d) and out.stride() == (1, n))))
        if not ok:
            raise InvalidArgument("generate: out must be a CUDA float64 tensor of n*d values "
                                  "(flat, or an (n, d) column-major view with stride (1, n))")
        ctx = _ctx(out)  # out's device, ordered on its current torch stream
        vel, ptr = out.view(d, n).t() if out.dim() == 1 else out, out.data_ptr()
    _marshal.check(lib().vdfcg_generate(ctx.handle, d, m, fr.ctypes.data, mu.ctypes.data,
                                        cv.ctypes.data, n, seed & 0xFFFFFFFFFFFFFFFF, ptr,
                                        temp.ctypes.data), last_error)
    return ParticleSet(velocities=vel, species_label=label, nominal_temperature=temp)


def validate_fit_config(config: FitConfig, d: int) -> None:
    """FitConfig::validate (wgmm.cpp:65-76); host-only."""
    cfg = _abi.fit_config_struct(config, d)
    _marshal.check(lib().vdfcg_validate_fit_config(C.byref(cfg), d), last_error)


from .codec import (DecodedModel, decode_histogram, decode_model,  # noqa: E402,F401
                    encode_histogram, histogram_sidecar, model_from_json, model_to_json)
from .stream import RecordStream, read_index, read_record  # noqa: E402,F401
from .cells import (CellBatch, CellMetrics, MultiDevice, ParticleBatch, bin_cells,  # noqa: E402,F401
                    bin_cells_indexed, cell_metrics, compress_cells, compress_cells_indexed,
                    fit_cells, pack_cells, partition_cells, synth_cells)
