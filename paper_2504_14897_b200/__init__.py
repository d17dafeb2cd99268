"""B200-native histogram -> weighted-GMM compression path (arXiv 2504.14897).

Drop-in for the reference library's hot-path entry points (proj/include/vdfc/
histogram.hpp, wgmm.hpp, codec.hpp). All compute runs in sm_100a CUDA kernels inside
libvdfcg.so behind the C-ABI in include/vdfcg.h; this package is the host-side mirror
of the reference interface. There is no CPU fallback: the compute entry points raise
if the CUDA library cannot be loaded or no device is present.
"""
from .types import (AffineMap, AxisRange, CodecError, CovarianceRepairError, EStep,  # noqa: F401
                    FitConfig, FitResult, GaussianComponent, GmmModel, GridSpec, Histogram2D,
                    InvalidArgument, ModelMeta, ParticleSet, Plane, PruneEvent, WeightedPoints,
                    plane_axes)

__all__ = [
    "AffineMap", "AxisRange", "CodecError", "CovarianceRepairError", "EStep", "FitConfig",
    "FitResult", "GaussianComponent", "GmmModel", "GridSpec", "Histogram2D", "InvalidArgument",
    "ModelMeta", "ParticleSet", "Plane", "PruneEvent", "WeightedPoints", "plane_axes",
]


def __getattr__(name):
    # Compute entry points live in .api, which binds the CUDA library on first use.
    import importlib
    if name.startswith("_") or name in ("api", "cells", "build"):
        raise AttributeError(name)
    api = importlib.import_module(__name__ + ".api")
    try:
        return getattr(api, name)
    except AttributeError:
        raise AttributeError(name) from None
