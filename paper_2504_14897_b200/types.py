"""Python mirror of the reference value types on the hot path.

Each dataclass restates one reference struct (proj/include/vdfc/*.hpp) with numpy
arrays in place of Eigen matrices (same shapes, column-major semantics where the
reference stores matrices). Exceptions mirror the reference's exception classes:
``std::invalid_argument`` -> :class:`InvalidArgument` (a ``ValueError``),
``std::runtime_error`` -> ``RuntimeError``, ``CovarianceRepairError`` /
``CodecError`` (types.hpp:83-101) -> the classes below.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class CovarianceRepairError(RuntimeError):
    """vdfc::CovarianceRepairError (types.hpp:99-101)."""


class CodecError(RuntimeError):
    """vdfc::CodecError (types.hpp:93-96)."""


class Plane(enum.IntEnum):
    """types.hpp:18."""
    uv = 0
    vw = 1
    uw = 2


def plane_axes(p: Plane) -> tuple[int, int]:
    """types.hpp:20-27."""
    return {Plane.uv: (0, 1), Plane.vw: (1, 2), Plane.uw: (0, 2)}[Plane(p)]


@dataclass
class AxisRange:
    """types.hpp:32-39."""
    lo: float = 0.0
    hi: float = 0.0

    def width(self) -> float:
        return self.hi - self.lo

    def valid(self) -> bool:
        return bool(np.isfinite(self.lo) and np.isfinite(self.hi) and self.lo < self.hi)


@dataclass
class GridSpec:
    """types.hpp:43-55."""
    n_bins: int
    x: AxisRange
    y: AxisRange

    def dx(self) -> float:
        return self.x.width() / self.n_bins

    def dy(self) -> float:
        return self.y.width() / self.n_bins

    def center_x(self, i: int) -> float:
        return self.x.lo + (i + 0.5) * self.dx()

    def center_y(self, j: int) -> float:
        return self.y.lo + (j + 0.5) * self.dy()

    def bin_area(self) -> float:
        return self.dx() * self.dy()

    def valid(self) -> bool:
        return self.n_bins >= 1 and self.x.valid() and self.y.valid()


@dataclass
class AffineMap:
    """types.hpp:59-81: z = (x - offset) / scale."""
    scale: np.ndarray
    offset: np.ndarray

    @staticmethod
    def identity(d: int) -> "AffineMap":
        return AffineMap(np.ones(d), np.zeros(d))

    def dim(self) -> int:
        return len(self.scale)

    def is_identity(self) -> bool:
        return bool(np.all(self.scale == 1.0) and np.all(self.offset == 0.0))

    def forward(self, x):
        return (np.asarray(x) - self.offset) / self.scale

    def inverse(self, z):
        return np.asarray(z) * self.scale + self.offset

    def volume(self) -> float:
        return float(np.prod(self.scale))


@dataclass
class ParticleSet:
    """synthdata.hpp:13-28. ``velocities`` is N x d (stored column-major, i.e. SoA)."""
    velocities: np.ndarray
    weights: Optional[np.ndarray] = None
    species_label: str = ""
    nominal_temperature: Optional[np.ndarray] = None

    def count(self) -> int:
        return int(self.velocities.shape[0])

    def dimension(self) -> int:
        return int(self.velocities.shape[1]) if self.velocities.ndim == 2 else 0

    def has_weights(self) -> bool:
        return self.weights is not None and len(self.weights) > 0

    def total_weight(self) -> float:
        return float(np.sum(self.weights)) if self.has_weights() else float(self.count())

    def validate(self) -> None:
        """synthdata.cpp:18-31. The per-particle weight check runs on the device."""
        d = self.dimension()
        if d not in (2, 3):
            raise InvalidArgument("particle dimension must be 2 or 3")
        if self.has_weights() and len(self.weights) != self.count():
            raise InvalidArgument("weights size does not match particle count")
        t = self.nominal_temperature
        if t is None or len(t) != d:
            raise InvalidArgument("nominal_temperature must have one entry per axis")
        if not np.all(np.asarray(t) > 0.0):
            raise InvalidArgument("nominal_temperature must be > 0 on every axis")


@dataclass
class Histogram2D:
    """histogram.hpp:16-28. ``counts[i, j]`` = x bin i, y bin j."""
    counts: np.ndarray
    range_x: AxisRange
    range_y: AxisRange
    plane: Plane = Plane.uv
    n_bins: int = 0
    out_of_range_count: float = 0.0
    species_label: str = ""

    def in_range_count(self) -> float:
        return float(np.sum(self.counts))

    def degenerate(self) -> bool:
        return not (self.in_range_count() > 0.0)

    def grid(self) -> GridSpec:
        return GridSpec(self.n_bins, self.range_x, self.range_y)


@dataclass
class WeightedPoints:
    """histogram.hpp:33-43."""
    points: np.ndarray  # N x d
    weights: np.ndarray  # N
    total_weight: float = 0.0

    def count(self) -> int:
        return int(self.points.shape[0])

    def dimension(self) -> int:
        return int(self.points.shape[1])

    @staticmethod
    def from_(pts, w) -> "WeightedPoints":
        """WeightedPoints::from (histogram.cpp:12-18)."""
        pts = np.asarray(pts, dtype=float)
        w = np.asarray(w, dtype=float)
        out = WeightedPoints(pts, w, float(np.sum(w)))
        out.validate()
        return out

    def validate(self) -> None:
        """histogram.cpp:20-26."""
        if self.points.shape[0] != len(self.weights):
            raise InvalidArgument("weighted points: weight count does not match point count")
        if self.points.shape[0] == 0:
            raise InvalidArgument("weighted points: empty")
        if not np.all(self.weights >= 0.0):
            raise InvalidArgument("weighted points: weights must be >= 0")
        if not np.any(self.weights > 0.0):
            raise InvalidArgument("weighted points: at least one weight must be > 0")


@dataclass
class GaussianComponent:
    """wgmm.hpp:14-22."""
    weight: float
    mean: np.ndarray
    covariance: np.ndarray

    def set_covariance(self, m) -> None:
        m = np.array(m, dtype=float)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise InvalidArgument("covariance must be square")
        iu = np.triu_indices(m.shape[0], 1)
        m[(iu[1], iu[0])] = m[iu]
        self.covariance = m


@dataclass
class GmmModel:
    """wgmm.hpp:27-39."""
    components: list
    normalization: AffineMap
    dimension: int = 0

    def size(self) -> int:
        return len(self.components)

    def validate(self) -> None:
        """wgmm.cpp:46-63."""
        if self.dimension < 1:
            raise InvalidArgument("model dimension must be positive")
        if not self.components:
            raise InvalidArgument("model has no components")
        if self.normalization.dim() != self.dimension:
            raise InvalidArgument("normalization map dimension mismatch")
        total = 0.0
        for c in self.components:
            if not c.weight > 0.0:
                raise InvalidArgument("component weight must be > 0")
            if len(c.mean) != self.dimension or np.shape(c.covariance) != (self.dimension,) * 2:
                raise InvalidArgument("component dimension mismatch")
            if not np.array_equal(c.covariance, np.transpose(c.covariance)):
                raise InvalidArgument("component covariance is not symmetric")
            total += c.weight
        if abs(total - 1.0) > 1e-12:
            raise InvalidArgument("component weights must sum to 1")


@dataclass
class FitConfig:
    """wgmm.hpp:41-56 (defaults identical)."""
    initial_components: int = 12
    max_em_iterations: int = 100
    prune_threshold: float = 0.005
    prune_check_interval: int = 10
    loglik_rel_tolerance: float = 1e-6
    seed: int = 0
    warm_start: Optional[GmmModel] = None
    temperature: Optional[np.ndarray] = None
    # Not in the reference: FP32 E-step on the cell-batched path (tolerance 1e-4).
    estep_fp32: bool = False


@dataclass
class PruneEvent:
    """wgmm.hpp:58-62."""
    iteration: int = 0
    component: int = 0
    weight: float = 0.0


@dataclass
class FitResult:
    """wgmm.hpp:64-70."""
    model: GmmModel
    loglik_trace: list = field(default_factory=list)
    iterations_used: int = 0
    pruning_events: list = field(default_factory=list)
    converged: bool = False


@dataclass
class EStep:
    """wgmm.hpp:88-92. ``responsibilities`` is M x N."""
    responsibilities: np.ndarray
    loglik: float
    unrepairable: list


@dataclass
class ModelMeta:
    """codec.hpp:20-25."""
    species_label: str = ""
    plane: Optional[Plane] = None
    cycle: int = 0
    axis_ranges: list = field(default_factory=list)
