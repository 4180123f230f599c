"""Domain types and constants of the render + upscale path.

Mirrors the reference's ``splinesplat.core`` surface that the hot path uses
(core.py:23-149): the blend constants, the exception classes (so callers'
``except`` clauses keep working), ``logistic``/``logit`` and the struct-of-
arrays float64 ``Scene`` container.  A ``Scene`` is a host (numpy) object;
the GPU path uploads it once and caches the device copy (see
``device.DeviceScene``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

ALPHA_CLAMP = 0.999          # core.py:23 — keeps 1 - alpha >= 1e-3 for the inversion
ALPHA_CULL = 1.0 / 255.0     # core.py:24 — per-pixel contribution threshold
EARLY_TERMINATION = 1e-4     # core.py:25 — stop once 1 - A drops below this
TILE = 16                    # raster_forward.py:24


class ParameterError(ValueError):
    """Out-of-domain parameters (core.py:28-29)."""


class DegenerateCovarianceError(ParameterError):
    """Numerically singular covariance (core.py:32-33)."""


class DimensionError(ValueError):
    """Invalid or mismatched image dimensions (core.py:36-37)."""


class UnsupportedScaleError(ValueError):
    """Upscaling factor below 1 (core.py:40-41)."""


def logistic(x):
    """core.py:44-45."""
    return 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))


def logit(p):
    """core.py:48-50."""
    p = np.asarray(p, dtype=np.float64)
    return np.log(p) - np.log1p(-p)


@dataclass(frozen=True)
class Gaussian2D:
    """One splat in reference-resolution pixels (core.py:53-72): a value object;
    the renderer only ever sees the struct-of-arrays ``Scene``."""

    mean: tuple
    log_scale: tuple
    rotation: float
    opacity_logit: float
    color: tuple
    depth: float

    def __post_init__(self):
        flat = [*self.mean, *self.log_scale, self.rotation, self.opacity_logit, *self.color, self.depth]
        if not np.all(np.isfinite(np.asarray(flat, dtype=np.float64))):
            raise ParameterError("Gaussian2D requires finite parameters")

    @property
    def opacity(self) -> float:
        return float(logistic(self.opacity_logit))


@dataclass
class Scene:
    """Splats over a reference-resolution canvas, struct-of-arrays float64.

    Same fields, shapes and validation as the reference Scene (core.py:75-106).
    ``version`` is bumped by :meth:`touch`; the device cache keys on
    (id, version) so in-place edits must call it (or build a new Scene).
    """

    means: np.ndarray
    log_scales: np.ndarray
    rotations: np.ndarray
    opacity_logits: np.ndarray
    colors: np.ndarray
    depths: np.ndarray
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    reference_resolution: tuple = (64, 64)
    version: int = 0

    def __post_init__(self):
        self.means = np.atleast_2d(np.asarray(self.means, dtype=np.float64))
        self.log_scales = np.atleast_2d(np.asarray(self.log_scales, dtype=np.float64))
        self.rotations = np.atleast_1d(np.asarray(self.rotations, dtype=np.float64))
        self.opacity_logits = np.atleast_1d(np.asarray(self.opacity_logits, dtype=np.float64))
        self.colors = np.atleast_2d(np.asarray(self.colors, dtype=np.float64))
        self.depths = np.atleast_1d(np.asarray(self.depths, dtype=np.float64))
        self.background = np.asarray(self.background, dtype=np.float64).reshape(3)
        w, h = self.reference_resolution
        if w <= 0 or h <= 0:
            raise DimensionError("reference_resolution must be positive")
        if not np.all(np.isfinite(self.depths)):
            raise ParameterError("depth keys must be finite")

    @property
    def n(self) -> int:
        return len(self.depths)

    def gaussian(self, i: int) -> Gaussian2D:
        """Splat ``i`` as a value object (core.py:117-125)."""
        return Gaussian2D(mean=tuple(float(v) for v in self.means[i]),
                          log_scale=tuple(float(v) for v in self.log_scales[i]),
                          rotation=float(self.rotations[i]), opacity_logit=float(self.opacity_logits[i]),
                          color=tuple(float(v) for v in self.colors[i]), depth=float(self.depths[i]))

    @property
    def gaussians(self) -> list:
        """Every splat as a Gaussian2D, storage order (core.py:113-115)."""
        return [self.gaussian(i) for i in range(self.n)]

    @classmethod
    def from_gaussians(cls, gaussians, background=(0.0, 0.0, 0.0), reference_resolution=(64, 64)) -> "Scene":
        """Struct-of-arrays scene from value objects (core.py:127-143)."""
        gs = list(gaussians)

        def col(get, width):
            a = np.asarray([get(g) for g in gs], dtype=np.float64)
            return a.reshape(len(gs), width) if width > 1 else a.reshape(len(gs))

        return cls(col(lambda g: g.mean, 2), col(lambda g: g.log_scale, 2), col(lambda g: g.rotation, 1),
                   col(lambda g: g.opacity_logit, 1), col(lambda g: g.color, 3), col(lambda g: g.depth, 1),
                   np.asarray(background, dtype=np.float64), reference_resolution)

    def touch(self) -> None:
        """Mark parameters as changed (invalidates the device copy)."""
        self.version += 1

    @classmethod
    def empty(cls, background=(0.0, 0.0, 0.0), reference_resolution=(64, 64)) -> "Scene":
        return cls(np.zeros((0, 2)), np.zeros((0, 2)), np.zeros(0), np.zeros(0),
                   np.zeros((0, 3)), np.zeros(0), np.asarray(background, np.float64),
                   reference_resolution)

    @classmethod
    def from_arrays(cls, obj) -> "Scene":
        """Adopt any object exposing the reference Scene's field names."""
        return cls(obj.means, obj.log_scales, obj.rotations, obj.opacity_logits,
                   obj.colors, obj.depths, obj.background, tuple(obj.reference_resolution))

    def copy(self) -> "Scene":
        return Scene(self.means.copy(), self.log_scales.copy(), self.rotations.copy(),
                     self.opacity_logits.copy(), self.colors.copy(), self.depths.copy(),
                     self.background.copy(), self.reference_resolution)


def covariance_from_params(log_scale, rotation: float) -> np.ndarray:
    """Sigma = R diag(exp(2 l)) R^T (core.py:175-182); host helper for tests."""
    log_scale = np.asarray(log_scale, dtype=np.float64)
    if not (np.all(np.isfinite(log_scale)) and math.isfinite(rotation)):
        raise ParameterError("log_scale and rotation must be finite")
    c, s = math.cos(rotation), math.sin(rotation)
    r = np.array([[c, -s], [s, c]])
    return r @ np.diag(np.exp(2.0 * log_scale)) @ r.T
