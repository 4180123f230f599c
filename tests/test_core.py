"""Host-side domain types of the drop-in (core.py:53-149): Gaussian2D value
objects and the Scene container's conversions and validation (no GPU)."""

import math

import numpy as np
import pytest

from paper_2503_14171_b200.core import Gaussian2D, ParameterError, Scene, DimensionError, logistic


def _scene(n=5, seed=0):
    rng = np.random.default_rng(seed)
    return Scene(rng.uniform(0, 64, (n, 2)), rng.normal(1.0, 0.3, (n, 2)), rng.uniform(-3, 3, n),
                 rng.normal(0, 1, n), rng.uniform(0, 1, (n, 3)), rng.uniform(0, 1, n),
                 np.array([0.1, 0.2, 0.3]), (64, 48))


def test_gaussians_round_trip_through_from_gaussians():
    sc = _scene()
    gs = sc.gaussians
    assert len(gs) == sc.n and all(isinstance(g, Gaussian2D) for g in gs)
    g2 = sc.gaussian(2)
    assert g2.mean == (sc.means[2, 0], sc.means[2, 1]) and g2.depth == sc.depths[2]
    assert g2.opacity == pytest.approx(float(logistic(sc.opacity_logits[2])), rel=0, abs=0)
    back = Scene.from_gaussians(gs, background=sc.background, reference_resolution=sc.reference_resolution)
    for f in ("means", "log_scales", "rotations", "opacity_logits", "colors", "depths", "background"):
        assert np.array_equal(getattr(back, f), getattr(sc, f)), f
        assert getattr(back, f).dtype == np.float64
    assert back.reference_resolution == (64, 48)


def test_from_gaussians_empty_has_reference_shapes():
    sc = Scene.from_gaussians([])
    assert sc.n == 0 and sc.means.shape == (0, 2) and sc.log_scales.shape == (0, 2)
    assert sc.colors.shape == (0, 3) and sc.rotations.shape == (0,) and sc.reference_resolution == (64, 64)


def test_gaussian2d_rejects_non_finite_parameters():
    ok = dict(mean=(1.0, 2.0), log_scale=(0.0, 0.0), rotation=0.0, opacity_logit=0.0,
              color=(0.5, 0.5, 0.5), depth=0.5)
    Gaussian2D(**ok)
    for key, bad in (("mean", (math.nan, 0.0)), ("rotation", math.inf), ("color", (0.0, -math.inf, 0.0)),
                     ("depth", math.nan)):
        with pytest.raises(ParameterError):
            Gaussian2D(**{**ok, key: bad})
    with pytest.raises(Exception):
        Gaussian2D(**ok).depth = 1.0   # frozen value object


def test_scene_validation():
    with pytest.raises(DimensionError):
        Scene.from_gaussians([], reference_resolution=(0, 4))
    sc = _scene()
    with pytest.raises(ParameterError):
        Scene(sc.means, sc.log_scales, sc.rotations, sc.opacity_logits, sc.colors,
              np.where(np.arange(sc.n) == 1, np.nan, sc.depths))
