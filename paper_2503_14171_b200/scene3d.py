"""3D front-end: 3D Gaussians + pinhole camera -> the 2D
splat scene of the reference path (EWA local-affine projection).

``project_gaussians`` runs ``splat_project_3d`` on the GPU and returns a
``DeviceScene`` in the reference's 2D parametrisation (core.py:75-93, 175-182),
so ``render_forward`` / ``upscale_spline`` / ``render_backward`` apply unchanged;
``render_forward_3d`` chains the two.  The reference package itself is 2D-only,
so this stage is pinned to the float64 restatement ``oracle.project_gaussians``,
not to reference outputs ("parity unpinned" for f3).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import DimensionError, ParameterError
from .device import DeviceScene


@dataclass
class Scene3D:
    """3D Gaussians, struct-of-arrays float64 (host)."""

    means: np.ndarray            # (N, 3) world positions
    log_scales: np.ndarray       # (N, 3)
    quats: np.ndarray            # (N, 4) w, x, y, z (normalised on use)
    opacity_logits: np.ndarray   # (N,)
    colors: np.ndarray           # (N, 3)
    background: np.ndarray = None

    def __post_init__(self):
        self.means = np.asarray(self.means, np.float64).reshape(-1, 3)
        n = len(self.means)
        self.log_scales = np.asarray(self.log_scales, np.float64).reshape(n, 3)
        self.quats = np.asarray(self.quats, np.float64).reshape(n, 4)
        self.opacity_logits = np.asarray(self.opacity_logits, np.float64).reshape(n)
        self.colors = np.asarray(self.colors, np.float64).reshape(n, 3)
        self.background = np.zeros(3) if self.background is None else np.asarray(self.background, np.float64)
        for a in (self.means, self.log_scales, self.quats, self.opacity_logits, self.colors):
            if not np.all(np.isfinite(a)):
                raise ParameterError("3D scene contains non-finite values")

    @property
    def n(self) -> int:
        return len(self.means)


@dataclass
class Camera:
    """Pinhole camera: x_cam = R x_world + t; pixel = (fx x/z + cx, fy y/z + cy) on a
    width x height image (the 2D scene's reference resolution)."""

    R: np.ndarray
    t: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float = 0.01

    @classmethod
    def look_at(cls, eye, target, up, fov_y_deg: float, width: int, height: int, near: float = 0.01):
        eye, target, up = (np.asarray(v, np.float64) for v in (eye, target, up))
        f = target - eye
        f /= np.linalg.norm(f)
        r = np.cross(f, up)
        r /= np.linalg.norm(r)
        d = np.cross(f, r)                     # image y points down
        R = np.stack([r, d, f])                # rows: camera x, y, z axes
        fy = 0.5 * height / np.tan(np.radians(fov_y_deg) / 2)
        return cls(R, -R @ eye, fy, fy, width / 2.0, height / 2.0, width, height, near)

    def c_struct(self) -> _lib.CameraT:
        if self.fx <= 0 or self.fy <= 0 or self.near <= 0:
            raise ParameterError("camera focal lengths and near plane must be positive")
        if self.width <= 0 or self.height <= 0:
            raise DimensionError("camera image dimensions must be positive")
        c = _lib.CameraT()
        R = np.asarray(self.R, np.float64).reshape(9)
        t = np.asarray(self.t, np.float64).reshape(3)
        for i in range(9):
            c.R[i] = float(R[i])
        for i in range(3):
            c.t[i] = float(t[i])
        c.fx, c.fy, c.cx, c.cy, c.near_plane = (float(v) for v in (self.fx, self.fy, self.cx, self.cy, self.near))
        return c


def project_gaussians(scene: Scene3D, camera: Camera, device=None) -> DeviceScene:
    """The 2D scene this camera sees (device, float64, prepared: depth-sorted)."""
    dev = device or torch.device("cuda", torch.cuda.current_device())
    n = scene.n

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(dev)

    mu, ls3, q, lg = up(scene.means), up(scene.log_scales), up(scene.quats), up(scene.opacity_logits)
    out = {"means": torch.empty((n, 2), dtype=torch.float64, device=dev),
           "log_scales": torch.empty((n, 2), dtype=torch.float64, device=dev),
           "rotations": torch.empty(n, dtype=torch.float64, device=dev),
           "opacity_logits": torch.empty(n, dtype=torch.float64, device=dev),
           "depths": torch.empty(n, dtype=torch.float64, device=dev)}
    cam = camera.c_struct()
    _lib.check(_lib.load().splat_project_3d(n, _lib.ptr(mu), _lib.ptr(ls3), _lib.ptr(q), _lib.ptr(lg), cam,
                                            _lib.ptr(out["means"]), _lib.ptr(out["log_scales"]),
                                            _lib.ptr(out["rotations"]), _lib.ptr(out["opacity_logits"]),
                                            _lib.ptr(out["depths"]), _lib.stream_ptr()))
    return DeviceScene(**out, colors=up(scene.colors), background=tuple(float(v) for v in scene.background),
                       reference_resolution=(camera.width, camera.height)).prepare()


def render_forward_3d(scene: Scene3D, camera: Camera, out_width: int, out_height: int, **kw):
    """Project, then render with analytic gradients at out_width x out_height."""
    from .raster_forward import render_forward
    return render_forward(project_gaussians(scene, camera), out_width, out_height, **kw)


def synthetic_scene_3d(n: int, seed: int = 5, extent: float = 1.0, scale_range=(0.005, 0.03)) -> Scene3D:
    """Random Gaussians in a cube of half-size ``extent`` around the origin."""
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 4))
    return Scene3D(means=rng.uniform(-extent, extent, (n, 3)),
                   log_scales=np.log(rng.uniform(scale_range[0], scale_range[1], (n, 3))),
                   quats=q / np.linalg.norm(q, axis=1, keepdims=True),
                   opacity_logits=np.log(p := rng.uniform(0.15, 0.85, n)) - np.log1p(-p),
                   colors=rng.uniform(0.0, 1.0, (n, 3)),
                   background=np.array([0.12, 0.10, 0.14]))
