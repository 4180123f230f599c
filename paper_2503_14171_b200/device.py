"""Device-resident scenes and per-view frame workspaces.

A host ``Scene`` (numpy float64, reference layout) is uploaded once and
prepared once per scene (stable depth sort + view-independent float64 terms,
``splat_scene_prepare``); the device copy is cached on the Scene object, keyed
by the identity of its arrays and its ``version`` counter (call
``Scene.touch()`` after editing arrays in place).  SURVEY.md 8(b): a per-call
upload of ~80 MB at 1M splats would cost milliseconds over PCIe.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import ParameterError, Scene

FIELDS = ("means", "log_scales", "rotations", "opacity_logits", "colors", "depths")


def _device(device=None) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2503_14171_b200 needs a CUDA device (B200, sm_100a)")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


@dataclass
class DeviceScene:
    """Float64 scene parameters on the GPU (storage order) + prepared constants."""

    means: torch.Tensor
    log_scales: torch.Tensor
    rotations: torch.Tensor
    opacity_logits: torch.Tensor
    colors: torch.Tensor
    depths: torch.Tensor
    background: tuple
    reference_resolution: tuple
    const: torch.Tensor | None = None   # splat_scene_prepare output (uint8 blob)

    @property
    def n(self) -> int:
        return int(self.depths.shape[0])

    @property
    def device(self) -> torch.device:
        return self.means.device

    def c_scene(self) -> _lib.SceneT:
        s = _lib.SceneT()
        s.n = self.n
        for f in FIELDS:
            setattr(s, f, _lib.ptr(getattr(self, f)) if self.n else None)
        return s

    def prepare(self, stream=None) -> "DeviceScene":
        """(Re)compute the per-scene constants (depth order, conic terms)."""
        lib = _lib.load()
        n = self.n
        cbytes = lib.splat_scene_const_bytes(n)
        wbytes = lib.splat_scene_workspace_bytes(n)
        if self.const is None or self.const.numel() < cbytes:
            self.const = torch.empty(cbytes, dtype=torch.uint8, device=self.device)
        ws = torch.empty(wbytes, dtype=torch.uint8, device=self.device)
        cs = self.c_scene()
        _lib.check(lib.splat_scene_prepare(cs, _lib.ptr(self.const), cbytes, _lib.ptr(ws), wbytes,
                                           _lib.stream_ptr(stream)))
        self._ws = ws  # keep alive until the stream has consumed it
        return self

    def refresh(self, stream=None) -> "DeviceScene":
        """Recompute the per-scene terms after an in-place parameter update (same depth order)."""
        if self.const is None:
            return self.prepare(stream)
        lib = _lib.load()
        _lib.check(lib.splat_scene_refresh(self.c_scene(), _lib.ptr(self.const), self.const.numel(),
                                           _lib.stream_ptr(stream)))
        return self

    def order(self) -> torch.Tensor:
        """Rank -> storage index (sort_by_depth), int64."""
        lib = _lib.load()
        if self.n == 0:
            return torch.zeros(0, dtype=torch.int64, device=self.device)
        p = lib.splat_scene_order(_lib.ptr(self.const), self.n)
        off = p - self.const.data_ptr()
        return self.const[off:off + 4 * self.n].view(torch.int32).to(torch.int64)

    @classmethod
    def from_host(cls, scene: Scene, device=None) -> "DeviceScene":
        dev = _device(device)
        t = {f: torch.from_numpy(np.ascontiguousarray(getattr(scene, f), dtype=np.float64)).to(
            dev, non_blocking=False) for f in FIELDS}
        n = scene.n
        t["means"] = t["means"].reshape(n, 2)
        t["log_scales"] = t["log_scales"].reshape(n, 2)
        t["colors"] = t["colors"].reshape(n, 3)
        return cls(**t, background=tuple(float(v) for v in scene.background),
                   reference_resolution=tuple(scene.reference_resolution)).prepare()


def _cache_key(scene: Scene):
    return (scene.version,) + tuple(id(getattr(scene, f)) for f in FIELDS)


def to_device(scene, device=None) -> DeviceScene:
    """Device copy of a Scene (cached) or pass a DeviceScene through."""
    if isinstance(scene, DeviceScene):
        if scene.const is None:
            scene.prepare()
        return scene
    if not isinstance(scene, Scene):
        scene = Scene.from_arrays(scene)
    if not np.all(np.isfinite(scene.depths)):
        raise ParameterError("depth keys must be finite")
    key = _cache_key(scene)
    dev = _device(device)
    cached = getattr(scene, "_device_cache", None)
    if cached is not None and cached[0] == key and cached[1].device == dev:
        return cached[1]
    ds = DeviceScene.from_host(scene, dev)
    scene._device_cache = (key, ds)
    return ds
