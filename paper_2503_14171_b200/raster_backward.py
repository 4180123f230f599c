"""Reverse mode of the gradient rasterizer — drop-in for splinesplat.raster_backward.

``PixelAdjoint`` (raster_backward.py:25-37), ``SceneGrads`` (:40-53),
``invert_alpha_state`` (:56-70, scalar host helper) and
``render_backward(scene, fwd, adj, *, threads=1)`` (:73-153) with the
reference's validation (DimensionError on shape mismatch, ParameterError on
non-finite adjoints) and storage-order gradients.

The GPU path (csrc/raster_bwd.cu) replays each pixel's contributors back to
front from the forward's float64 terminal state, so ``fwd`` should come from
``render_forward(..., train=True)``; a GradientImage without that private
state is re-rendered in training mode first (SURVEY.md 8(b) "Hidden state").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import DimensionError, ParameterError
from .device import DeviceScene, to_device
from .raster_forward import GradientImage, make_view, render_forward

__all__ = ["PixelAdjoint", "SceneGrads", "invert_alpha_state", "render_backward", "GradBuffer"]


@dataclass
class PixelAdjoint:
    """Upstream adjoints for each GradientImage channel (all (H, W, 3)).

    Stored packed as (H, W, 4, 3) = [w, wx, wy, wxy]; a SourceAdjoint from
    upscale_backward already has that layout and is adopted without a copy.
    """

    planes: torch.Tensor

    w = property(lambda s: s.planes[:, :, 0, :])
    wx = property(lambda s: s.planes[:, :, 1, :])
    wy = property(lambda s: s.planes[:, :, 2, :])
    wxy = property(lambda s: s.planes[:, :, 3, :])

    @classmethod
    def of(cls, w, wx, wy, wxy, device=None) -> "PixelAdjoint":
        dev = device or torch.device("cuda", torch.cuda.current_device())

        def t(a):
            a = a if torch.is_tensor(a) else torch.from_numpy(np.asarray(a))
            return a.to(device=dev, dtype=torch.float32)
        shapes = {tuple(x.shape) for x in (w, wx, wy, wxy)}
        if len(shapes) != 1:
            raise DimensionError("adjoint dimensions must match the forward image")
        return cls(torch.stack([t(w), t(wx), t(wy), t(wxy)], dim=2).contiguous())

    @classmethod
    def from_source(cls, src) -> "PixelAdjoint":
        """Adopt an upscale_backward SourceAdjoint (same packed layout)."""
        return cls(src.planes)

    @classmethod
    def zeros(cls, width: int, height: int, device=None) -> "PixelAdjoint":
        dev = device or torch.device("cuda", torch.cuda.current_device())
        return cls(torch.zeros((height, width, 4, 3), dtype=torch.float32, device=dev))


class GradBuffer:
    """Flat float32 storage-order gradients: [means | log_scales | rotations | logits | colors]."""

    def __init__(self, n: int, device):
        self.n = n
        self.flat = torch.zeros(11 * max(n, 1), dtype=torch.float32, device=device)

    def zero_(self):
        self.flat.zero_()
        return self

    def grads(self) -> "SceneGrads":
        n, f = self.n, self.flat
        return SceneGrads(d_means=f[0:2 * n].view(n, 2), d_log_scales=f[2 * n:4 * n].view(n, 2),
                          d_rotations=f[4 * n:5 * n], d_opacity_logits=f[5 * n:6 * n],
                          d_colors=f[6 * n:9 * n].view(n, 3))


@dataclass
class SceneGrads:
    """Per-splat parameter gradients in the scene's storage order (raster_backward.py:40-53)."""

    d_means: torch.Tensor           # (N, 2)
    d_log_scales: torch.Tensor      # (N, 2)
    d_rotations: torch.Tensor       # (N,)
    d_opacity_logits: torch.Tensor  # (N,)
    d_colors: torch.Tensor          # (N, 3)

    FIELDS = ("d_means", "d_log_scales", "d_rotations", "d_opacity_logits", "d_colors")

    def numpy(self) -> dict:
        return {f: getattr(self, f).double().cpu().numpy() for f in self.FIELDS}


def invert_alpha_state(a_i, ax_i, ay_i, axy_i, alpha, alpha_x, alpha_y, alpha_xy):
    """Step the accumulated-alpha state back across one splat (raster_backward.py:56-70)."""
    om = 1.0 - alpha
    if om < 1e-3:
        raise ParameterError("inversion requires 1 - alpha >= 1e-3")
    a_prev = (a_i - alpha) / om
    t = 1.0 - a_prev
    ax_prev = (ax_i - t * alpha_x) / om
    ay_prev = (ay_i - t * alpha_y) / om
    axy_prev = (axy_i - t * alpha_xy + ax_prev * alpha_y + ay_prev * alpha_x) / om
    return a_prev, ax_prev, ay_prev, axy_prev


def _as_adjoint(adj, h: int, w: int) -> PixelAdjoint:
    if isinstance(adj, PixelAdjoint):
        pa = adj
    elif hasattr(adj, "planes") and hasattr(adj, "d_color"):
        pa = PixelAdjoint.from_source(adj)
    else:
        for a in (adj.w, adj.wx, adj.wy, adj.wxy):
            if tuple(a.shape) != (h, w, 3):
                raise DimensionError("adjoint dimensions must match the forward image")
        pa = PixelAdjoint.of(adj.w, adj.wx, adj.wy, adj.wxy)
    if tuple(pa.planes.shape) != (h, w, 4, 3):
        raise DimensionError("adjoint dimensions must match the forward image")
    if not pa.planes.is_contiguous():
        pa = PixelAdjoint(pa.planes.contiguous())
    return pa


def render_backward(scene, fwd: GradientImage, adj, *, threads: int = 1, view=None,
                    out: GradBuffer | None = None, accumulate: bool = False,
                    check_finite: bool = True) -> SceneGrads:
    """Backpropagate channel adjoints to splat parameter gradients (raster_backward.py:73-153)."""
    del threads
    h, w = fwd.height, fwd.width
    pa = _as_adjoint(adj, h, w)
    if check_finite and not bool(torch.isfinite(pa.planes).all()):
        raise ParameterError("adjoint must be finite")
    ds = to_device(scene)
    if out is None:
        out = GradBuffer(ds.n, ds.device)
    elif not accumulate:
        out.zero_()
    if ds.n == 0:
        return out.grads()
    if fwd.state is None or fwd.frame is None or fwd.scene is not ds:
        # no private float64 terminal state: re-render this view in training mode
        fwd = render_forward(ds, w, h, view=view, train=True)
    lib = _lib.load()
    frame = fwd.frame
    v = fwd.view if fwd.view is not None else make_view(ds, w, h, view)
    nbytes = lib.splat_backward_workspace_bytes(ds.n, frame.capacity)
    bws = torch.empty(nbytes, dtype=torch.uint8, device=ds.device)
    _lib.check(lib.splat_render_backward(_lib.ptr(ds.const), ds.c_scene(), v, w, h, fwd.c_gimg(),
                                         _lib.ptr(pa.planes), _lib.ptr(frame.ws), frame.nbytes, frame.capacity,
                                         _lib.ptr(bws), nbytes, _lib.ptr(out.flat), int(bool(accumulate)),
                                         _lib.stream_ptr()))
    out._ws = bws
    return out.grads()


def render_backward_rank(ds: DeviceScene, fwd: GradientImage, adj, rank_grads: torch.Tensor,
                         accumulate: bool = True, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Multi-view training building block: add this view's render-space gradient
    terms, view-scaled and in rank order ((n, 9) float32), into ``rank_grads``;
    :func:`chain_grads` maps the sum over views to parameter gradients once
    (raster_backward.py:126-152 applied to the summed terms; the chain is linear)."""
    h, w = fwd.height, fwd.width
    pa = _as_adjoint(adj, h, w)
    if ds.n == 0:
        return rank_grads
    if fwd.state is None or fwd.frame is None or fwd.scene is not ds:
        raise ParameterError("render_backward_rank needs the training-mode forward of this scene")
    lib = _lib.load()
    frame = fwd.frame
    nbytes = lib.splat_backward_workspace_bytes(ds.n, frame.capacity)
    if workspace is not None and workspace.numel() >= nbytes:
        bws = workspace
    else:
        bws = torch.empty(nbytes, dtype=torch.uint8, device=ds.device)
    _lib.check(lib.splat_render_backward_rank(_lib.ptr(ds.const), ds.c_scene(), fwd.view, w, h, fwd.c_gimg(),
                                              _lib.ptr(pa.planes), _lib.ptr(frame.ws), frame.nbytes,
                                              frame.capacity, _lib.ptr(bws), nbytes, _lib.ptr(rank_grads),
                                              int(bool(accumulate)), _lib.stream_ptr()))
    rank_grads._bws = bws   # keep the workspace alive while the stream uses it
    return rank_grads


def chain_grads(ds: DeviceScene, rank_grads: torch.Tensor, out: GradBuffer, accumulate: bool = False) -> GradBuffer:
    """Parameter gradients (storage order) from summed rank-order terms."""
    lib = _lib.load()
    _lib.check(lib.splat_chain_grads(_lib.ptr(ds.const), ds.c_scene(), _lib.ptr(rank_grads), _lib.ptr(out.flat),
                                     int(bool(accumulate)), _lib.stream_ptr()))
    return out
