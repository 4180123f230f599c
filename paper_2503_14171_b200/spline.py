"""Gradient-aware bicubic spline upscaling — drop-in for splinesplat.spline's hot path.

``upscale_spline`` (spline.py:162-178), ``upscale_backward`` (spline.py:191-229),
``SourceAdjoint`` (spline.py:181-188), ``fd_gradients`` / ``fd_gradients_backward``
(spline.py:274-297), with the reference's argument meaning, output sizing
(``_output_size``, spline.py:94-99) and exceptions.  Inputs may be a GPU
``GradientImage`` or anything with ``color/d_dx/d_dy/d_dxdy`` (H, W, 3) arrays;
outputs are float32 CUDA tensors.  Kernels: csrc/upscale.cu.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import DimensionError, UnsupportedScaleError
from .raster_forward import GradientImage

__all__ = ["upscale_spline", "upscale_backward", "SourceAdjoint", "fd_gradients",
           "fd_gradients_backward", "output_size", "upscale_plan", "check_output"]


def output_size(in_w: int, in_h: int, factor: float):
    """spline.py:94-99: round-half-up of each scaled dimension."""
    if factor < 1.0:
        raise UnsupportedScaleError(f"upscale factor must be >= 1, got {factor}")
    return int(math.floor(in_w * factor + 0.5)), int(math.floor(in_h * factor + 0.5))


def _as_gimg(img) -> GradientImage:
    if isinstance(img, GradientImage):
        return img
    return GradientImage.from_planes(img.color, img.d_dx, img.d_dy, img.d_dxdy)


def _planes(img: GradientImage) -> torch.Tensor:
    p = img.planes
    if not p.is_contiguous():
        p = p.contiguous()
    return p


def check_output(out: torch.Tensor, out_w: int, out_h: int, device) -> None:
    """A caller-provided destination must be exactly what the kernels write:
    (out_h, out_w, 3) float32, contiguous, on ``device``, and 16-byte aligned
    when rows are written with 16-byte (TMA bulk / vector) stores, i.e. when
    out_w % 4 == 0.  Anything else would be written out of bounds or fault."""
    if not torch.is_tensor(out):
        raise DimensionError("out must be a torch tensor")
    if tuple(out.shape) != (out_h, out_w, 3):
        raise DimensionError(f"out must have shape {(out_h, out_w, 3)}, got {tuple(out.shape)}")
    if out.dtype != torch.float32:
        raise DimensionError("out must be float32")
    if out.device != torch.device(device):
        raise DimensionError(f"out must be on {device}, got {out.device}")
    align = 16 if out_w % 4 == 0 else 4
    if not out.is_contiguous() or out.data_ptr() % align:
        raise DimensionError(f"out must be contiguous and {align}-byte aligned")


_plans: dict = {}


def upscale_plan(in_w: int, in_h: int, out_w: int, out_h: int, device) -> torch.Tensor:
    """Cached per-size axis maps (splat_upscale_plan)."""
    key = (in_w, in_h, out_w, out_h, str(device))
    plan = _plans.get(key)
    if plan is None:
        lib = _lib.load()
        nbytes = lib.splat_upscale_plan_bytes(in_w, in_h, out_w, out_h)
        plan = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _lib.check(lib.splat_upscale_plan(in_w, in_h, out_w, out_h, _lib.ptr(plan), _lib.stream_ptr()))
        _plans[key] = plan
    return plan


def upscale_spline(img, factor: float, *, out_size=None, clamp: bool = True,
                   out: torch.Tensor | None = None) -> torch.Tensor:
    """Upscale from value + analytic derivative planes (spline.py:162-178)."""
    g = _as_gimg(img)
    if out_size is None:
        out_w, out_h = output_size(g.width, g.height, factor)
    else:
        out_w, out_h = (int(v) for v in out_size)
        if out_w < g.width or out_h < g.height:
            raise UnsupportedScaleError("output must be at least source size")
    lib = _lib.load()
    src = _planes(g)
    if src.data_ptr() % 16:
        src = src.clone()   # the source planes are staged with 16-byte bulk copies
    if out is None:
        out = torch.empty((out_h, out_w, 3), dtype=torch.float32, device=src.device)
    else:
        check_output(out, out_w, out_h, src.device)
    plan = upscale_plan(g.width, g.height, out_w, out_h, src.device)
    _lib.check(lib.splat_upscale_forward(_lib.ptr(src), g.width, g.height, _lib.ptr(out), out_w, out_h,
                                         int(bool(clamp)), _lib.ptr(plan), _lib.stream_ptr()))
    return out


@dataclass
class SourceAdjoint:
    """Adjoints of the four upscaler input channels per source pixel (spline.py:181-188).

    Views into one packed (H, W, 4, 3) buffer, which is also the layout the
    rasterizer backward consumes as its PixelAdjoint.
    """

    planes: torch.Tensor

    d_color = property(lambda s: s.planes[:, :, 0, :])
    d_dx = property(lambda s: s.planes[:, :, 1, :])
    d_dy = property(lambda s: s.planes[:, :, 2, :])
    d_dxdy = property(lambda s: s.planes[:, :, 3, :])


def upscale_backward(img, factor: float, adjoint, *, out_size=None,
                     out: torch.Tensor | None = None) -> SourceAdjoint:
    """Exact transpose of the linear upscale map, clamp excluded (spline.py:191-229).

    Gather form: every source pixel's 12 adjoints are written once, in a fixed
    order — deterministic and atomic-free.  ``img`` is used only for its size.
    """
    w, h = img.width, img.height
    if out_size is None:
        out_w, out_h = output_size(w, h, factor)
    else:
        out_w, out_h = (int(v) for v in out_size)
    dev = img.planes.device if isinstance(img, GradientImage) else torch.device("cuda", torch.cuda.current_device())
    adj = adjoint if torch.is_tensor(adjoint) else torch.from_numpy(np.asarray(adjoint))
    adj = adj.to(device=dev, dtype=torch.float32).contiguous()
    if tuple(adj.shape) != (out_h, out_w, 3):
        raise DimensionError("adjoint dimensions must match the upscaled output")
    lib = _lib.load()
    if out is None:
        dsrc = torch.empty((h, w, 4, 3), dtype=torch.float32, device=dev)
    else:
        if tuple(out.shape) != (h, w, 4, 3) or out.dtype != torch.float32 or not out.is_contiguous() \
                or out.device != dev or out.data_ptr() % 16:
            raise DimensionError("out must be a contiguous 16-byte aligned (H, W, 4, 3) float32 tensor")
        dsrc = out
    _lib.check(lib.splat_upscale_backward(_lib.ptr(adj), out_w, out_h, _lib.ptr(dsrc), w, h,
                                          _lib.stream_ptr()))
    return SourceAdjoint(dsrc)


def fd_gradients(image) -> GradientImage:
    """Derivative planes from central differences of a plain image (spline.py:274-288)."""
    t = image if torch.is_tensor(image) else torch.from_numpy(np.asarray(image, dtype=np.float64))
    t = t.to(device=torch.device("cuda", torch.cuda.current_device()) if not t.is_cuda else t.device,
             dtype=torch.float32).contiguous()
    if t.dim() != 3 or t.shape[2] != 3:
        raise DimensionError("fd_gradients expects an (H, W, 3) image")
    h, w = t.shape[:2]
    if h < 2 or w < 2:
        raise DimensionError("finite differences need at least 2x2 pixels")
    lib = _lib.load()
    planes = torch.empty((h, w, 4, 3), dtype=torch.float32, device=t.device)
    _lib.check(lib.splat_fd_gradients(_lib.ptr(t), w, h, _lib.ptr(planes), _lib.stream_ptr()))
    return GradientImage(planes=planes, alphas=torch.zeros((4, h, w), dtype=torch.float32, device=t.device),
                         contrib_count=torch.zeros((h, w), dtype=torch.int32, device=t.device))


def fd_gradients_backward(adj) -> torch.Tensor:
    """Fold adjoints of FD-estimated channels back onto the colour (spline.py:291-297)."""
    if isinstance(adj, SourceAdjoint):
        planes = adj.planes.contiguous()
    else:
        planes = torch.stack([torch.as_tensor(np.asarray(a)) if not torch.is_tensor(a) else a
                              for a in (adj.d_color, adj.d_dx, adj.d_dy, adj.d_dxdy)], dim=2)
        planes = planes.to(device=torch.device("cuda", torch.cuda.current_device()),
                           dtype=torch.float32).contiguous()
    h, w = planes.shape[:2]
    lib = _lib.load()
    out = torch.empty((h, w, 3), dtype=torch.float32, device=planes.device)
    scratch = torch.empty((h, w, 3), dtype=torch.float32, device=planes.device)
    _lib.check(lib.splat_fd_gradients_backward(_lib.ptr(planes), w, h, _lib.ptr(out), _lib.ptr(scratch),
                                               _lib.stream_ptr()))
    return out
