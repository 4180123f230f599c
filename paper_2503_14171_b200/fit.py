"""Upscale-aware training step — the config-5 path of the reference fit loop.

Mirrors splinesplat.fit's hot pieces: ``loss`` (fit.py:94-108, L1 + SSIM with
its analytic adjoint), ``AdamState`` / ``adam_step`` (fit.py:132-160) and
``DEFAULT_LEARNING_RATES`` (fit.py:25-31).  ``ViewTrainer`` runs one training
step of the loop body (fit.py:188-223) over a batch of camera views:

    render_forward(train) -> upscale_spline(out_size) -> loss
    -> upscale_backward -> render_backward (accumulated over views)
    -> all_reduce(SUM) of the flat gradient buffer over the process group
    -> adam_step on the float64 parameters

Each rank renders its own views; the only collective is the NCCL all-reduce of
the 11 N float32 gradients.  All arithmetic runs in
libsplat_b200.so; torch provides the buffers, streams and the collective.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import DimensionError, ParameterError
from .device import DeviceScene, to_device
from .distributed import allreduce_grads
from .raster_backward import GradBuffer, PixelAdjoint, render_backward
from .raster_forward import render_forward
from .spline import fd_gradients, fd_gradients_backward, upscale_backward, upscale_spline

UPSCALE_MODES = ("spline_analytic", "bicubic_fd")   # fit.py:23 (minus "none": no upscaling)

DEFAULT_LEARNING_RATES = {       # fit.py:25-31
    "means": 2e-3,               # in normalized image units; scaled by max(W, H)
    "log_scales": 5e-3,
    "rotations": 1e-3,
    "opacity_logits": 5e-2,
    "colors": 2.5e-2,
}
PARAM_GROUPS = tuple(DEFAULT_LEARNING_RATES)
SSIM_WINDOW = 11

_loss_ws: dict = {}


def _tensor(a, device=None):
    dev = device or torch.device("cuda", torch.cuda.current_device())
    t = a if torch.is_tensor(a) else torch.from_numpy(np.asarray(a))
    return t.to(device=dev, dtype=torch.float32).contiguous()


def loss_device(pred: torch.Tensor, target: torch.Tensor, ssim_weight: float,
                adj: torch.Tensor | None = None, value: torch.Tensor | None = None):
    """Loss on the device without a host sync: returns (value (2,) float64 [loss, ssim], adjoint)."""
    if tuple(pred.shape) != tuple(target.shape):
        raise DimensionError("prediction and target dimensions differ")
    h, w = int(pred.shape[0]), int(pred.shape[1])
    lib = _lib.load()
    key = (w, h, str(pred.device))
    ws = _loss_ws.get(key)
    if ws is None:
        ws = torch.empty(lib.splat_loss_workspace_bytes(w, h), dtype=torch.uint8, device=pred.device)
        _loss_ws[key] = ws
    if adj is None:
        adj = torch.empty_like(pred)
    if value is None:
        value = torch.empty(2, dtype=torch.float64, device=pred.device)
    _lib.check(lib.splat_loss(_lib.ptr(pred), _lib.ptr(target), w, h, float(ssim_weight), _lib.ptr(adj),
                              _lib.ptr(value), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()))
    return value, adj


def loss(pred, target, ssim_weight: float):
    """(1 - lambda) L1 + lambda (1 - SSIM) and its adjoint (fit.py:94-108)."""
    p, t = _tensor(pred), _tensor(target)
    value, adj = loss_device(p, t, ssim_weight)
    return float(value[0].item()), adj


@dataclass
class AdamState:
    """fit.py:132-141: per-group first/second moments (float64) and the step count."""

    m: dict
    v: dict
    t: int = 0

    @classmethod
    def like(cls, params: dict) -> "AdamState":
        return cls(m={k: torch.zeros_like(v) for k, v in params.items()},
                   v={k: torch.zeros_like(v) for k, v in params.items()})


def adam_step(params: dict, grads: dict, state: AdamState, lrs: dict, beta1: float = 0.9,
              beta2: float = 0.999, eps: float = 1e-8):
    """Bias-corrected Adam over named groups, in place on the float64 device params (fit.py:144-160)."""
    lib = _lib.load()
    state.t += 1
    bc1 = 1.0 - beta1 ** state.t
    bc2 = 1.0 - beta2 ** state.t
    st = _lib.stream_ptr()
    for k, p in params.items():
        g = grads[k]
        if tuple(g.shape) != tuple(p.shape):
            raise DimensionError(f"gradient shape mismatch for group {k}")
        g = g.to(dtype=torch.float32).contiguous()
        _lib.check(lib.splat_adam_step(_lib.ptr(p), _lib.ptr(g), _lib.ptr(state.m[k]), _lib.ptr(state.v[k]),
                                       p.numel(), float(lrs[k]), beta1, beta2, bc1, bc2, eps, st))
    return params, state


def scene_params(ds: DeviceScene) -> dict:
    return {"means": ds.means, "log_scales": ds.log_scales, "rotations": ds.rotations,
            "opacity_logits": ds.opacity_logits, "colors": ds.colors}


def grads_dict(gb: GradBuffer) -> dict:
    g = gb.grads()
    return {"means": g.d_means, "log_scales": g.d_log_scales, "rotations": g.d_rotations,
            "opacity_logits": g.d_opacity_logits, "colors": g.d_colors}


@dataclass
class ViewTrainer:
    """One upscale-aware training step over a batch of views (config 5).

    ``targets[i]`` is the (H, W, 3) float32 device image for ``views[i]``;
    renders are ``render_size`` and are upscaled to ``out_size`` = (W, H).
    With ``group`` (a torch.distributed process group) the accumulated
    gradient buffer is all-reduced (SUM) before the Adam update, so every
    rank applies the identical update to its replica of the parameters.
    """

    scene: object
    render_size: tuple
    out_size: tuple
    views: list
    targets: list
    ssim_weight: float = 0.2
    upscale_mode: str = "spline_analytic"
    lrs: dict = field(default_factory=lambda: dict(DEFAULT_LEARNING_RATES))
    group: object = None

    def __post_init__(self):
        self.ds = to_device(self.scene)
        if self.upscale_mode not in UPSCALE_MODES:
            raise ParameterError(f"upscale_mode must be one of {UPSCALE_MODES}")
        if len(self.targets) != len(self.views):
            raise ParameterError("one target per view")
        w, h = self.out_size
        self.lrs = dict(self.lrs)
        self.lrs["means"] = self.lrs["means"] * max(w, h)          # fit.py:184
        self.grads = GradBuffer(self.ds.n, self.ds.device)
        self.state = AdamState.like(scene_params(self.ds))
        self.values = torch.zeros((max(len(self.views), 1), 2), dtype=torch.float64, device=self.ds.device)
        self._adj = torch.empty((h, w, 3), dtype=torch.float32, device=self.ds.device)
        self._calibrate()

    def _calibrate(self):
        """Size the pair buffers once (host-synchronous), with headroom for the
        scene to evolve; steps then run without any host synchronisation and
        overflow is caught by :meth:`check` (counters[1] of every frame)."""
        from .raster_forward import _capacity_hint, _initial_capacity
        rw, rh = self.render_size
        need = 0
        for v in self.views:
            img = render_forward(self.ds, rw, rh, view=v, train=True)
            need = max(need, img.stats.get("pairs", 0))
        key = (self.ds.n, rw, rh)
        _capacity_hint[key] = max(_initial_capacity(self.ds.n, rw, rh), int(need * 1.5) + 4096)
        self._frames = []

    def check(self) -> None:
        """Synchronise and raise if any frame of the last step overflowed its pair buffer."""
        for f in self._frames:
            if int(f.counters()[1].item()):
                self._calibrate()
                raise RuntimeError("pair capacity exceeded during the training step; buffers were "
                                   "re-sized, repeat the step")

    def step(self) -> torch.Tensor:
        """One step; returns the per-view [loss, ssim] rows (device, no host sync)."""
        ds, (rw, rh), (w, h) = self.ds, self.render_size, self.out_size
        self.grads.zero_()
        self._frames = []
        for i, (v, tgt) in enumerate(zip(self.views, self.targets)):
            fwd = render_forward(ds, rw, rh, view=v, train=True, sync_check=False)
            self._frames.append(fwd.frame)
            # fit.py:192-212: the analytic channels, or classical bicubic from FD planes
            src = fwd if self.upscale_mode == "spline_analytic" else fd_gradients(fwd.color)
            pred = upscale_spline(src, 1.0, out_size=(w, h))
            loss_device(pred, tgt, self.ssim_weight, adj=self._adj, value=self.values[i])
            sadj = upscale_backward(src, 1.0, self._adj, out_size=(w, h))
            if self.upscale_mode == "spline_analytic":
                adj = PixelAdjoint.from_source(sadj)
            else:
                adj = PixelAdjoint.zeros(rw, rh, ds.device)
                adj.planes[:, :, 0, :] = fd_gradients_backward(sadj)
            render_backward(ds, fwd, adj, out=self.grads, accumulate=True, check_finite=False)
        allreduce_grads(self.grads.flat, self.group)
        adam_step(scene_params(ds), grads_dict(self.grads), self.state, self.lrs)
        ds.refresh()   # view-independent terms for the updated parameters (depth order is fixed)
        return self.values
