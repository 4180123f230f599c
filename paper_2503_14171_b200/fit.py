"""Upscale-aware training step — the config-5 path of the reference fit loop.

Mirrors splinesplat.fit's hot pieces: ``loss`` (fit.py:94-108, L1 + SSIM with
its analytic adjoint), ``AdamState`` / ``adam_step`` (fit.py:132-160) and
``DEFAULT_LEARNING_RATES`` (fit.py:25-31).  ``ViewTrainer`` runs one training
step of the loop body (fit.py:188-223) over a batch of camera views:

    render_forward(train) -> upscale_spline(out_size) -> loss
    -> upscale_backward -> rasterizer backward to rank-order render-space
       terms (accumulated over views, two views in flight)
    -> all_reduce(SUM) of the terms over the process group
    -> parametrisation chain (once) -> adam_step on the float64 parameters

Each rank renders its own views; the only collective is the NCCL all-reduce of
the 9 N float32 terms.  All arithmetic runs in
libsplat_b200.so; torch provides the buffers, streams and the collective.
"""

from __future__ import annotations

import ctypes

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import DimensionError, ParameterError, Scene, logit
from .device import DeviceScene, to_device
from .distributed import allreduce_grads
from .raster_backward import GradBuffer, PixelAdjoint, chain_grads, render_backward, render_backward_rank
from .raster_forward import render_forward
from .spline import fd_gradients, fd_gradients_backward, upscale_backward, upscale_spline

UPSCALE_MODES = ("spline_analytic", "bicubic_fd")   # ViewTrainer (fit.py:23 minus "none")
FIT_UPSCALE_MODES = ("spline_analytic", "bicubic_fd", "none")   # fit.py:23

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
                adj: torch.Tensor | None = None, value: torch.Tensor | None = None, slot: int = 0):
    """Loss on the device without a host sync: returns (value (2,) float64 [loss, ssim], adjoint).
    ``slot`` selects a private workspace (one per concurrently used stream)."""
    if tuple(pred.shape) != tuple(target.shape):
        raise DimensionError("prediction and target dimensions differ")
    h, w = int(pred.shape[0]), int(pred.shape[1])
    lib = _lib.load()
    key = (w, h, str(pred.device), slot)
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
    keys = list(params)
    gs = []
    for k in keys:
        g = grads[k]
        if tuple(g.shape) != tuple(params[k].shape):
            raise DimensionError(f"gradient shape mismatch for group {k}")
        gs.append(g.to(dtype=torch.float32).contiguous())
    # every group in one launch (splat_adam_step_groups); the per-group entry point is the same arithmetic
    for i in range(0, len(keys), 8):
        ks = keys[i:i + 8]
        ng = len(ks)
        arr = lambda xs: (ctypes.c_void_p * ng)(*[_lib.ptr(x) for x in xs])
        _lib.check(lib.splat_adam_step_groups(
            ng, arr([params[k] for k in ks]), arr(gs[i:i + ng]), arr([state.m[k] for k in ks]),
            arr([state.v[k] for k in ks]), (ctypes.c_int64 * ng)(*[params[k].numel() for k in ks]),
            (ctypes.c_double * ng)(*[float(lrs[k]) for k in ks]), beta1, beta2, bc1, bc2, eps, st))
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
    streams: int = 2   # views in flight at once (the rasterizer backward of one view has
                       # only W/16 x H/16 tile CTAs; a second view fills the idle SMs)

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
        self.streams = max(1, min(int(self.streams), max(len(self.views), 1)))
        self._streams = [torch.cuda.Stream(device=self.ds.device) for _ in range(self.streams)]
        # per stream: render-space gradient terms in rank order, summed over that stream's views
        self._slot_rank = [torch.empty((max(self.ds.n, 1), 9), dtype=torch.float32, device=self.ds.device)
                           for _ in range(self.streams)]
        self._adjs = [torch.empty((h, w, 3), dtype=torch.float32, device=self.ds.device)
                      for _ in range(self.streams)]
        self._calibrate()
        self._copy_stream = None
        self._staged = None      # (targets, event) uploaded ahead of the next step

    def prefetch_targets(self, host_targets) -> None:
        """Upload the next step's targets (pinned host tensors) on a copy stream,
        into a second buffer set, so the PCIe transfer overlaps the current step.
        The next :meth:`step` waits for the copies and swaps the buffers in."""
        dev = self.ds.device
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(device=dev)
            self._spare = [torch.empty_like(t) for t in self.targets]
            self._spare_free = torch.cuda.Event()
            self._spare_free.record(torch.cuda.current_stream(dev))
        cs = self._copy_stream
        cs.wait_event(self._spare_free)          # the step that last read these buffers is done
        with torch.cuda.stream(cs):
            for dst, src in zip(self._spare, host_targets):
                dst.copy_(src, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(cs)
        self._staged = (self._spare, ev)

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
        cap = max(_initial_capacity(self.ds.n, rw, rh), int(need * 1.5) + 4096)
        _capacity_hint[key] = cap
        # per-stream steady-state buffers, reused by every view of that stream in every
        # step (stream order makes the reuse safe): the training image, its bin
        # workspace, the upscaled prediction, the source adjoint, the backward workspace
        from .raster_forward import Frame, GradientImage
        w, h = self.out_size
        dev, lib = self.ds.device, _lib.load()
        self._imgs = [GradientImage.empty(rw, rh, dev, train=True) for _ in range(self.streams)]
        self._frames = [Frame(self.ds.n, rw, rh, cap, dev) for _ in range(self.streams)]
        self._preds = [torch.empty((h, w, 3), dtype=torch.float32, device=dev) for _ in range(self.streams)]
        self._sadjs = [torch.empty((rh, rw, 4, 3), dtype=torch.float32, device=dev) for _ in range(self.streams)]
        nb = lib.splat_backward_workspace_bytes(self.ds.n, cap)
        self._bws = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(self.streams)]

    def check(self) -> None:
        """Synchronise and raise if any frame of the last step overflowed its pair buffer."""
        for f in self._frames:
            if int(f.counters()[1].item()):
                self._calibrate()
                raise RuntimeError("pair capacity exceeded during the training step; buffers were "
                                   "re-sized, repeat the step")

    def step(self) -> torch.Tensor:
        """One step; returns the per-view [loss, ssim] rows (device, no host sync).

        View i runs on stream i mod ``streams`` and accumulates into that stream's
        gradient buffer (views in order); the buffers are then folded into one in
        stream order, so the sum is deterministic for a fixed ``streams``."""
        ds, (rw, rh), (w, h) = self.ds, self.render_size, self.out_size
        main = torch.cuda.current_stream(ds.device)
        if self._staged is not None:            # targets prefetched by prefetch_targets()
            spare, ev = self._staged
            main.wait_event(ev)
            self._spare, self.targets = self.targets, spare
            self._staged = None
            # the old buffers were last read by the previous step, which precedes this point
            self._spare_free.record(main)
        for st in self._streams:
            st.wait_stream(main)
        for i, (v, tgt) in enumerate(zip(self.views, self.targets)):
            k = i % self.streams
            with torch.cuda.stream(self._streams[k]):
                adj_img = self._adjs[k]
                fwd = render_forward(ds, rw, rh, view=v, train=True, sync_check=False, out=self._imgs[k],
                                     frame=self._frames[k])
                # fit.py:192-212: the analytic channels, or classical bicubic from FD planes
                src = fwd if self.upscale_mode == "spline_analytic" else fd_gradients(fwd.color)
                pred = upscale_spline(src, 1.0, out_size=(w, h), out=self._preds[k])
                loss_device(pred, tgt, self.ssim_weight, adj=adj_img, value=self.values[i], slot=k)
                sadj = upscale_backward(src, 1.0, adj_img, out_size=(w, h), out=self._sadjs[k])
                if self.upscale_mode == "spline_analytic":
                    adj = PixelAdjoint.from_source(sadj)
                else:
                    adj = PixelAdjoint.zeros(rw, rh, ds.device)
                    adj.planes[:, :, 0, :] = fd_gradients_backward(sadj)
                render_backward_rank(ds, fwd, adj, self._slot_rank[k], accumulate=i >= self.streams,
                                     workspace=self._bws[k])
        for st in self._streams:
            main.wait_stream(st)
        lib = _lib.load()
        acc = self._slot_rank[0]
        for k in range(1, self.streams):   # fixed stream order: deterministic for a fixed `streams`
            _lib.check(lib.splat_grad_accumulate(_lib.ptr(acc), _lib.ptr(self._slot_rank[k]), acc.numel(),
                                                 _lib.stream_ptr(main)))
        allreduce_grads(acc, self.group)   # rank order is the same on every replica
        chain_grads(ds, acc, self.grads)   # the parametrisation chain once per step (it is linear)
        adam_step(scene_params(ds), grads_dict(self.grads), self.state, self.lrs)
        ds.refresh()   # view-independent terms for the updated parameters (depth order is fixed)
        return self.values


# ---- the single-image fit driver: fit.py:37-245 --------------------------

@dataclass
class FitConfig:
    """fit.py:37-61, same fields, defaults and validation."""

    iterations: int = 1000
    num_gaussians: int = 100
    render_scale: float = 1.0
    upscale_mode: str = "spline_analytic"
    learning_rates: dict = field(default_factory=lambda: dict(DEFAULT_LEARNING_RATES))
    ssim_weight: float = 0.2
    seed: int = 0
    log_every: int = 50
    prune_interval: int = 0      # 0 disables opacity pruning
    prune_opacity: float = 0.005

    def __post_init__(self):
        if self.iterations <= 0:
            raise ParameterError("iterations must be positive")
        if self.num_gaussians <= 0:
            raise ParameterError("num_gaussians must be positive")
        if self.render_scale < 1.0:
            raise ParameterError("render_scale must be >= 1")
        if self.upscale_mode not in FIT_UPSCALE_MODES:
            raise ParameterError(f"upscale_mode must be one of {FIT_UPSCALE_MODES}")
        if self.render_scale > 1.0 and self.upscale_mode == "none":
            raise ParameterError("render_scale > 1 requires an upscale mode")
        if not 0.0 <= self.ssim_weight <= 1.0:
            raise ParameterError("ssim_weight must be in [0, 1]")


@dataclass
class FitRow:
    """fit.py:64-74."""

    iteration: int
    loss: float
    psnr: float
    ssim: float
    t_forward_ms: float
    t_upscale_ms: float
    t_backward_ms: float
    t_opt_ms: float
    t_total_ms: float = 0.0


CSV_COLUMNS = ("iter", "loss", "psnr", "ssim", "t_forward_ms", "t_upscale_ms",
               "t_backward_ms", "t_opt_ms")
PSNR_CAP_DB = 99.0   # baselines.py psnr cap


@dataclass
class FitReport:
    """fit.py:81-91: logged rows + the fitted scene (host, float64)."""

    rows: list
    scene: Scene

    def write_csv(self, stream):
        stream.write(",".join(CSV_COLUMNS) + "\n")
        for r in self.rows:
            stream.write(f"{r.iteration},{r.loss!r},{r.psnr!r},{r.ssim!r},"
                         f"{r.t_forward_ms!r},{r.t_upscale_ms!r},"
                         f"{r.t_backward_ms!r},{r.t_opt_ms!r}\n")


def init_scene(target, n: int, seed: int) -> Scene:
    """Random splats covering the image, coloured by the target underneath (fit.py:111-129).
    Host numpy with the reference's RNG calls, so the initial scene is bit-identical."""
    if n <= 0:
        raise ParameterError("need at least one splat")
    target = np.asarray(target.cpu().numpy() if torch.is_tensor(target) else target, dtype=np.float64)
    h, w = target.shape[:2]
    rng = np.random.default_rng(seed)
    means = np.stack([rng.uniform(0, w, n), rng.uniform(0, h, n)], axis=1)
    s = np.sqrt(w * h / (np.pi * n))
    log_scales = np.full((n, 2), np.log(s))
    px = np.clip(means[:, 0].astype(np.int64), 0, w - 1)
    py = np.clip(means[:, 1].astype(np.int64), 0, h - 1)
    colors = target[py, px].copy()
    depths = rng.uniform(0.0, 1.0, n)
    return Scene(means=means, log_scales=log_scales, rotations=np.zeros(n),
                 opacity_logits=np.full(n, logit(0.5)), colors=colors, depths=depths,
                 background=np.zeros(3), reference_resolution=(w, h))


def _psnr(pred: torch.Tensor, target: torch.Tensor) -> float:
    mse = float(((pred.double() - target.double()) ** 2).mean().item())
    if mse == 0.0:
        return PSNR_CAP_DB
    return float(min(10.0 * np.log10(1.0 / mse), PSNR_CAP_DB))


def _prune(ds: DeviceScene, state: AdamState, keep: torch.Tensor):
    """Drop splats (fit.py:227-236): same depth keys, so the surviving order is unchanged."""
    fields = {f: getattr(ds, f)[keep].contiguous()
              for f in ("means", "log_scales", "rotations", "opacity_logits", "colors", "depths")}
    nd = DeviceScene(**fields, background=ds.background, reference_resolution=ds.reference_resolution).prepare()
    ns = AdamState(m={k: v[keep].contiguous() for k, v in state.m.items()},
                   v={k: v[keep].contiguous() for k, v in state.v.items()}, t=state.t)
    return nd, ns


def fit(target, cfg: FitConfig, *, threads: int = 1) -> FitReport:
    """Optimise a fresh scene against ``target`` (fit.py:163-245), every step on the GPU:
    render (training state) -> spline / FD upscale or clip -> L1+SSIM and adjoint ->
    upscale backward -> rasterizer backward -> Adam (float64 params) -> optional pruning.
    Rows are logged every ``log_every`` iterations (the only host synchronisations)."""
    del threads
    tgt_host = np.asarray(target.cpu().numpy() if torch.is_tensor(target) else target, dtype=np.float64)
    if tgt_host.size == 0:
        raise DimensionError("target image is empty")
    h, w = tgt_host.shape[:2]
    ssim_ok = h >= SSIM_WINDOW and w >= SSIM_WINDOW
    if cfg.ssim_weight > 0.0 and not ssim_ok:
        raise DimensionError("target too small for the SSIM window; set ssim_weight=0")
    low_w = max(1, int(np.floor(w / cfg.render_scale + 0.5)))
    low_h = max(1, int(np.floor(h / cfg.render_scale + 0.5)))
    upscaling = cfg.upscale_mode != "none" and (low_w, low_h) != (w, h)

    scene = init_scene(tgt_host, cfg.num_gaussians, cfg.seed)
    ds = DeviceScene.from_host(scene)
    tgt = _tensor(tgt_host, ds.device)
    lrs = dict(cfg.learning_rates)
    lrs["means"] = lrs["means"] * max(w, h)
    state = AdamState.like(scene_params(ds))
    value = torch.zeros(2, dtype=torch.float64, device=ds.device)
    metric = torch.zeros(2, dtype=torch.float64, device=ds.device)
    adj_img = torch.empty((h, w, 3), dtype=torch.float32, device=ds.device)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    rows = []
    for it in range(cfg.iterations):
        ev[0].record()
        fwd = render_forward(ds, low_w, low_h, train=True)
        ev[1].record()
        if upscaling:
            src = fwd if cfg.upscale_mode == "spline_analytic" else fd_gradients(fwd.color)
            pred = upscale_spline(src, cfg.render_scale, out_size=(w, h))
        else:
            src = fwd
            pred = upscale_spline(fwd, 1.0)   # factor 1 = clip(colour), fit.py:200
        ev[2].record()
        loss_device(pred, tgt, cfg.ssim_weight, adj=adj_img, value=value)
        if upscaling:
            sadj = upscale_backward(src, cfg.render_scale, adj_img, out_size=(w, h))
            if cfg.upscale_mode == "bicubic_fd":
                adj = PixelAdjoint.zeros(low_w, low_h, ds.device)
                adj.planes[:, :, 0, :] = fd_gradients_backward(sadj)
            else:
                adj = PixelAdjoint.from_source(sadj)
        else:
            adj = PixelAdjoint.zeros(low_w, low_h, ds.device)
            adj.planes[:, :, 0, :] = adj_img
        gb = GradBuffer(ds.n, ds.device)
        render_backward(ds, fwd, adj, out=gb, check_finite=False)
        ev[3].record()
        adam_step(scene_params(ds), grads_dict(gb), state, lrs)
        ds.refresh()
        if (cfg.prune_interval > 0 and (it + 1) % cfg.prune_interval == 0 and it + 1 < cfg.iterations):
            keep = 1.0 / (1.0 + torch.exp(-ds.opacity_logits)) >= cfg.prune_opacity
            nkeep = int(keep.sum().item())
            if 0 < nkeep < ds.n:
                ds, state = _prune(ds, state, keep)
        ev[4].record()
        if it % cfg.log_every == 0 or it == cfg.iterations - 1:
            torch.cuda.synchronize()
            if ssim_ok:
                if cfg.ssim_weight > 0.0:
                    s = float(value[1].item())
                else:
                    loss_device(pred, tgt, 1.0, adj=torch.empty_like(pred), value=metric)
                    s = float(metric[1].item())
            else:
                s = float("nan")
            t = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
            rows.append(FitRow(iteration=it, loss=float(value[0].item()), psnr=_psnr(pred, tgt), ssim=s,
                               t_forward_ms=t[0], t_upscale_ms=t[1], t_backward_ms=t[2], t_opt_ms=t[3],
                               t_total_ms=ev[0].elapsed_time(ev[4])))
    if not np.isfinite(rows[-1].loss):
        raise ParameterError("fit diverged to a non-finite loss")
    host = {f: getattr(ds, f).cpu().numpy() for f in ("means", "log_scales", "rotations", "opacity_logits",
                                                      "colors", "depths")}
    return FitReport(rows=rows, scene=Scene(**host, background=np.asarray(ds.background),
                                            reference_resolution=tuple(ds.reference_resolution)))
