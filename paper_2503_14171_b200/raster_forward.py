"""Render with analytic image gradients — drop-in for splinesplat.raster_forward.

Same public surface as the reference module (raster_forward.py:27-187):
``GradientImage``, ``sort_by_depth``, ``RenderPack``, ``prepare_scene``,
``tile_grid``, ``bin_tiles`` and ``render_forward(scene, out_width,
out_height, *, tiled=True, threads=1)``.  Arrays are float32 CUDA tensors (HWC)
instead of float64 numpy; ``tiled``/``threads`` are accepted and ignored (the
reference guarantees they never change the output).  Extra keywords: ``view``
(a ``scenes.View`` camera) and ``train`` (keep the float64 terminal state the
backward pass inverts from).

All work runs in libsplat_b200.so (sm_100a): preprocess -> tile binning
(per-block histograms, column scan, staged stable fill) -> tile rasterizer ->
exact float64 re-render of the few pixels whose termination was too close to
call.  ``render_at_points`` (raster_forward.py:190-233) evaluates the blend at
arbitrary positions in float64 for finite-difference checks.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import ALPHA_CLAMP, ALPHA_CULL, EARLY_TERMINATION, TILE, DimensionError, Scene  # noqa: F401
from .device import DeviceScene, to_device

__all__ = ["GradientImage", "RenderPack", "TileBins", "Frame", "sort_by_depth", "prepare_scene",
           "tile_grid", "bin_tiles", "render_forward", "render_at_points", "make_view"]

PLANES = ("color", "d_dx", "d_dy", "d_dxdy")
BIN_OFFSETS, BIN_KEYS, BIN_ATOMIC, BIN_COUNT_ONLY = 1, 2, 4, 8   # splat_bin_tiles flags (include/splat_b200.h)
ALPHAS = ("alpha", "alpha_dx", "alpha_dy", "alpha_dxdy")


@dataclass
class GradientImage:
    """Rendered colour plus analytic spatial gradients and alpha state.

    Field names and shapes follow raster_forward.py:27-40; the colour and
    derivative fields are views into one packed (H, W, 4, 3) float32 buffer
    (the upscaler's input layout), the alpha fields views of a (4, H, W) buffer.
    """

    planes: torch.Tensor                 # (H, W, 4, 3)
    alphas: torch.Tensor                 # (4, H, W)
    contrib_count: torch.Tensor          # (H, W) int32
    last: torch.Tensor | None = None     # (H, W) int32: tile-list end of the last contributor
    state: torch.Tensor | None = None    # (H, W, 4) float64 terminal (T, A_x, A_y, A_xy)
    frame: "Frame | None" = None         # bins of the render (kept for the backward pass)
    scene: DeviceScene | None = None
    view: "_lib.ViewT | None" = None
    stats: dict = field(default_factory=dict)

    color = property(lambda s: s.planes[:, :, 0, :])
    d_dx = property(lambda s: s.planes[:, :, 1, :])
    d_dy = property(lambda s: s.planes[:, :, 2, :])
    d_dxdy = property(lambda s: s.planes[:, :, 3, :])
    alpha = property(lambda s: s.alphas[0])
    alpha_dx = property(lambda s: s.alphas[1])
    alpha_dy = property(lambda s: s.alphas[2])
    alpha_dxdy = property(lambda s: s.alphas[3])

    @property
    def width(self) -> int:
        return self.planes.shape[1]

    @property
    def height(self) -> int:
        return self.planes.shape[0]

    @classmethod
    def empty(cls, width: int, height: int, device=None, train: bool = False) -> "GradientImage":
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        return cls(planes=torch.empty((height, width, 4, 3), dtype=torch.float32, device=dev),
                   alphas=torch.empty((4, height, width), dtype=torch.float32, device=dev),
                   contrib_count=torch.empty((height, width), dtype=torch.int32, device=dev),
                   last=torch.empty((height, width), dtype=torch.int32, device=dev),
                   state=(torch.empty((height, width, 4), dtype=torch.float64, device=dev)
                          if train else None))

    @classmethod
    def zeros(cls, width: int, height: int, device=None) -> "GradientImage":
        img = cls.empty(width, height, device)
        img.planes.zero_()
        img.alphas.zero_()
        img.contrib_count.zero_()
        img.last.zero_()
        return img

    @classmethod
    def from_planes(cls, color, d_dx, d_dy, d_dxdy, device=None) -> "GradientImage":
        """Pack user-provided (H, W, 3) planes (numpy or torch) into a GradientImage."""
        def t(a):
            if not torch.is_tensor(a):
                a = np.asarray(a)
                a = torch.as_tensor(a if a.flags.writeable else a.copy())
            return a.to(device=device or torch.device("cuda", torch.cuda.current_device()),
                        dtype=torch.float32)
        planes = torch.stack([t(color), t(d_dx), t(d_dy), t(d_dxdy)], dim=2).contiguous()
        h, w = planes.shape[:2]
        img = cls(planes=planes, alphas=torch.zeros((4, h, w), dtype=torch.float32, device=planes.device),
                  contrib_count=torch.zeros((h, w), dtype=torch.int32, device=planes.device))
        return img

    def c_gimg(self) -> _lib.GimgT:
        g = _lib.GimgT()
        g.planes = _lib.ptr(self.planes)
        g.alpha = _lib.ptr(self.alphas)
        g.count = _lib.ptr(self.contrib_count)
        g.last = _lib.ptr(self.last)
        g.state = _lib.ptr(self.state)
        return g

    def numpy(self) -> dict:
        """Host float64 copies of the reference fields (for comparisons)."""
        out = {f: getattr(self, f).double().cpu().numpy() for f in PLANES + ALPHAS}
        out["contrib_count"] = self.contrib_count.cpu().numpy()
        return out


def make_view(scene: DeviceScene, out_w: int, out_h: int, view=None) -> _lib.ViewT:
    """The C view struct: kx = out_w / ref_w exactly as prepare_scene (raster_forward.py:81-85)."""
    v = _lib.ViewT()
    ref_w, ref_h = scene.reference_resolution
    if view is not None:
        ref_w, ref_h = view.reference_resolution(ref_w, ref_h)
        v.ox, v.oy = float(view.ox), float(view.oy)
    else:
        v.ox = v.oy = 0.0
    v.kx = out_w / ref_w
    v.ky = out_h / ref_h
    for i in range(3):
        v.bg[i] = float(scene.background[i])
    return v


class Frame:
    """Workspace of one render: pack, bboxes, pairs, sorted bins, tile ranges."""

    GUARD_BYTE = 0xA5

    def __init__(self, n: int, width: int, height: int, capacity: int, device, guard: int = 0):
        lib = _lib.load()
        self.n, self.width, self.height, self.capacity = n, width, height, int(capacity)
        self.nbytes = lib.splat_frame_workspace_bytes(n, width, height, self.capacity)
        self.guard = int(guard) // 256 * 256
        if self.guard:   # test aid: canary bytes either side of the workspace (see guards_intact)
            self._buf = torch.full((self.nbytes + 2 * self.guard,), self.GUARD_BYTE, dtype=torch.uint8,
                                   device=device)
            self.ws = self._buf[self.guard:self.guard + self.nbytes]
        else:
            self.ws = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        self.ptrs = _lib.FramePtrsT()
        _lib.check(lib.splat_frame_pointers(_lib.ptr(self.ws), n, width, height, self.capacity,
                                            self.ptrs))
        self.counters().zero_()

    def guards_intact(self) -> bool:
        """True when no kernel wrote into the canary bytes around the workspace."""
        if not self.guard:
            return True
        g = self.guard
        return bool((self._buf[:g] == self.GUARD_BYTE).all()) and bool((self._buf[g + self.nbytes:] == self.GUARD_BYTE).all())

    def _view(self, ptr, count, dtype, shape):
        off = ptr - self.ws.data_ptr()
        size = torch.empty((), dtype=dtype).element_size()
        return self.ws[off:off + count * size].view(dtype).view(shape)

    @property
    def ntiles(self) -> int:
        return ((self.width + TILE - 1) // TILE) * ((self.height + TILE - 1) // TILE)

    def counters(self) -> torch.Tensor:
        return self._view(self.ptrs.counters, 32, torch.int32, (32,))

    def bboxes(self) -> torch.Tensor:
        return self._view(self.ptrs.bboxes, 4 * max(self.n, 1), torch.int16, (max(self.n, 1), 4))[:self.n]

    def touched(self) -> torch.Tensor:
        return self._view(self.ptrs.touched, max(self.n, 1), torch.int32, (max(self.n, 1),))[:self.n]

    def pairs(self, count: int):
        k = self._view(self.ptrs.keys, max(self.capacity, 1), torch.int32, (max(self.capacity, 1),))
        r = self._view(self.ptrs.ranks, max(self.capacity, 1), torch.int32, (max(self.capacity, 1),))
        return k[:count], r[:count]

    def ranges(self) -> torch.Tensor:
        return self._view(self.ptrs.ranges, 2 * self.ntiles, torch.int32, (self.ntiles, 2))

    def fixup_list(self, count: int) -> torch.Tensor:
        return self._view(self.ptrs.fixup, self.width * self.height, torch.int32,
                          (self.width * self.height,))[:count]


_capacity_hint: dict = {}


def _initial_capacity(n: int, width: int, height: int) -> int:
    ntiles = ((width + TILE - 1) // TILE) * ((height + TILE - 1) // TILE)
    return _capacity_hint.get((n, width, height), max(4 * n, 4 * ntiles, 1 << 16))


def sort_by_depth(scene) -> torch.Tensor:
    """Indices ordering splats front to back; ties keep list order (raster_forward.py:59-61).

    Computed by the device radix sort of ``splat_scene_prepare``.
    """
    return to_device(scene).order()


@dataclass
class RenderPack:
    """Depth-sorted render-resolution splat parameters (raster_forward.py:64-76), on the GPU."""

    order: torch.Tensor     # (N,) int64
    means: torch.Tensor     # (N, 2) float64
    conics: torch.Tensor    # (N, 3) float64
    sigmas: torch.Tensor    # (N,) float64
    colors: torch.Tensor    # (N, 3) float64
    bboxes: torch.Tensor    # (N, 4) int64 x0, x1, y0, y1
    valid: torch.Tensor     # (N,) bool
    kx: float
    ky: float
    frame: Frame | None = None


def prepare_scene(scene, out_w: int, out_h: int, *, view=None) -> RenderPack:
    """raster_forward.py:79-123 on the device (bit-identical bboxes / validity)."""
    lib = _lib.load()
    ds = to_device(scene)
    v = make_view(ds, out_w, out_h, view)
    frame = Frame(ds.n, out_w, out_h, _initial_capacity(ds.n, out_w, out_h), ds.device)
    st = _lib.stream_ptr()
    _lib.check(lib.splat_prepare_view(_lib.ptr(ds.const), ds.n, v, out_w, out_h, _lib.ptr(frame.ws),
                                      frame.nbytes, frame.capacity, st))
    pack64 = torch.empty((max(ds.n, 1), 6), dtype=torch.float64, device=ds.device)
    _lib.check(lib.splat_view_pack64(_lib.ptr(ds.const), ds.n, v, _lib.ptr(pack64), st))
    pack64 = pack64[:ds.n]
    order = ds.order()
    return RenderPack(order=order, means=pack64[:, 0:2].contiguous(), conics=pack64[:, 2:5].contiguous(),
                      sigmas=pack64[:, 5].contiguous(), colors=ds.colors[order],
                      bboxes=frame.bboxes().to(torch.int64), valid=frame.touched() > 0,
                      kx=v.kx, ky=v.ky, frame=frame)


def tile_grid(out_w: int, out_h: int):
    """Half-open pixel ranges of the 16x16 tiles, row-major (raster_forward.py:126-133)."""
    return [(tx0, min(tx0 + TILE, out_w), ty0, min(ty0 + TILE, out_h))
            for ty0 in range(0, out_h, TILE) for tx0 in range(0, out_w, TILE)]


@dataclass
class TileBins:
    """Per-tile candidate lists as CSR: ranks[offsets[t]:offsets[t+1]] ascending."""

    offsets: torch.Tensor   # (ntiles + 1,) int64
    ranks: torch.Tensor     # (pairs,) int64
    keys: torch.Tensor      # (pairs,) int64 tile id per pair

    def __len__(self):
        return self.offsets.numel() - 1

    def __getitem__(self, t):
        return self.ranks[int(self.offsets[t]):int(self.offsets[t + 1])]


def _grow_and_bin(pack: RenderPack, out_w: int, out_h: int, lib, st, flags: int = 0):
    frame = pack.frame
    _lib.check(lib.splat_bin_tiles(frame.n, out_w, out_h, _lib.ptr(frame.ws), frame.nbytes,
                                   frame.capacity, BIN_OFFSETS | BIN_KEYS | flags, st))
    cnt = frame.counters()[:2].cpu()
    return int(cnt[0]), bool(cnt[1])


def bin_tiles(pack: RenderPack, out_w: int, out_h: int, *, _flags: int = 0):
    """(tiles, TileBins) — raster_forward.py:136-149 via per-block tile histograms,
    a column scan and a stable staged fill (``_flags=BIN_ATOMIC`` selects the
    large-grid path: per-pair atomics + per-tile sort)."""
    lib = _lib.load()
    st = _lib.stream_ptr()
    total, overflow = _grow_and_bin(pack, out_w, out_h, lib, st, _flags)
    if overflow:
        raise RuntimeError("pair capacity exceeded in bin_tiles; re-run prepare_scene")
    frame = pack.frame
    keys, ranks = frame.pairs(total)
    ranges = frame.ranges().to(torch.int64)
    offsets = torch.zeros(frame.ntiles + 1, dtype=torch.int64, device=ranges.device)
    # offsets from the per-tile counts
    counts = ranges[:, 1] - ranges[:, 0]
    offsets[1:] = torch.cumsum(counts, 0)
    return tile_grid(out_w, out_h), TileBins(offsets, ranks.to(torch.int64), keys.to(torch.int64))


def render_forward(scene, out_width: int, out_height: int, *, tiled: bool = True, threads: int = 1,
                   view=None, train: bool = False, out: GradientImage | None = None,
                   sync_check: bool = True, frame: "Frame | None" = None) -> GradientImage:
    """Render with analytic gradients (raster_forward.py:152-187).

    ``out`` / ``frame`` reuse a caller's image and bin workspace (steady-state loops);
    a reused frame keeps its capacity, and an overflow stays flagged in its counters."""
    del tiled, threads  # output-invariant by the reference's contract
    if out_width <= 0 or out_height <= 0:
        raise DimensionError("output dimensions must be positive")
    lib = _lib.load()
    ds = to_device(scene)
    img = out if out is not None else GradientImage.empty(out_width, out_height, ds.device, train)
    if train and img.state is None:
        img.state = torch.empty((out_height, out_width, 4), dtype=torch.float64, device=ds.device)
    v = make_view(ds, out_width, out_height, view)
    img.scene, img.view = ds, v
    st = _lib.stream_ptr()
    if frame is not None and (frame.n, frame.width, frame.height) != (ds.n, out_width, out_height):
        raise DimensionError("frame workspace was sized for another scene or resolution")
    cap = frame.capacity if frame is not None else _initial_capacity(ds.n, out_width, out_height)
    while True:
        if frame is None or frame.capacity < cap:
            frame = Frame(ds.n, out_width, out_height, cap, ds.device)
        _lib.check(lib.splat_render_forward(_lib.ptr(ds.const), ds.n, v, out_width, out_height,
                                            int(train), img.c_gimg(), _lib.ptr(frame.ws), frame.nbytes,
                                            frame.capacity, st))
        if not sync_check:
            break
        c = frame.counters()[:4].cpu()
        if not int(c[1]):
            img.stats = {"pairs": int(c[0]), "fixup_pixels": int(c[2])}
            break
        cap = int(int(c[0]) * 1.25) + 1024
        _capacity_hint[(ds.n, out_width, out_height)] = cap
    img.frame = frame
    return img


def render_at_points(scene, xs, ys, out_width: int, out_height: int, *, with_state: bool = False, view=None):
    """Blended colour at arbitrary continuous positions (raster_forward.py:190-233),
    float64 on the device, for finite-difference checks of the gradient planes.
    Returns an (npts, 3) float64 tensor (and the (npts, 2n) bool blend signature)."""
    import ctypes
    lib = _lib.load()
    pack = prepare_scene(scene, out_width, out_height, view=view)
    dev = pack.means.device
    x = torch.as_tensor(np.atleast_1d(np.asarray(xs, np.float64)) if not torch.is_tensor(xs) else xs,
                        dtype=torch.float64).to(dev).contiguous().reshape(-1)
    y = torch.as_tensor(np.atleast_1d(np.asarray(ys, np.float64)) if not torch.is_tensor(ys) else ys,
                        dtype=torch.float64).to(dev).contiguous().reshape(-1)
    if x.numel() != y.numel():
        raise DimensionError("xs and ys must have the same length")
    n, npts = int(pack.sigmas.numel()), x.numel()
    pack64 = torch.cat([pack.means, pack.conics, pack.sigmas[:, None]], 1).contiguous()
    cols = pack.colors.to(torch.float64).contiguous()
    valid = pack.valid.to(torch.uint8).contiguous()
    out = torch.empty((npts, 3), dtype=torch.float64, device=dev)
    state = torch.zeros((npts, 2 * n), dtype=torch.uint8, device=dev) if with_state else None
    ds = to_device(scene)
    bg = (ctypes.c_double * 3)(*ds.background)
    _lib.check(lib.splat_render_points(_lib.ptr(pack64), _lib.ptr(cols), _lib.ptr(valid), n, _lib.ptr(x),
                                       _lib.ptr(y), npts, bg, _lib.ptr(out), _lib.ptr(state), _lib.stream_ptr()))
    if with_state:
        return out, state.bool()
    return out
