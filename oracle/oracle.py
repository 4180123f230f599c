"""CPU ORACLE — test infrastructure only; never the product path.

A float64 numpy/C restatement of the reference's gradient-aware render +
spline-upscale path (splinesplat, /root/reference/pkg/src/splinesplat).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product package ``paper_2503_14171_b200`` does not
import it and fails loudly when its CUDA library is missing.

Parity pin: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors written by the reference itself (``tests/golden/make_golden.py``
imports the reference in the build container and runs it on seeded scenes).

Each function cites the reference file:line it restates.  The per-pixel loops
live in ``raster_oracle.c`` (built by ``oracle/Makefile`` into
``oracle/liboracle.so``; OpenMP over 16x16 tiles like the reference's
ThreadPoolExecutor, raster_forward.py:181-186).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

ALPHA_CLAMP = 0.999          # core.py:23
ALPHA_CULL = 1.0 / 255.0     # core.py:24
EARLY_TERMINATION = 1e-4     # core.py:25
LOG_CULL = float(np.log(ALPHA_CULL))  # _kernels.py:29
TILE = 16                    # raster_forward.py:24

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile raster_oracle.c (checker only)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "raster_oracle.c"))):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int
        L = ctypes.c_int64
        D = ctypes.c_double
        _lib.oracle_forward.argtypes = [I, I, P, P, P, P, P, P, P, P, D,
                                        P, P, P, P, P, P, P, P, P, I]
        _lib.oracle_forward.restype = None
        _lib.oracle_forward_region.argtypes = [I, I, I, I, I, P, L, P, P, P, P, P, P, D,
                                               P, P, P, P, P, P, P, P, P]
        _lib.oracle_forward_region.restype = None
        _lib.oracle_backward.argtypes = [I, I, P, P, P, P, P, P, P, P, D,
                                         P, P, P, P, P, P, P, P, P, P, L, I]
        _lib.oracle_backward.restype = None
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def default_threads() -> int:
    return int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))


# ---------------------------------------------------------------------------
# Scene and preprocessing
# ---------------------------------------------------------------------------

def logistic(x):
    """core.py:44-45."""
    return 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))


@dataclass
class OScene:
    """Plain SoA float64 scene (fields as reference core.py:75-93)."""

    means: np.ndarray
    log_scales: np.ndarray
    rotations: np.ndarray
    opacity_logits: np.ndarray
    colors: np.ndarray
    depths: np.ndarray
    background: np.ndarray
    reference_resolution: tuple

    @property
    def n(self) -> int:
        return len(self.depths)

    @classmethod
    def of(cls, s) -> "OScene":
        """Adopt any object with the reference Scene's field names."""
        return cls(np.asarray(s.means, np.float64).reshape(-1, 2),
                   np.asarray(s.log_scales, np.float64).reshape(-1, 2),
                   np.asarray(s.rotations, np.float64).reshape(-1),
                   np.asarray(s.opacity_logits, np.float64).reshape(-1),
                   np.asarray(s.colors, np.float64).reshape(-1, 3),
                   np.asarray(s.depths, np.float64).reshape(-1),
                   np.asarray(s.background, np.float64).reshape(3),
                   tuple(s.reference_resolution))


@dataclass
class OPack:
    order: np.ndarray
    means: np.ndarray
    conics: np.ndarray
    sigmas: np.ndarray
    colors: np.ndarray
    bboxes: np.ndarray
    valid: np.ndarray
    kx: float
    ky: float


def sort_by_depth(depths) -> np.ndarray:
    """Stable ascending argsort — raster_forward.py:59-61."""
    return np.argsort(np.asarray(depths), kind="stable")


def prepare_scene(scene: OScene, out_w: int, out_h: int) -> OPack:
    """Rescale, conic, cull-ellipse bbox — raster_forward.py:79-123.

    Same float64 expression trees as the reference so bboxes/valid are
    bit-identical (the integer outputs the GPU path must reproduce exactly).
    """
    ref_w, ref_h = scene.reference_resolution
    kx = out_w / ref_w
    ky = out_h / ref_h
    order = sort_by_depth(scene.depths)
    means = scene.means[order] * np.array([kx, ky])
    ls = scene.log_scales[order]
    rot = scene.rotations[order]
    sig = logistic(scene.opacity_logits[order])
    e1 = np.exp(-2.0 * ls[:, 0])
    e2 = np.exp(-2.0 * ls[:, 1])
    co = np.cos(rot)
    si = np.sin(rot)
    n00 = e1 * co * co + e2 * si * si
    n01 = (e1 - e2) * si * co
    n11 = e1 * si * si + e2 * co * co
    conics = np.empty((len(order), 3))
    conics[:, 0] = n00 / (2.0 * kx * kx)
    conics[:, 1] = n01 / (2.0 * kx * ky)
    conics[:, 2] = n11 / (2.0 * ky * ky)
    q = np.log(np.maximum(sig / ALPHA_CULL, 1.0))
    det = e1 * e2 / (4.0 * kx * kx * ky * ky)
    rx = np.sqrt(q * conics[:, 2] / det)
    ry = np.sqrt(q * conics[:, 0] / det)
    bb = np.empty((len(order), 4), dtype=np.int64)
    bb[:, 0] = np.clip(np.floor(means[:, 0] - rx).astype(np.int64) - 1, 0, out_w)
    bb[:, 1] = np.clip(np.ceil(means[:, 0] + rx).astype(np.int64) + 1, 0, out_w)
    bb[:, 2] = np.clip(np.floor(means[:, 1] - ry).astype(np.int64) - 1, 0, out_h)
    bb[:, 3] = np.clip(np.ceil(means[:, 1] + ry).astype(np.int64) + 1, 0, out_h)
    valid = (sig >= ALPHA_CULL) & (bb[:, 1] > bb[:, 0]) & (bb[:, 3] > bb[:, 2])
    return OPack(order, means, conics, sig, np.ascontiguousarray(scene.colors[order]),
                 bb, valid, kx, ky)


def tile_counts(out_w: int, out_h: int):
    """raster_forward.py:126-133 — row-major grid of 16x16 tiles."""
    return (out_w + TILE - 1) // TILE, (out_h + TILE - 1) // TILE


def bin_tiles_csr(pack: OPack, out_w: int, out_h: int):
    """Per-tile candidate lists as CSR (offsets, ranks) — raster_forward.py:136-149.

    Vectorised: every valid rank emits (tile, rank) for each tile its bbox
    touches; a stable sort by tile keeps ranks ascending within a tile, which
    is exactly the reference's append order.
    """
    ntx, nty = tile_counts(out_w, out_h)
    v = np.flatnonzero(pack.valid)
    bb = pack.bboxes[v]
    tx0 = bb[:, 0] // TILE
    tx1 = (bb[:, 1] - 1) // TILE
    ty0 = bb[:, 2] // TILE
    ty1 = (bb[:, 3] - 1) // TILE
    nx = tx1 - tx0 + 1
    ny = ty1 - ty0 + 1
    cnt = nx * ny
    total = int(cnt.sum())
    rank = np.repeat(v, cnt)
    start = np.repeat(np.cumsum(cnt) - cnt, cnt)
    local = np.arange(total) - start
    rnx = np.repeat(nx, cnt)
    tx = np.repeat(tx0, cnt) + local % rnx
    ty = np.repeat(ty0, cnt) + local // rnx
    tile = ty * ntx + tx
    perm = np.argsort(tile, kind="stable")
    ranks = rank[perm].astype(np.int64)
    counts = np.bincount(tile, minlength=ntx * nty)
    off = np.zeros(ntx * nty + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return off, ranks, tile[perm].astype(np.int64)


# ---------------------------------------------------------------------------
# Rasterizer
# ---------------------------------------------------------------------------

@dataclass
class OGradientImage:
    """raster_forward.py:27-56 field layout (HWC float64)."""

    color: np.ndarray
    d_dx: np.ndarray
    d_dy: np.ndarray
    d_dxdy: np.ndarray
    alpha: np.ndarray
    alpha_dx: np.ndarray
    alpha_dy: np.ndarray
    alpha_dxdy: np.ndarray
    contrib_count: np.ndarray

    @classmethod
    def zeros(cls, w: int, h: int) -> "OGradientImage":
        s3, s1 = (h, w, 3), (h, w)
        return cls(np.zeros(s3), np.zeros(s3), np.zeros(s3), np.zeros(s3),
                   np.zeros(s1), np.zeros(s1), np.zeros(s1), np.zeros(s1),
                   np.zeros(s1, dtype=np.int32))

    FIELDS = ("color", "d_dx", "d_dy", "d_dxdy", "alpha", "alpha_dx", "alpha_dy",
              "alpha_dxdy", "contrib_count")


def render_forward(scene, out_w: int, out_h: int, *, tiled: bool = True,
                   threads: int | None = None) -> OGradientImage:
    """raster_forward.py:152-187."""
    scene = OScene.of(scene)
    if out_w <= 0 or out_h <= 0:
        raise ValueError("output dimensions must be positive")
    img = OGradientImage.zeros(out_w, out_h)
    if scene.n == 0:
        img.color[:] = scene.background
        return img
    pack = prepare_scene(scene, out_w, out_h)
    lib = _load()
    args = [_ptr(pack.means), _ptr(pack.conics), _ptr(pack.sigmas), _ptr(pack.colors),
            _ptr(pack.bboxes), _ptr(scene.background), LOG_CULL,
            _ptr(img.color), _ptr(img.d_dx), _ptr(img.d_dy), _ptr(img.d_dxdy),
            _ptr(img.alpha), _ptr(img.alpha_dx), _ptr(img.alpha_dy), _ptr(img.alpha_dxdy),
            _ptr(img.contrib_count)]
    if not tiled:
        cand = np.flatnonzero(pack.valid).astype(np.int64)
        lib.oracle_forward_region(out_w, 0, out_w, 0, out_h, _ptr(cand), len(cand), *args)
        return img
    off, ranks, _ = bin_tiles_csr(pack, out_w, out_h)
    lib.oracle_forward(out_w, out_h, _ptr(off), _ptr(ranks), *args,
                       threads if threads else default_threads())
    return img


def render_backward_sorted(scene: OScene, pack: OPack, fwd: OGradientImage, adj,
                           threads: int | None = None) -> np.ndarray:
    """Render-space gradients in rank order, (N, 9) — raster_backward.py:87-124."""
    h, w = fwd.color.shape[:2]
    off, ranks, _ = bin_tiles_csr(pack, w, h)
    out9 = np.zeros((scene.n, 9))
    c = np.ascontiguousarray
    planes = [c(fwd.alpha, dtype=np.float64), c(fwd.alpha_dx, dtype=np.float64),
              c(fwd.alpha_dy, dtype=np.float64), c(fwd.alpha_dxdy, dtype=np.float64)]
    cnt = c(fwd.contrib_count, dtype=np.int32)
    aw = [c(a, dtype=np.float64) for a in adj]
    _load().oracle_backward(w, h, _ptr(off), _ptr(ranks), _ptr(pack.means), _ptr(pack.conics),
                            _ptr(pack.sigmas), _ptr(pack.colors), _ptr(pack.bboxes),
                            _ptr(scene.background), LOG_CULL,
                            *[_ptr(p) for p in planes], _ptr(cnt), *[_ptr(a) for a in aw],
                            _ptr(out9), scene.n, threads if threads else default_threads())
    return out9


def chain_to_params(scene: OScene, pack: OPack, g9: np.ndarray) -> dict:
    """Render-space -> stored parametrization — raster_backward.py:126-152."""
    order = pack.order
    ls = scene.log_scales[order]
    rot = scene.rotations[order]
    sig = pack.sigmas
    kx, ky = pack.kx, pack.ky
    dn00 = g9[:, 6] / (2.0 * kx * kx)
    dn01 = g9[:, 7] / (2.0 * kx * ky)
    dn11 = g9[:, 8] / (2.0 * ky * ky)
    e1 = np.exp(-2.0 * ls[:, 0])
    e2 = np.exp(-2.0 * ls[:, 1])
    co = np.cos(rot)
    si = np.sin(rot)
    d_l1 = -2.0 * e1 * (dn00 * co * co + dn01 * si * co + dn11 * si * si)
    d_l2 = -2.0 * e2 * (dn00 * si * si - dn01 * si * co + dn11 * co * co)
    sin2 = 2.0 * si * co
    cos2 = co * co - si * si
    d_rot = (e2 - e1) * sin2 * dn00 + (e1 - e2) * cos2 * dn01 + (e1 - e2) * sin2 * dn11
    n = scene.n
    out = {"d_means": np.zeros((n, 2)), "d_log_scales": np.zeros((n, 2)),
           "d_rotations": np.zeros(n), "d_opacity_logits": np.zeros(n),
           "d_colors": np.zeros((n, 3))}
    out["d_colors"][order] = g9[:, 0:3]
    out["d_opacity_logits"][order] = g9[:, 3] * sig * (1.0 - sig)
    out["d_means"][order, 0] = g9[:, 4] * kx
    out["d_means"][order, 1] = g9[:, 5] * ky
    out["d_log_scales"][order, 0] = d_l1
    out["d_log_scales"][order, 1] = d_l2
    out["d_rotations"][order] = d_rot
    return out


def render_backward(scene, fwd: OGradientImage, adj, threads: int | None = None) -> dict:
    """raster_backward.py:73-153; adj = (w, wx, wy, wxy) each (H, W, 3)."""
    scene = OScene.of(scene)
    n = scene.n
    if n == 0:
        return {"d_means": np.zeros((0, 2)), "d_log_scales": np.zeros((0, 2)),
                "d_rotations": np.zeros(0), "d_opacity_logits": np.zeros(0),
                "d_colors": np.zeros((0, 3))}
    h, w = fwd.color.shape[:2]
    pack = prepare_scene(scene, w, h)
    g9 = render_backward_sorted(scene, pack, fwd, adj, threads)
    return chain_to_params(scene, pack, g9)


# ---------------------------------------------------------------------------
# Spline upscaler
# ---------------------------------------------------------------------------

def output_size(in_w: int, in_h: int, factor: float):
    """spline.py:94-99."""
    if factor < 1.0:
        raise ValueError("upscale factor must be >= 1")
    return int(np.floor(in_w * factor + 0.5)), int(np.floor(in_h * factor + 0.5))


def axis_map(n_out: int, n_in: int):
    """Center-aligned mapping, spline.py:102-112."""
    scale = n_out / n_in
    s = (np.arange(n_out) + 0.5) / scale - 0.5
    i0 = np.floor(s).astype(np.int64)
    return i0, s - i0


def hermite_weights(t: np.ndarray) -> np.ndarray:
    """Rows [1, t, t^2, t^3] @ C^-1 (spline.py:21-32) in closed form:
    value at 0, value at 1, slope at 0, slope at 1."""
    t = np.asarray(t, dtype=np.float64)
    t2 = t * t
    t3 = t2 * t
    return np.stack([1.0 - 3.0 * t2 + 2.0 * t3, 3.0 * t2 - 2.0 * t3,
                     t - 2.0 * t2 + t3, t3 - t2], axis=-1)


def _corner_index(i0: np.ndarray, n: int):
    return np.clip(i0, 0, n - 1), np.clip(i0 + 1, 0, n - 1)


def upscale_spline(color, d_dx, d_dy, d_dxdy, factor: float, *, out_size=None,
                   clamp: bool = True) -> np.ndarray:
    """Bicubic Hermite upscale from value + analytic derivative planes.

    spline.py:115-178: F = C A C^T per unit subdomain, corners replicated at
    the border (np.pad edge), evaluated as sum_k sum_l hx_k hy_l F[k, l].
    """
    color = np.asarray(color, np.float64)
    in_h, in_w = color.shape[:2]
    if out_size is None:
        out_w, out_h = output_size(in_w, in_h, factor)
    else:
        out_w, out_h = out_size
        if out_w < in_w or out_h < in_h:
            raise ValueError("output must be at least source size")
    ix0, tx = axis_map(out_w, in_w)
    iy0, ty = axis_map(out_h, in_h)
    hx = hermite_weights(tx)   # (Wo, 4)
    hy = hermite_weights(ty)   # (Ho, 4)
    xa, xb = _corner_index(ix0, in_w)
    ya, yb = _corner_index(iy0, in_h)
    f = color
    fx = np.asarray(d_dx, np.float64)
    fy = np.asarray(d_dy, np.float64)
    fxy = np.asarray(d_dxdy, np.float64)
    # y pass: for each output row, combine the two source rows (values + y-slopes)
    def ypass(vplane, dplane):
        return (hy[:, 0, None, None] * vplane[ya] + hy[:, 1, None, None] * vplane[yb]
                + hy[:, 2, None, None] * dplane[ya] + hy[:, 3, None, None] * dplane[yb])
    gv = ypass(f, fy)      # (Ho, W, 3): value-in-x along each output row
    gd = ypass(fx, fxy)    # (Ho, W, 3): x-slope along each output row
    out = (hx[None, :, 0, None] * gv[:, xa] + hx[None, :, 1, None] * gv[:, xb]
           + hx[None, :, 2, None] * gd[:, xa] + hx[None, :, 3, None] * gd[:, xb])
    return np.clip(out, 0.0, 1.0) if clamp else out


def _axis_adjoint(g: np.ndarray, idx_a, idx_b, wts, n_in: int, axis: int):
    """Transpose of the two-corner combination along one axis: returns the
    (value, slope) source adjoints."""
    g = np.moveaxis(g, axis, 0)
    shape = (n_in,) + g.shape[1:]
    dv = np.zeros(shape)
    dd = np.zeros(shape)
    ex = (slice(None),) + (None,) * (g.ndim - 1)
    np.add.at(dv, idx_a, wts[:, 0][ex] * g)
    np.add.at(dv, idx_b, wts[:, 1][ex] * g)
    np.add.at(dd, idx_a, wts[:, 2][ex] * g)
    np.add.at(dd, idx_b, wts[:, 3][ex] * g)
    return np.moveaxis(dv, 0, axis), np.moveaxis(dd, 0, axis)


def upscale_backward(in_w: int, in_h: int, factor: float, adjoint: np.ndarray, *,
                     out_size=None):
    """Exact transpose of the linear upscale map (no clamp) — spline.py:191-243.

    Returns (d_color, d_dx, d_dy, d_dxdy), each (H, W, 3).
    """
    if out_size is None:
        out_w, out_h = output_size(in_w, in_h, factor)
    else:
        out_w, out_h = out_size
    adjoint = np.asarray(adjoint, np.float64)
    if adjoint.shape != (out_h, out_w, 3):
        raise ValueError("adjoint dimensions must match the upscaled output")
    ix0, tx = axis_map(out_w, in_w)
    iy0, ty = axis_map(out_h, in_h)
    xa, xb = _corner_index(ix0, in_w)
    ya, yb = _corner_index(iy0, in_h)
    gv, gd = _axis_adjoint(adjoint, xa, xb, hermite_weights(tx), in_w, axis=1)  # (Ho, W, 3)
    d_color, d_dy = _axis_adjoint(gv, ya, yb, hermite_weights(ty), in_h, axis=0)
    d_dx, d_dxdy = _axis_adjoint(gd, ya, yb, hermite_weights(ty), in_h, axis=0)
    return d_color, d_dx, d_dy, d_dxdy


def _diff_x(f):
    """Central differences along x, one-sided at borders — spline.py:246-253."""
    out = np.empty_like(f)
    out[:, 1:-1] = 0.5 * (f[:, 2:] - f[:, :-2])
    out[:, 0] = f[:, 1] - f[:, 0]
    out[:, -1] = f[:, -1] - f[:, -2]
    return out


def _diff_x_t(g):
    """Transpose of _diff_x — spline.py:256-264."""
    out = np.zeros_like(g)
    out[:, 2:] += 0.5 * g[:, 1:-1]
    out[:, :-2] -= 0.5 * g[:, 1:-1]
    out[:, 1] += g[:, 0]
    out[:, 0] -= g[:, 0]
    out[:, -1] += g[:, -1]
    out[:, -2] -= g[:, -1]
    return out


def fd_gradients(image):
    """spline.py:274-288: (color, d_dx, d_dy, d_dxdy) from finite differences."""
    image = np.asarray(image, np.float64)
    d_dx = _diff_x(image)
    d_dy = _diff_x(image.swapaxes(0, 1)).swapaxes(0, 1)
    d_dxdy = _diff_x(d_dy)
    return image.copy(), d_dx, d_dy, d_dxdy


def fd_gradients_backward(d_color, d_dx, d_dy, d_dxdy):
    """spline.py:291-297."""
    def ty(g):
        return _diff_x_t(g.swapaxes(0, 1)).swapaxes(0, 1)
    return d_color + _diff_x_t(d_dx) + ty(d_dy) + ty(_diff_x_t(d_dxdy))


# ---------------------------------------------------------------------------
# Loss (L1 + SSIM) and Adam
# ---------------------------------------------------------------------------

SSIM_WINDOW = 11      # baselines.py:15
SSIM_SIGMA = 1.5      # baselines.py:16
SSIM_C1 = 0.01 ** 2   # baselines.py:17
SSIM_C2 = 0.03 ** 2   # baselines.py:18


def ssim_window() -> np.ndarray:
    """baselines.py:116-120."""
    half = SSIM_WINDOW // 2
    x = np.arange(-half, half + 1, dtype=np.float64)
    w = np.exp(-(x * x) / (2.0 * SSIM_SIGMA * SSIM_SIGMA))
    return w / w.sum()


def _corr1d(img: np.ndarray, w: np.ndarray, axis: int) -> np.ndarray:
    """Zero-padded correlation along one axis (scipy correlate1d mode=constant)."""
    half = len(w) // 2
    img = np.moveaxis(img, axis, 0)
    pad = np.zeros((img.shape[0] + 2 * half,) + img.shape[1:])
    pad[half:half + img.shape[0]] = img
    out = np.zeros_like(img)
    for k in range(len(w)):
        out += w[k] * pad[k:k + img.shape[0]]
    return np.moveaxis(out, 0, axis)


def _filter2(img, w):
    """baselines.py:123-125."""
    return _corr1d(_corr1d(img, w, 0), w, 1)


def ssim_with_grad(pred, target):
    """baselines.py:128-143 + 170-203."""
    pred = np.asarray(pred, np.float64)
    target = np.asarray(target, np.float64)
    h, w = pred.shape[:2]
    half = SSIM_WINDOW // 2
    win = ssim_window()
    nch = pred.shape[2]
    inner = (h - 2 * half) * (w - 2 * half)
    grad = np.zeros_like(pred)
    vals = []
    for c in range(nch):
        x = pred[:, :, c]
        y = target[:, :, c]
        ux, uy = _filter2(x, win), _filter2(y, win)
        vx, vy, vxy = _filter2(x * x, win), _filter2(y * y, win), _filter2(x * y, win)
        sxx = vx - ux * ux
        syy = vy - uy * uy
        sxy = vxy - ux * uy
        n1 = 2.0 * ux * uy + SSIM_C1
        n2 = 2.0 * sxy + SSIM_C2
        d1 = ux * ux + uy * uy + SSIM_C1
        d2 = sxx + syy + SSIM_C2
        smap = (n1 * n2) / (d1 * d2)
        vals.append(np.mean(smap[half:h - half, half:w - half]))
        g = np.zeros((h, w))
        g[half:h - half, half:w - half] = 1.0 / (inner * nch)
        p = n1 / d1
        q = n2 / d2
        g_ux = g * (q * (2.0 * uy * d1 - 2.0 * ux * n1) / (d1 * d1)
                    + p * (-2.0 * uy / d2 + 2.0 * ux * n2 / (d2 * d2)))
        g_vx = g * p * (-n2 / (d2 * d2))
        g_vxy = g * p * (2.0 / d2)
        grad[:, :, c] = (_filter2(g_ux, win) + 2.0 * x * _filter2(g_vx, win)
                         + y * _filter2(g_vxy, win))
    return float(np.mean(vals)), grad


def loss(pred, target, ssim_weight: float):
    """fit.py:94-108: (1-l) L1 + l (1 - SSIM) and its adjoint."""
    pred = np.asarray(pred, np.float64)
    target = np.asarray(target, np.float64)
    diff = pred - target
    adj = (1.0 - ssim_weight) * np.sign(diff) / diff.size
    value = (1.0 - ssim_weight) * np.mean(np.abs(diff))
    if ssim_weight > 0.0:
        s, ds = ssim_with_grad(pred, target)
        value += ssim_weight * (1.0 - s)
        adj = adj - ssim_weight * ds
    return value, adj


def adam_step(params: dict, grads: dict, m: dict, v: dict, t: int, lrs: dict,
              beta1=0.9, beta2=0.999, eps=1e-8):
    """fit.py:144-160; returns (new_params, m, v, t)."""
    t += 1
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    out = {}
    for k, p in params.items():
        g = grads[k]
        m[k] = beta1 * m[k] + (1.0 - beta1) * g
        v[k] = beta2 * v[k] + (1.0 - beta2) * g * g
        out[k] = p - lrs[k] * (m[k] / bc1) / (np.sqrt(v[k] / bc2) + eps)
    return out, m, v, t


# ---- 3D front-end ---------------------------------------

def project_gaussians(means3, log_scales3, quats, opacity_logits, R, t, fx, fy, cx, cy, near):
    """float64 restatement of the EWA local-affine projection (PAPER.md:154-162:
    Sigma' = J W Sigma W^T J^T) into the reference's 2D parametrisation
    (core.py:175-182).  The reference package is 2D-only, so this restatement is
    the pin for csrc/project.cu ("parity unpinned" w.r.t. the reference itself).
    Returns (means2 (N,2), log_scales2 (N,2), rotations (N,), opacity_logits (N,), depths (N,))."""
    mu = np.asarray(means3, np.float64).reshape(-1, 3)
    R = np.asarray(R, np.float64).reshape(3, 3)
    t = np.asarray(t, np.float64).reshape(3)
    cam = mu @ R.T + t
    x, y, z = cam[:, 0], cam[:, 1], cam[:, 2]
    ok = z > near
    zs = np.where(ok, z, 1.0)
    q = np.asarray(quats, np.float64).reshape(-1, 4)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w_, a_, b_, c_ = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    Q = np.stack([
        np.stack([1 - 2 * (b_ * b_ + c_ * c_), 2 * (a_ * b_ - w_ * c_), 2 * (a_ * c_ + w_ * b_)], -1),
        np.stack([2 * (a_ * b_ + w_ * c_), 1 - 2 * (a_ * a_ + c_ * c_), 2 * (b_ * c_ - w_ * a_)], -1),
        np.stack([2 * (a_ * c_ - w_ * b_), 2 * (b_ * c_ + w_ * a_), 1 - 2 * (a_ * a_ + b_ * b_)], -1)], 1)
    s2 = np.exp(2.0 * np.asarray(log_scales3, np.float64).reshape(-1, 3))
    J = np.zeros((len(mu), 2, 3))
    J[:, 0, 0] = fx / zs
    J[:, 0, 2] = -fx * x / (zs * zs)
    J[:, 1, 1] = fy / zs
    J[:, 1, 2] = -fy * y / (zs * zs)
    M = J @ R @ Q                                        # (N, 2, 3)
    S = np.einsum("nik,nk,njk->nij", M, s2, M)           # M diag(s2) M^T
    a, b, c = S[:, 0, 0], S[:, 0, 1], S[:, 1, 1]
    h = 0.5 * (a + c)
    d = np.sqrt(0.25 * (a - c) ** 2 + b * b)
    lmax = h + d
    lmin = np.maximum(h - d, 1e-12 * lmax)
    means2 = np.stack([fx * x / zs + cx, fy * y / zs + cy], 1)
    ls2 = np.stack([0.5 * np.log(lmax), 0.5 * np.log(lmin)], 1)
    rot = 0.5 * np.arctan2(2.0 * b, a - c)
    logits = np.where(ok, np.asarray(opacity_logits, np.float64).reshape(-1), -100.0)
    means2[~ok] = (cx, cy)
    ls2[~ok] = 0.0
    rot[~ok] = 0.0
    return means2, ls2, rot, logits, z
