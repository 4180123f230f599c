"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the reference is importable there, never on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
    python tests/golden/make_golden.py

Every fixture stores the float64 scene / image inputs and the reference's own
outputs.  tests/test_oracle_golden.py pins the CPU oracle against them
(bit-exact for integer outputs and the rasterizer, <=1e-12 elsewhere), and the
GPU parity tests compare the CUDA path against the same files.

Scene recipes come from the reference test fixtures (pkg/tests/conftest.py:7-77
``smooth_scene``/``sharp_scene``/``random_gradient_image``) and the reference
tests that pin the path (test_raster_forward.py, test_raster_backward.py,
test_spline.py); the larger ones use this repo's synthetic generator
(paper_2503_14171_b200/scenes.py, mirroring corpus.bench_scene).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from splinesplat import core as rcore                       # noqa: E402
import importlib                                             # noqa: E402
rfit = importlib.import_module("splinesplat.fit")
from splinesplat import raster_backward as rb               # noqa: E402
from splinesplat import raster_forward as rf                # noqa: E402
from splinesplat import spline as rsp                       # noqa: E402
from conftest import random_gradient_image, sharp_scene, smooth_scene  # noqa: E402

from paper_2503_14171_b200 import scenes as S               # noqa: E402

FWD_FIELDS = ("color", "d_dx", "d_dy", "d_dxdy", "alpha", "alpha_dx", "alpha_dy",
              "alpha_dxdy", "contrib_count")


def _scene_arrays(sc):
    return dict(means=sc.means, log_scales=sc.log_scales, rotations=sc.rotations,
                opacity_logits=sc.opacity_logits, colors=sc.colors, depths=sc.depths,
                background=sc.background,
                ref_res=np.array(sc.reference_resolution, dtype=np.float64))


def _as_ref(sc):
    return rcore.Scene(sc.means, sc.log_scales, sc.rotations, sc.opacity_logits, sc.colors,
                       sc.depths, sc.background, tuple(sc.reference_resolution))


def _bins(sc, w, h):
    if sc.n == 0:
        return dict()
    pack = rf.prepare_scene(sc, w, h)
    _, lists = rf.bin_tiles(pack, w, h)
    off = np.zeros(len(lists) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(x) for x in lists])
    ranks = np.concatenate(lists).astype(np.int64) if off[-1] else np.zeros(0, np.int64)
    return dict(order=pack.order, bboxes=pack.bboxes, valid=pack.valid,
                conics=pack.conics, sigmas=pack.sigmas, pmeans=pack.means,
                tile_off=off, tile_ranks=ranks)


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1024:.1f} KiB")


def forward_case(name, sc, w, h, upscale=None):
    img = rf.render_forward(sc, w, h, threads=8)
    out = _scene_arrays(sc)
    out.update(out_w=w, out_h=h)
    out.update({f: getattr(img, f) for f in FWD_FIELDS})
    out.update(_bins(sc, w, h))
    if upscale is not None:
        out["up_factor"] = upscale
        out["up"] = rsp.upscale_spline(img, upscale)
    save("fwd_" + name, **out)


def single_splat_scene(opacity_logit=8.0, color=(1.0, 0.0, 0.0), scale=6.0, size=33):
    # test_raster_forward.py:16-26
    c = (size - 1) / 2 + 0.5
    return rcore.Scene(means=np.array([[c, c]]), log_scales=np.log([[scale, scale]]),
                       rotations=np.zeros(1), opacity_logits=np.array([opacity_logit]),
                       colors=np.array([color]), depths=np.zeros(1), background=np.zeros(3),
                       reference_resolution=(size, size))


def forward_cases():
    for seed, n, w, h in [(0, 25, 40, 56), (1, 60, 64, 64), (2, 5, 17, 31)]:
        sc = sharp_scene(seed, n, max(w, h))
        sc.reference_resolution = (w, h)
        forward_case(f"sharp{seed}", sc, w, h)
    forward_case("smooth1", smooth_scene(1, 25, 64), 64, 64)
    forward_case("clamped", single_splat_scene(), 33, 33)
    forward_case("unclamped", single_splat_scene(opacity_logit=float(rcore.logit(0.7))), 33, 33)
    # test_raster_forward.py:64-90 two-splat closed form
    two = rcore.Scene(means=np.array([[8.0, 8.0], [9.0, 8.5]]),
                      log_scales=np.log(np.full((2, 2), 5.0)), rotations=np.zeros(2),
                      opacity_logits=rcore.logit(np.array([0.6, 0.45])),
                      colors=np.array([[0.9, 0.2, 0.1], [0.1, 0.5, 0.8]]),
                      depths=np.array([1.0, 2.0]), background=np.array([0.25, 0.3, 0.35]),
                      reference_resolution=(16, 16))
    forward_case("two_splat", two, 16, 16)
    zero = sharp_scene(3, 10, 24)
    zero.opacity_logits = np.full(zero.n, -40.0)
    forward_case("zero_opacity", zero, 24, 24)
    ext = sharp_scene(3, 4, 24)
    ext.log_scales = np.array([[10.0, 10.0], [-10.0, -10.0], [10.0, -10.0], [0.0, 0.0]])
    forward_case("extreme_scales", ext, 24, 24)
    # test_raster_forward.py:151-187 — early termination fires
    rng = np.random.default_rng(5)
    n = 40
    term = rcore.Scene(means=rng.uniform(8, 16, (n, 2)), log_scales=np.log(rng.uniform(6, 9, (n, 2))),
                       rotations=np.zeros(n), opacity_logits=rcore.logit(rng.uniform(0.6, 0.9, n)),
                       colors=rng.uniform(0, 1, (n, 3)), depths=rng.uniform(0, 1, n),
                       background=rng.uniform(0, 1, 3), reference_resolution=(24, 24))
    forward_case("termination", term, 24, 24)
    forward_case("one_pixel", sharp_scene(2, 6, 32), 1, 1)
    forward_case("thin_row", sharp_scene(2, 6, 32), 32, 1)
    forward_case("nonuniform", smooth_scene(77, 5, 64), 40, 20)
    forward_case("empty", rcore.Scene.from_gaussians([], background=(0.2, 0.4, 0.6),
                                                      reference_resolution=(4, 4)), 4, 4)
    # depth ties keep storage order (SPEC stable sort)
    ties = sharp_scene(4, 50, 48)
    ties.depths = np.round(ties.depths * 4) / 4
    forward_case("depth_ties", ties, 48, 48)
    # view model on a synthetic canvas (scenes.view_scene)
    canvas = S.synthetic_scene(1500, 96, 54, (0.6, 3.0), seed=3)
    view = S.View(1.2, 11.25, 7.5)
    forward_case("view_zoom", _as_ref(S.view_scene(canvas, view)), 96, 54, upscale=2.0)
    # C1: 10k splats, 128x128, x2 (BASELINE.json configs[0])
    c1 = S.CONFIGS["c1"]
    sc = S.synthetic_scene(c1.n, c1.width, c1.height, c1.scale_range, seed=5)
    forward_case("c1", _as_ref(sc), c1.width, c1.height, upscale=c1.factor)


def upscale_cases():
    for name, seed, w, h, factor, size in [("f1", 1, 11, 8, 1.0, None),
                                           ("f2", 3, 13, 9, 2.0, None),
                                           ("f4", 4, 10, 7, 4.0, None),
                                           ("f25", 6, 7, 9, 2.5, None),
                                           ("f17", 2, 10, 10, 1.7, None),
                                           ("size", 5, 9, 6, 2.0, (23, 17))]:
        img = random_gradient_image(seed, w, h)
        if factor == 1.0:
            img.color[:] = np.clip(img.color, 0, 1)
        out = rsp.upscale_spline(img, factor, out_size=size)
        raw = rsp.upscale_spline(img, factor, out_size=size, clamp=False)
        rng = np.random.default_rng(seed + 100)
        adj = rng.normal(0, 1, raw.shape)
        back = rsp.upscale_backward(img, factor, adj, out_size=size)
        save("up_" + name, color=img.color, d_dx=img.d_dx, d_dy=img.d_dy, d_dxdy=img.d_dxdy,
             factor=factor, out_size=np.array(size if size else (-1, -1)), out=out, raw=raw,
             adjoint=adj, b_color=back.d_color, b_dx=back.d_dx, b_dy=back.d_dy,
             b_dxdy=back.d_dxdy)


def backward_case(name, sc, w, h, adj=None, seed=0):
    img = rf.render_forward(sc, w, h, threads=8)
    if adj is None:
        rng = np.random.default_rng(seed)
        adj = rb.PixelAdjoint(*[rng.normal(0, 1, (h, w, 3)) for _ in range(4)])
    g = rb.render_backward(sc, img, adj, threads=8)
    out = _scene_arrays(sc)
    out.update(out_w=w, out_h=h, w=adj.w, wx=adj.wx, wy=adj.wy, wxy=adj.wxy,
               d_means=g.d_means, d_log_scales=g.d_log_scales, d_rotations=g.d_rotations,
               d_opacity_logits=g.d_opacity_logits, d_colors=g.d_colors)
    out.update({f: getattr(img, f) for f in FWD_FIELDS})
    save("bwd_" + name, **out)


def backward_cases():
    backward_case("sharp8", sharp_scene(8, 30, 48), 48, 48, seed=2)
    backward_case("smooth_nonuniform", smooth_scene(77, 5, 64), 40, 20, seed=0)
    clamped = rcore.Scene(means=np.array([[8.5, 8.5]]), log_scales=np.log([[6.0, 6.0]]),
                          rotations=np.zeros(1), opacity_logits=np.array([10.0]),
                          colors=np.array([[0.2, 0.6, 0.9]]), depths=np.zeros(1),
                          background=np.zeros(3), reference_resolution=(16, 16))
    adj = rb.PixelAdjoint.zeros(16, 16)
    adj.w[8, 8, :] = 1.0
    backward_case("clamped", clamped, 16, 16, adj=adj)
    zero = sharp_scene(5, 6, 20)
    zero.opacity_logits = zero.opacity_logits.copy()
    zero.opacity_logits[2] = -40.0
    backward_case("culled", zero, 20, 20, seed=1)
    # a C5-shaped miniature: 2-10 px splats on a 192x108 canvas rendered at 48x27
    sc = S.synthetic_scene(1500, 192, 108, (2.0, 10.0), seed=5)
    backward_case("mini_c5", _as_ref(sc), 48, 27, seed=4)


def loss_cases():
    rng = np.random.default_rng(21)
    pred = rng.uniform(0, 1, (32, 40, 3))
    target = rng.uniform(0, 1, (32, 40, 3))
    v02, a02 = rfit.loss(pred, target, 0.2)
    v0, a0 = rfit.loss(pred, target, 0.0)
    v1, a1 = rfit.loss(pred, target, 1.0)
    save("loss", pred=pred, target=target, v02=v02, a02=a02, v0=v0, a0=a0, v1=v1, a1=a1)


def fd_cases():
    rng = np.random.default_rng(31)
    image = rng.uniform(0, 1, (9, 12, 3))
    g = rsp.fd_gradients(image)
    adj = [rng.normal(0, 1, (9, 12, 3)) for _ in range(4)]
    back = rsp.fd_gradients_backward(rsp.SourceAdjoint(*adj))
    save("fd", image=image, d_dx=g.d_dx, d_dy=g.d_dy, d_dxdy=g.d_dxdy,
         a_color=adj[0], a_dx=adj[1], a_dy=adj[2], a_dxdy=adj[3], back=back)


def train_case():
    """One upscale-aware training step, reference fit.py:188-223 body."""
    canvas = (128, 72)
    model = S.synthetic_scene(800, canvas[0], canvas[1], (2.0, 6.0), seed=5)
    target_scene = S.synthetic_scene(800, canvas[0], canvas[1], (2.0, 6.0), seed=7)
    tgt = np.clip(rf.render_forward(_as_ref(target_scene), *canvas, threads=8).color, 0, 1)
    sc = _as_ref(model)
    low_w, low_h = 32, 18
    fwd = rf.render_forward(sc, low_w, low_h, threads=8)
    pred = rsp.upscale_spline(fwd, 4.0, out_size=canvas)
    value, dpred = rfit.loss(pred, tgt, 0.2)
    sadj = rsp.upscale_backward(fwd, 4.0, dpred, out_size=canvas)
    adj = rb.PixelAdjoint(w=sadj.d_color, wx=sadj.d_dx, wy=sadj.d_dy, wxy=sadj.d_dxdy)
    g = rb.render_backward(sc, fwd, adj, threads=8)
    lrs = dict(rfit.DEFAULT_LEARNING_RATES)
    lrs["means"] = lrs["means"] * max(canvas)
    params = rfit._scene_params(sc)
    state = rfit.AdamState.like(params)
    grads = {"means": g.d_means, "log_scales": g.d_log_scales, "rotations": g.d_rotations,
             "opacity_logits": g.d_opacity_logits, "colors": g.d_colors}
    new, state = rfit.adam_step(params, grads, state, lrs)
    out = _scene_arrays(sc)
    out.update(target=tgt, low_w=low_w, low_h=low_h, pred=pred, loss=value, dpred=dpred,
               d_means=g.d_means, d_log_scales=g.d_log_scales, d_rotations=g.d_rotations,
               d_opacity_logits=g.d_opacity_logits, d_colors=g.d_colors,
               **{"new_" + k: v for k, v in new.items()})
    save("train_step", **out)


def io_case():
    """Wire formats (reference io.py): scene JSON v1 text, a GIMG dump of a
    reference render, the reference upscale of the re-loaded dump, and display
    encoding of values in and beyond [0, 1]."""
    import tempfile
    from splinesplat import io as rio
    sc = _as_ref(sharp_scene(seed=4, n=60, size=40))
    w, h = 40, 24
    with tempfile.TemporaryDirectory() as d:
        rio.save_scene(os.path.join(d, "s.json"), sc)
        text = open(os.path.join(d, "s.json"), "rb").read()
        img = rf.render_forward(sc, w, h, threads=8)
        rio.save_gradient_dump(os.path.join(d, "g.gimg"), img)
        blob = open(os.path.join(d, "g.gimg"), "rb").read()
        back = rio.load_gradient_dump(os.path.join(d, "g.gimg"))
    up = rsp.upscale_spline(back, 2.0)
    rng = np.random.default_rng(3)
    enc_in = np.concatenate([rng.uniform(-0.1, 1.1, 4000), np.linspace(0.0, 1.0, 1001),
                             [0.0, 1.0, -1.0, 2.0]]).astype(np.float32)
    enc_out = rio.encode_display(enc_in.astype(np.float64))
    save("io", scene_json=np.frombuffer(text, dtype=np.uint8), gimg=np.frombuffer(blob, dtype=np.uint8),
         up=up, enc_in=enc_in, enc_out=enc_out, out_w=w, out_h=h, **_scene_arrays(sc))


def fit_cases():
    """The single-image fit driver (reference fit.py:163-245): short runs in each
    upscale mode with per-iteration rows and pruning, from a rendered target."""
    tsc = _as_ref(sharp_scene(seed=2, n=120, size=48))
    target = np.clip(rf.render_forward(tsc, 48, 32, threads=8).color, 0.0, 1.0)
    cases = {
        "spline": dict(iterations=6, num_gaussians=50, render_scale=2.0, upscale_mode="spline_analytic",
                       log_every=1, prune_interval=3, prune_opacity=0.475, seed=1),
        "fd": dict(iterations=4, num_gaussians=50, render_scale=2.0, upscale_mode="bicubic_fd",
                   log_every=1, seed=2),
        "none": dict(iterations=4, num_gaussians=50, render_scale=1.0, upscale_mode="none",
                     log_every=2, ssim_weight=0.0, seed=3),
    }
    for name, kw in cases.items():
        cfg = rfit.FitConfig(**kw)
        rep = rfit.fit(target, cfg, threads=8)
        rows = np.array([[r.iteration, r.loss, r.psnr, r.ssim] for r in rep.rows], dtype=np.float64)
        sc = rep.scene
        save("fit_" + name, target=target, rows=rows, cfg=np.array(repr(kw)),
             means=sc.means, log_scales=sc.log_scales, rotations=sc.rotations,
             opacity_logits=sc.opacity_logits, colors=sc.colors, depths=sc.depths)


def points_case():
    """render_at_points (raster_forward.py:190-233) at random continuous positions,
    with the blend signature."""
    sc = _as_ref(sharp_scene(seed=6, n=40, size=48))
    rng = np.random.default_rng(12)
    xs = rng.uniform(-2.0, 50.0, 300)
    ys = rng.uniform(-2.0, 40.0, 300)
    out, state = rf.render_at_points(sc, xs, ys, 48, 36, with_state=True)
    save("points", xs=xs, ys=ys, out=out, state=state, out_w=48, out_h=36, **_scene_arrays(sc))


def recon_case():
    """The reference's self-reconstruction benchmark target (tests/conftest.py:45-65)."""
    from conftest import reconstruction_target
    _, target = reconstruction_target()
    save("recon_target", target=target)


if __name__ == "__main__":
    forward_cases()
    upscale_cases()
    backward_cases()
    loss_cases()
    fd_cases()
    train_case()
    io_case()
    fit_cases()
    points_case()
    recon_case()
