"""Pin the CPU oracle against golden vectors written by the reference itself.

The fixtures (tests/golden/*.npz) come from tests/golden/make_golden.py, which
runs the reference package.  The oracle must reproduce them bit-exactly where
the arithmetic is the same (preprocess, binning, rasterizer forward/backward)
and to float64 round-off elsewhere (upscaler, loss).
"""

import numpy as np
import pytest

from conftest import golden, golden_names, scene_of

FIELDS = ("color", "d_dx", "d_dy", "d_dxdy", "alpha", "alpha_dx", "alpha_dy",
          "alpha_dxdy", "contrib_count")


@pytest.mark.parametrize("name", golden_names("fwd_"))
def test_oracle_forward_bitexact(oracle, name):
    g = golden(name)
    sc = scene_of(g)
    w, h = int(g["out_w"]), int(g["out_h"])
    img = oracle.render_forward(sc, w, h)
    for f in FIELDS:
        assert np.array_equal(getattr(img, f), g[f]), (name, f)
    if sc.n:
        pack = oracle.prepare_scene(oracle.OScene.of(sc), w, h)
        assert np.array_equal(pack.order, g["order"])
        assert np.array_equal(pack.bboxes, g["bboxes"])
        assert np.array_equal(pack.valid, g["valid"])
        assert np.array_equal(pack.conics, g["conics"])
        off, ranks, _ = oracle.bin_tiles_csr(pack, w, h)
        assert np.array_equal(off, g["tile_off"])
        assert np.array_equal(ranks, g["tile_ranks"])
    if "up" in g:
        up = oracle.upscale_spline(img.color, img.d_dx, img.d_dy, img.d_dxdy, float(g["up_factor"]))
        assert np.abs(up - g["up"]).max() < 1e-12


@pytest.mark.parametrize("name", ["fwd_sharp0", "fwd_sharp2", "fwd_termination"])
def test_oracle_untiled_equals_tiled(oracle, name):
    # reference test_raster_forward.py:190-197 (tiled == untiled bitwise)
    g = golden(name)
    sc = scene_of(g)
    w, h = int(g["out_w"]), int(g["out_h"])
    a = oracle.render_forward(sc, w, h, tiled=False)
    for f in FIELDS:
        assert np.array_equal(getattr(a, f), g[f]), f


@pytest.mark.parametrize("name", golden_names("up_"))
def test_oracle_upscale(oracle, name):
    g = golden(name)
    size = None if g["out_size"][0] < 0 else tuple(int(v) for v in g["out_size"])
    f = float(g["factor"])
    out = oracle.upscale_spline(g["color"], g["d_dx"], g["d_dy"], g["d_dxdy"], f, out_size=size)
    raw = oracle.upscale_spline(g["color"], g["d_dx"], g["d_dy"], g["d_dxdy"], f, out_size=size,
                                clamp=False)
    assert out.shape == g["out"].shape
    assert np.abs(out - g["out"]).max() < 1e-12
    assert np.abs(raw - g["raw"]).max() < 1e-12
    h, w = g["color"].shape[:2]
    back = oracle.upscale_backward(w, h, f, g["adjoint"], out_size=size)
    for got, key in zip(back, ("b_color", "b_dx", "b_dy", "b_dxdy")):
        assert np.abs(got - g[key]).max() < 1e-11, key


@pytest.mark.parametrize("name", golden_names("bwd_"))
def test_oracle_backward_bitexact(oracle, name):
    g = golden(name)
    sc = scene_of(g)
    w, h = int(g["out_w"]), int(g["out_h"])
    img = oracle.render_forward(sc, w, h)
    grads = oracle.render_backward(sc, img, (g["w"], g["wx"], g["wy"], g["wxy"]))
    for k in ("d_means", "d_log_scales", "d_rotations", "d_opacity_logits", "d_colors"):
        assert np.array_equal(grads[k], g[k]), k


def test_oracle_loss(oracle):
    g = golden("loss")
    for lam, v, a in ((0.2, "v02", "a02"), (0.0, "v0", "a0"), (1.0, "v1", "a1")):
        value, adj = oracle.loss(g["pred"], g["target"], lam)
        assert abs(value - float(g[v])) < 1e-12
        assert np.abs(adj - g[a]).max() < 1e-15


def test_oracle_fd(oracle):
    g = golden("fd")
    _, dx, dy, dxy = oracle.fd_gradients(g["image"])
    assert np.array_equal(dx, g["d_dx"]) and np.array_equal(dy, g["d_dy"])
    assert np.array_equal(dxy, g["d_dxdy"])
    back = oracle.fd_gradients_backward(g["a_color"], g["a_dx"], g["a_dy"], g["a_dxdy"])
    assert np.abs(back - g["back"]).max() < 1e-14


def test_oracle_training_step(oracle):
    g = golden("train_step")
    sc = scene_of(g)
    lw, lh = int(g["low_w"]), int(g["low_h"])
    tgt = g["target"]
    H, W = tgt.shape[:2]
    fwd = oracle.render_forward(sc, lw, lh)
    pred = oracle.upscale_spline(fwd.color, fwd.d_dx, fwd.d_dy, fwd.d_dxdy, 4.0, out_size=(W, H))
    assert np.abs(pred - g["pred"]).max() < 1e-12
    value, dpred = oracle.loss(pred, tgt, 0.2)
    assert abs(value - float(g["loss"])) < 1e-12
    adj = oracle.upscale_backward(lw, lh, 4.0, dpred, out_size=(W, H))
    grads = oracle.render_backward(sc, fwd, adj)
    for k in ("d_means", "d_log_scales", "d_rotations", "d_opacity_logits", "d_colors"):
        ref = g[k]
        assert np.abs(grads[k] - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max()), k
    lrs = {"means": 2e-3 * max(W, H), "log_scales": 5e-3, "rotations": 1e-3,
           "opacity_logits": 5e-2, "colors": 2.5e-2}
    params = {"means": sc.means, "log_scales": sc.log_scales, "rotations": sc.rotations,
              "opacity_logits": sc.opacity_logits, "colors": sc.colors}
    m = {k: np.zeros_like(v) for k, v in params.items()}
    v = {k: np.zeros_like(x) for k, x in params.items()}
    gmap = {"means": grads["d_means"], "log_scales": grads["d_log_scales"],
            "rotations": grads["d_rotations"], "opacity_logits": grads["d_opacity_logits"],
            "colors": grads["d_colors"]}
    new, *_ = oracle.adam_step(params, gmap, m, v, 0, lrs)
    for k in new:
        assert np.abs(new[k] - g["new_" + k]).max() < 1e-9, k
