"""The batched multi-view pipeline equals per-view render_forward + upscale_spline."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_pipeline_matches_single_view_api():
    import torch
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200.pipeline import ViewPipeline
    sc = P.synthetic_scene(30000, 320, 180, (0.5, 2.5), seed=5)
    views = P.random_views(5, 320, 180, seed=2)
    for slots in (1, 3):
        pipe = ViewPipeline(sc, 320, 180, factor=4.0, slots=slots, views_for_capacity=views)
        outs = pipe.render(views, keep=True)
        pipe.join()
        torch.cuda.synchronize()
        pipe.check()
        for v, got in zip(views, outs):
            ref = P.upscale_spline(P.render_forward(sc, 320, 180, view=v), 4.0)
            assert torch.equal(got, ref)


def test_pipeline_host_ring_copies():
    import torch
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200.pipeline import ViewPipeline
    sc = P.synthetic_scene(5000, 96, 54, (0.5, 2.5), seed=1)
    views = P.random_views(4, 96, 54, seed=3)
    pipe = ViewPipeline(sc, 96, 54, factor=2.0, slots=2, views_for_capacity=views)
    ring = [torch.empty((108, 192, 3)).pin_memory() for _ in range(4)]
    pipe.render(views, host_out=ring)
    pipe.join()
    torch.cuda.synchronize()
    for i, v in enumerate(views):
        ref = P.upscale_spline(P.render_forward(sc, 96, 54, view=v), 2.0).cpu()
        assert torch.equal(ring[i], ref)


def test_pipeline_overflow_is_detected():
    import torch
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200.pipeline import ViewPipeline
    sc = P.synthetic_scene(5000, 96, 54, (0.5, 2.5), seed=1)
    pipe = ViewPipeline(sc, 96, 54, factor=2.0, capacity=100)
    pipe.render([None])
    torch.cuda.synchronize()
    with pytest.raises(RuntimeError):
        pipe.check()


def test_batched_views_api():
    """render_upscale_views: (V, Ho, Wo, 3) batch == per-view reference API."""
    import torch
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200.pipeline import render_upscale_views
    sc = P.synthetic_scene(8000, 128, 72, (0.5, 2.5), seed=4)
    views = P.random_views(6, 128, 72, seed=5)
    out = render_upscale_views(sc, 128, 72, views, factor=2.0, slots=3)
    assert tuple(out.shape) == (6, 144, 256, 3)
    for i, v in enumerate(views):
        assert torch.equal(out[i], P.upscale_spline(P.render_forward(sc, 128, 72, view=v), 2.0))


def test_stage_timed_pipeline_is_bitwise_the_fused_one():
    """Stage timing runs the raster kernel and the exact fix-up as separate calls
    (splat_rasterize(..., SPLAT_RASTER_DEFER_FIXUP) + splat_fixup): same frames, bit for bit,
    on a scene whose termination boundary exercises the fix-up."""
    import torch
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200.pipeline import ViewPipeline
    sc = P.synthetic_scene(60000, 320, 180, (0.5, 2.5), seed=9)
    views = P.random_views(4, 320, 180, seed=6)
    a = ViewPipeline(sc, 320, 180, factor=4.0, slots=1, views_for_capacity=views)
    b = ViewPipeline(sc, 320, 180, factor=4.0, slots=1, capacity=a.capacity)
    b.enable_stage_timing(True)
    fa, fb = a.render(views, keep=True), b.render(views, keep=True)
    torch.cuda.synchronize()
    assert set(b.stage_times_ms()) == {"prepare", "bin", "raster", "fixup", "upscale"}
    for x, y in zip(fa, fb):
        assert torch.equal(x, y)
    assert int(a.slots[0].frame.counters()[2]) > 0   # the last view did flag pixels for the fix-up


@pytest.mark.parametrize("w,h,factor", [(1, 1, 4.0), (3, 2, 4.0), (17, 1, 2.0), (5, 33, 2.0), (16, 16, 4.0)])
def test_pipeline_tiny_and_ragged_renders(w, h, factor):
    """Degenerate render sizes (1 pixel, 1-pixel rows / columns, single partial tiles)
    through the multi-slot pipeline equal the single-view API bitwise (the reference's
    degenerate-size tests, test_raster_forward.py:289-303)."""
    import torch
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200.pipeline import ViewPipeline
    sc = P.synthetic_scene(400, max(w, 8), max(h, 8), (0.5, 3.0), seed=w * 31 + h)
    views = P.random_views(3, max(w, 8), max(h, 8), seed=1)
    pipe = ViewPipeline(sc, w, h, factor=factor, slots=2, views_for_capacity=views)
    outs = pipe.render(views, keep=True)
    pipe.join()
    torch.cuda.synchronize()
    for v, got in zip(views, outs):
        assert torch.equal(got, P.upscale_spline(P.render_forward(sc, w, h, view=v), factor))


def test_pipeline_empty_scene_renders_background():
    """An empty scene (render_forward's early exit, raster_forward.py:162-164) through the
    pipeline: every upscaled frame is the background."""
    import torch
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200.pipeline import render_upscale_views
    sc = P.Scene.empty(background=(0.25, 0.5, 0.75), reference_resolution=(40, 24))
    out = render_upscale_views(sc, 40, 24, [None, None, None], factor=2.0, slots=2)
    torch.cuda.synchronize()
    bg = torch.tensor([0.25, 0.5, 0.75], device="cuda")
    assert tuple(out.shape) == (3, 48, 80, 3)
    assert torch.allclose(out, bg.expand_as(out), rtol=0, atol=1e-7)
