"""Small invocations of every kernel family for compute-sanitizer:

    compute-sanitizer --tool racecheck|synccheck|memcheck python tools/sanitize.py

C1-sized forward (inference + training mode, incl. the exact fix-up on a
termination-boundary scene), the backward on the bwd_mini_c5 golden (its
inter-warp ring slots), the x2/x4/generic upscalers and their backward (TMA /
mbarrier pipelines), the L1+SSIM loss, Adam, binning on both paths, and the
4-slot pipeline.  Each step is checked against the previous run's output so the
sanitized run is also a determinism check.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2503_14171_b200 as P  # noqa: E402
from conftest import golden, scene_of  # noqa: E402
from paper_2503_14171_b200 import fit  # noqa: E402
from paper_2503_14171_b200.pipeline import ViewPipeline  # noqa: E402
from paper_2503_14171_b200.raster_forward import BIN_ATOMIC  # noqa: E402


def main():
    torch.cuda.set_device(0)
    sc = P.synthetic_scene(10000, 128, 128, (1.28, 6.4), seed=5)        # C1
    img = P.render_forward(sc, 128, 128)
    up2 = P.upscale_spline(img, 2.0)
    up4 = P.upscale_spline(img, 4.0)
    upg = P.upscale_spline(img, 2.5)
    P.upscale_spline(P.render_forward(sc, 127, 65), 2.0)                  # odd width: generic x2
    print("forward + upscale ok", img.stats)
    # termination-boundary scene: the exact fix-up runs
    from test_gpu_forward import _shell_scene
    sh = _shell_scene(2, 96, 9, True)
    simg = P.render_forward(sh, 96, 96)
    timg = P.render_forward(sh, 96, 96, train=True)
    print("fix-up pixels", simg.stats, timg.stats)
    # binning, both paths
    pack = P.prepare_scene(sc, 128, 128)
    _, a = P.bin_tiles(pack, 128, 128)
    _, b = P.bin_tiles(pack, 128, 128, _flags=BIN_ATOMIC)
    assert torch.equal(a.ranks, b.ranks)
    # backward on the mini-C5 golden
    g = golden("bwd_mini_c5")
    gs = scene_of(g)
    w, h = int(g["out_w"]), int(g["out_h"])
    fimg = P.render_forward(gs, w, h, train=True)
    adj = P.PixelAdjoint.of(g["w"], g["wx"], g["wy"], g["wxy"])
    g1 = P.render_backward(gs, fimg, adj)
    g2 = P.render_backward(gs, fimg, adj)
    assert torch.equal(g1.d_means, g2.d_means)
    print("backward ok")
    # upscale backward (x4 and generic), loss, Adam via one training step
    P.upscale_backward(img, 4.0, torch.randn_like(up4))
    P.upscale_backward(img, 2.5, torch.randn_like(upg))
    P.upscale_backward(img, 2.0, torch.randn_like(up2))
    tsc = P.synthetic_scene(3000, 96, 64, (2.0, 6.0), seed=7)
    tgt = P.render_forward(tsc, 96, 64).color.clamp(0, 1).contiguous()
    tr = fit.ViewTrainer(P.synthetic_scene(3000, 96, 64, (2.0, 6.0), seed=5), (24, 16), (96, 64),
                         [None, None], [tgt, tgt])
    tr.step()
    tr.step()
    print("training step ok")
    # the 4-slot pipeline
    views = P.random_views(6, 128, 128, seed=2)
    pipe = ViewPipeline(sc, 128, 128, factor=4.0, slots=4, views_for_capacity=views)
    pipe.render(views)
    pipe.join()
    torch.cuda.synchronize()
    pipe.check()
    print("pipeline ok")
    torch.cuda.synchronize()
    print("SANITIZE DONE")


if __name__ == "__main__":
    main()
