"""Synthetic scenes, benchmark configurations and the camera-view model.

The generator mirrors the reference's benchmark scene (splinesplat
``corpus.bench_scene``, corpus.py:88-101) generalised to a W x H canvas, as
SURVEY.md section 8(d) specifies: host numpy PCG64 draws, so the CPU oracle and
the GPU path consume identical float64 parameters.

View model (the reference has none): view v = (zoom z, pan
o).  Rendering view v at W x H is *defined* as the reference's
``render_forward(Scene(means - o, ..., reference_resolution=(W/z, H/z)), W, H)``,
so the oracle for a view is the reference applied to a transformed scene and
the device receives the host-computed doubles kx = W/(W/z), ky = H/(H/z), o.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import Scene, logit

BACKGROUND = (0.12, 0.10, 0.14)   # corpus.py:99


def synthetic_scene(n: int, width: int, height: int, scale_range, seed: int = 5,
                    opacity_range=(0.15, 0.85)) -> Scene:
    """Random scene over a width x height reference canvas (corpus.py:88-101)."""
    rng = np.random.default_rng(seed)
    means = rng.uniform(0.0, 1.0, (n, 2)) * np.array([float(width), float(height)])
    return Scene(
        means=means,
        log_scales=np.log(rng.uniform(scale_range[0], scale_range[1], (n, 2))),
        rotations=rng.uniform(-np.pi, np.pi, n),
        opacity_logits=logit(rng.uniform(opacity_range[0], opacity_range[1], n)),
        colors=rng.uniform(0.0, 1.0, (n, 3)),
        depths=rng.uniform(0.0, 1.0, n),
        background=np.array(BACKGROUND),
        reference_resolution=(width, height),
    )


@dataclass(frozen=True)
class View:
    """A camera view: zoom z >= 1 about the pan offset (ox, oy) in reference pixels."""

    zoom: float = 1.0
    ox: float = 0.0
    oy: float = 0.0

    def reference_resolution(self, canvas_w: float, canvas_h: float):
        """Reference resolution of the view scene: the zoomed window of the canvas."""
        return (canvas_w / self.zoom, canvas_h / self.zoom)

    def scales(self, canvas_w: float, canvas_h: float, out_w: int, out_h: int):
        """(kx, ky) exactly as prepare_scene computes them for the view scene
        (raster_forward.py:81-85: kx = out_w / ref_w)."""
        ref_w, ref_h = self.reference_resolution(canvas_w, canvas_h)
        return out_w / ref_w, out_h / ref_h


def view_scene(scene: Scene, view: View) -> Scene:
    """The reference-side scene whose plain render *is* this view (oracle input)."""
    cw, ch = scene.reference_resolution
    return Scene(scene.means - np.array([view.ox, view.oy]), scene.log_scales,
                 scene.rotations, scene.opacity_logits, scene.colors, scene.depths,
                 scene.background, view.reference_resolution(cw, ch))


def random_views(n_views: int, width: int, height: int, seed: int = 11,
                 zoom_range=(1.0, 1.25)):
    """Seeded views whose window stays on the canvas."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_views):
        z = float(rng.uniform(*zoom_range))
        ox = float(rng.uniform(0.0, width - width / z))
        oy = float(rng.uniform(0.0, height - height / z))
        out.append(View(z, ox, oy))
    return out


def stereo_views(n_frames: int, width: int, height: int, disparity: float = 3.0, seed: int = 11,
                 zoom_range=(1.0, 1.25)):
    """Config 4: per frame a left/right eye pair — one seeded view panned by
    -/+ disparity/2 reference pixels (SURVEY.md 8(d) "stereo pair = 2 views")."""
    out = []
    for v in random_views(n_frames, width, height, seed=seed, zoom_range=zoom_range):
        ox = min(max(v.ox, disparity / 2), width - width / v.zoom - disparity / 2)
        out.append(View(v.zoom, ox - disparity / 2, v.oy))
        out.append(View(v.zoom, ox + disparity / 2, v.oy))
    return out


@dataclass(frozen=True)
class BenchConfig:
    """BASELINE.json configs, sizes from SURVEY.md 8(d)."""

    name: str
    n: int
    width: int          # render width
    height: int         # render height
    factor: float
    scale_range: tuple  # splat std-dev range in canvas pixels
    views: int = 1
    out_size: tuple | None = None
    canvas: tuple | None = None   # scene reference resolution (defaults to render size)

    @property
    def canvas_w(self) -> int:
        return self.canvas[0] if self.canvas else self.width

    @property
    def canvas_h(self) -> int:
        return self.canvas[1] if self.canvas else self.height

    @property
    def out_w(self) -> int:
        return self.out_size[0] if self.out_size else int(np.floor(self.width * self.factor + 0.5))

    @property
    def out_h(self) -> int:
        return self.out_size[1] if self.out_size else int(np.floor(self.height * self.factor + 0.5))


CONFIGS = {
    "c1": BenchConfig("c1", 10_000, 128, 128, 2.0, (1.28, 6.4)),
    "c2": BenchConfig("c2", 200_000, 960, 540, 2.0, (1.0, 4.0)),
    "c3": BenchConfig("c3", 1_000_000, 960, 540, 4.0, (0.5, 2.5), views=1024),
    "c4": BenchConfig("c4", 3_000_000, 1080, 1200, 2.0, (0.5, 2.5), views=2),
    # training: reference canvas 1920x1080 with 2-10 px splats, rendered at 480x270
    "c5": BenchConfig("c5", 1_000_000, 480, 270, 4.0, (2.0, 10.0), views=8,
                      out_size=(1920, 1080), canvas=(1920, 1080)),
}
