"""B200-native gradient-aware splat render + spline upscale path.

Drop-in for the hot path of the reference package ``splinesplat``
(render_forward / upscale_spline / upscale_backward / render_backward and the
inspectable stages sort_by_depth / prepare_scene / bin_tiles), computed by
hand-written sm_100a CUDA kernels in libsplat_b200.so behind a C ABI
(include/splat_b200.h).  There is no CPU fallback.
"""

from .core import (ALPHA_CLAMP, ALPHA_CULL, EARLY_TERMINATION, DegenerateCovarianceError,
                   DimensionError, Gaussian2D, ParameterError, Scene, UnsupportedScaleError, logistic,
                   logit)
from .raster_forward import (GradientImage, RenderPack, bin_tiles, prepare_scene, render_at_points,
                             render_forward, sort_by_depth, tile_grid)
from .raster_backward import (GradBuffer, PixelAdjoint, SceneGrads, invert_alpha_state,
                              render_backward)
from .scenes import View, random_views, synthetic_scene, view_scene
from .spline import (SourceAdjoint, fd_gradients, fd_gradients_backward, upscale_backward,
                     upscale_spline)

__version__ = "0.1.0"

__all__ = [
    "ALPHA_CLAMP", "ALPHA_CULL", "EARLY_TERMINATION", "DegenerateCovarianceError", "DimensionError",
    "ParameterError", "Scene", "Gaussian2D", "UnsupportedScaleError", "logistic", "logit", "GradientImage",
    "RenderPack", "bin_tiles", "prepare_scene", "render_at_points", "render_forward", "sort_by_depth",
    "tile_grid",
    "GradBuffer", "PixelAdjoint", "SceneGrads", "invert_alpha_state", "render_backward",
    "View", "random_views", "synthetic_scene", "view_scene", "SourceAdjoint", "fd_gradients",
    "fd_gradients_backward", "upscale_backward", "upscale_spline",
]
