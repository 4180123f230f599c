"""File formats either side of the path: scene JSON v1, GIMG gradient dumps,
display-encoded PNG (reference io.py).

Same names, formats and errors as ``splinesplat.io``:

* ``scene_to_dict`` / ``scene_from_dict`` / ``save_scene`` / ``load_scene`` —
  the version-1 JSON scene document (io.py:48-97).  Pure host code: the
  document is text, written with the same ``json.dump(indent=2)`` layout so a
  scene saved here is byte-identical to one saved by the reference.
* ``save_gradient_dump`` / ``load_gradient_dump`` — the "GIMG" file
  (io.py:100-137): 12-byte header + 16 planar float32 planes.  The device
  GradientImage is pixel-interleaved, so the planar body is produced / consumed
  by ``splat_gimg_pack`` / ``splat_gimg_unpack`` on the GPU and crosses PCIe
  once.  A loaded dump has zero ``contrib_count`` and no private state, so
  ``render_backward`` re-renders the view when given one.
* ``encode_display`` / ``decode_display`` / ``write_png`` / ``read_png`` —
  linear [0, 1] <-> 8-bit gamma 2.2 (io.py:28-45); the encode runs on the GPU
  (``splat_encode_display``), PIL does the PNG container on the host.
"""

from __future__ import annotations

import json
import struct

import numpy as np
import torch

from . import _lib
from .core import ParameterError, Scene
from .raster_forward import GradientImage

GAMMA = 2.2
SCENE_VERSION = 1
DUMP_MAGIC = b"GIMG"
DUMP_PLANES = ("color", "d_dx", "d_dy", "d_dxdy", "alpha", "alpha_dx", "alpha_dy", "alpha_dxdy")


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2503_14171_b200 needs a CUDA device (B200, sm_100a)")
    return torch.device("cuda", torch.cuda.current_device())


# ---- display encoding ---------------------------------------------------------------------------

def encode_display(img) -> np.ndarray | torch.Tensor:
    """Linear [0,1] floats to 8-bit gamma-2.2 display values (io.py:28-31).

    A CUDA tensor gives a CUDA uint8 tensor; anything else gives numpy uint8.
    """
    on_dev = torch.is_tensor(img) and img.is_cuda
    t = img if torch.is_tensor(img) else torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32))
    t = t.to(device=_device(), dtype=torch.float32).contiguous()
    out = torch.empty(t.shape, dtype=torch.uint8, device=t.device)
    _lib.check(_lib.load().splat_encode_display(_lib.ptr(t), t.numel(), _lib.ptr(out), _lib.stream_ptr()))
    return out if on_dev else out.cpu().numpy()


def decode_display(raw) -> np.ndarray:
    """8-bit display values to linear float64 (io.py:34-35)."""
    return (np.asarray(raw, dtype=np.float64) / 255.0) ** GAMMA


def write_png(path, img) -> None:
    from PIL import Image
    enc = encode_display(img)
    if torch.is_tensor(enc):
        enc = enc.cpu().numpy()
    Image.fromarray(enc, mode="RGB").save(path, format="PNG")


def read_png(path) -> np.ndarray:
    from PIL import Image
    with Image.open(path) as im:
        raw = np.asarray(im.convert("RGB"))
    return decode_display(raw)


# ---- scene JSON v1 ------------------------------------------------------------------------------

def scene_to_dict(scene) -> dict:
    """Version-1 scene document (io.py:48-65)."""
    sc = scene if isinstance(scene, Scene) else Scene.from_arrays(scene)
    return {
        "version": SCENE_VERSION,
        "reference_resolution": list(sc.reference_resolution),
        "background": [float(v) for v in sc.background],
        "gaussians": [
            {
                "mean": [float(m[0]), float(m[1])],
                "log_scale": [float(s[0]), float(s[1])],
                "rotation": float(r),
                "opacity_logit": float(o),
                "color": [float(c) for c in col],
                "depth": float(d),
            }
            for m, s, r, o, col, d in zip(sc.means, sc.log_scales, sc.rotations, sc.opacity_logits,
                                          sc.colors, sc.depths)
        ],
    }


def scene_from_dict(doc: dict) -> Scene:
    """Parse a version-1 document; ParameterError on a wrong version or non-finite values (io.py:68-87)."""
    if doc.get("version") != SCENE_VERSION:
        raise ParameterError(f"unsupported scene version {doc.get('version')!r}")
    ref = tuple(int(v) for v in doc["reference_resolution"])
    gs = doc["gaussians"]
    n = len(gs)

    def field(key, width):
        a = np.array([g[key] for g in gs], dtype=np.float64)
        return a.reshape(n, width) if width > 1 else a.reshape(n)

    means, log_scales = field("mean", 2), field("log_scale", 2)
    rotations, logits = field("rotation", 1), field("opacity_logit", 1)
    colors, depths = field("color", 3), field("depth", 1)
    background = np.asarray(doc["background"], dtype=np.float64)
    for a in (means, log_scales, rotations, logits, colors, depths, background):
        if not np.all(np.isfinite(a)):
            raise ParameterError("scene file contains non-finite values")
    return Scene(means, log_scales, rotations, logits, colors, depths, background, ref)


def save_scene(path, scene) -> None:
    with open(path, "w") as fh:
        json.dump(scene_to_dict(scene), fh, indent=2)
        fh.write("\n")


def load_scene(path) -> Scene:
    with open(path) as fh:
        return scene_from_dict(json.load(fh))


# ---- GIMG gradient dump -------------------------------------------------------------------------

def gradient_dump_bytes(img: GradientImage) -> bytes:
    """The GIMG file contents for a device GradientImage."""
    w, h = img.width, img.height
    body = torch.empty((16, h, w), dtype=torch.float32, device=img.planes.device)
    if w * h:
        _lib.check(_lib.load().splat_gimg_pack(_lib.ptr(img.planes.contiguous()), _lib.ptr(img.alphas.contiguous()),
                                               w, h, _lib.ptr(body), _lib.stream_ptr()))
    host = body.cpu().numpy()   # native little-endian float32 on x86-64 / aarch64
    return DUMP_MAGIC + struct.pack("<II", w, h) + host.astype("<f4", copy=False).tobytes()


def save_gradient_dump(path, img: GradientImage) -> None:
    """Write a GIMG dump (io.py:110-115)."""
    with open(path, "wb") as fh:
        fh.write(gradient_dump_bytes(img))


def gradient_image_from_dump(blob: bytes, device=None) -> GradientImage:
    if blob[:4] != DUMP_MAGIC:
        raise ParameterError("not a gradient dump (bad magic)")
    w, h = struct.unpack("<II", blob[4:12])
    payload = blob[12:]
    if len(payload) != w * h * 16 * 4:
        raise ParameterError("gradient dump payload has the wrong length")
    dev = device or _device()
    src = torch.from_numpy(np.frombuffer(payload, dtype="<f4").astype(np.float32)).to(dev)
    img = GradientImage.empty(w, h, dev)
    if w * h:
        _lib.check(_lib.load().splat_gimg_unpack(_lib.ptr(src), w, h, _lib.ptr(img.planes), _lib.ptr(img.alphas),
                                                 _lib.ptr(img.contrib_count), _lib.stream_ptr()))
    img.last = None    # no tile lists behind these planes
    return img


def load_gradient_dump(path, device=None) -> GradientImage:
    """Read a GIMG dump (io.py:118-137) into a device GradientImage."""
    with open(path, "rb") as fh:
        return gradient_image_from_dump(fh.read(), device)
