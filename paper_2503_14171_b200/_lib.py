"""ctypes binding of libsplat_b200.so (the C ABI in include/splat_b200.h).

The library is the only compute path: if it is missing or cannot be loaded,
every entry point raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

from .core import DimensionError, ParameterError, UnsupportedScaleError

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPLAT_B200_LIB selects an alternative in-tree build (kernel tuning experiments)
LIB_PATH = os.environ.get("SPLAT_B200_LIB", os.path.join(_HERE, "libsplat_b200.so"))

P = ctypes.c_void_p
I32 = ctypes.c_int
I64 = ctypes.c_int64
SZ = ctypes.c_size_t
D = ctypes.c_double

SPLAT_OK = 0
SPLAT_ERR_DIMENSION = 1
SPLAT_ERR_PARAMETER = 2
SPLAT_ERR_SCALE = 3
SPLAT_ERR_CAPACITY = 4
SPLAT_ERR_CUDA = 100


class SceneT(ctypes.Structure):
    _fields_ = [("n", I64), ("means", P), ("log_scales", P), ("rotations", P),
                ("opacity_logits", P), ("colors", P), ("depths", P)]


class ViewT(ctypes.Structure):
    _fields_ = [("kx", D), ("ky", D), ("ox", D), ("oy", D), ("bg", D * 3)]


class CameraT(ctypes.Structure):
    _fields_ = [("R", D * 9), ("t", D * 3), ("fx", D), ("fy", D), ("cx", D), ("cy", D), ("near_plane", D)]


class GimgT(ctypes.Structure):
    _fields_ = [("planes", P), ("alpha", P), ("count", P), ("last", P), ("state", P)]


class SlotT(ctypes.Structure):
    _fields_ = [("workspace", P), ("ws_bytes", SZ), ("pair_capacity", I64), ("image", GimgT), ("stream", P)]


class FramePtrsT(ctypes.Structure):
    _fields_ = [("bboxes", P), ("touched", P), ("offsets", P), ("keys", P), ("ranks", P),
                ("ranges", P), ("counters", P), ("fixup", P), ("pack", P)]


# name -> (restype, argtypes); mirrors include/splat_b200.h one to one
SIGNATURES = {
    "splat_last_error": (ctypes.c_char_p, []),
    "splat_abi_version": (I32, []),
    "splat_kernel_launches": (ctypes.c_uint64, []),
    "splat_build_checked": (I32, []),
    "splat_scene_const_bytes": (SZ, [I64]),
    "splat_scene_workspace_bytes": (SZ, [I64]),
    "splat_scene_prepare": (I32, [ctypes.POINTER(SceneT), P, SZ, P, SZ, P]),
    "splat_scene_refresh": (I32, [ctypes.POINTER(SceneT), P, SZ, P]),
    "splat_scene_order": (P, [P, I64]),
    "splat_frame_workspace_bytes": (SZ, [I64, I32, I32, I64]),
    "splat_frame_pointers": (I32, [P, I64, I32, I32, I64, ctypes.POINTER(FramePtrsT)]),
    "splat_render_forward": (I32, [P, I64, ctypes.POINTER(ViewT), I32, I32, I32,
                                   ctypes.POINTER(GimgT), P, SZ, I64, P]),
    "splat_prepare_view": (I32, [P, I64, ctypes.POINTER(ViewT), I32, I32, P, SZ, I64, P]),
    "splat_bin_tiles": (I32, [I64, I32, I32, P, SZ, I64, I32, P]),
    "splat_gimg_pack": (I32, [P, P, I32, I32, P, P]),
    "splat_gimg_unpack": (I32, [P, I32, I32, P, P, P, P]),
    "splat_encode_display": (I32, [P, I64, P, P]),
    "splat_grad_accumulate": (I32, [P, P, I64, P]),
    "splat_render_points": (I32, [P, P, P, I64, P, P, I64, ctypes.POINTER(D), P, P, P]),
    "splat_project_3d": (I32, [I64, P, P, P, P, ctypes.POINTER(CameraT), P, P, P, P, P, P]),
    "splat_render_views": (I32, [P, I64, ctypes.POINTER(ViewT), I32, I32, I32, ctypes.POINTER(SlotT), I32,
                                 ctypes.POINTER(P), I32, I32, I32, P]),
    "splat_fixup": (I32, [P, I64, ctypes.POINTER(ViewT), I32, I32, I32, ctypes.POINTER(GimgT), P, SZ, I64, P]),
    "splat_rasterize": (I32, [P, I64, ctypes.POINTER(ViewT), I32, I32, I32,
                              ctypes.POINTER(GimgT), P, SZ, I64, P]),
    "splat_view_pack64": (I32, [P, I64, ctypes.POINTER(ViewT), P, P]),
    "splat_backward_workspace_bytes": (SZ, [I64, I64]),
    "splat_render_backward": (I32, [P, ctypes.POINTER(SceneT), ctypes.POINTER(ViewT), I32, I32,
                                    ctypes.POINTER(GimgT), P, P, SZ, I64, P, SZ, P, I32, P]),
    "splat_render_backward_rank": (I32, [P, ctypes.POINTER(SceneT), ctypes.POINTER(ViewT), I32, I32,
                                         ctypes.POINTER(GimgT), P, P, SZ, I64, P, SZ, P, I32, P]),
    "splat_chain_grads": (I32, [P, ctypes.POINTER(SceneT), P, P, I32, P]),
    "splat_loss_workspace_bytes": (SZ, [I32, I32]),
    "splat_loss": (I32, [P, P, I32, I32, D, P, P, P, SZ, P]),
    "splat_adam_step": (I32, [P, P, P, P, I64, D, D, D, D, D, D, P]),
    "splat_adam_step_groups": (I32, [I32, P, P, P, P, P, P, D, D, D, D, D, P]),
    "splat_upscale_plan_bytes": (SZ, [I32, I32, I32, I32]),
    "splat_upscale_plan": (I32, [I32, I32, I32, I32, P, P]),
    "splat_upscale_forward": (I32, [P, I32, I32, P, I32, I32, I32, P, P]),
    "splat_upscale_backward": (I32, [P, I32, I32, P, I32, I32, P]),
    "splat_fd_gradients": (I32, [P, I32, I32, P, P]),
    "splat_fd_gradients_backward": (I32, [P, I32, I32, P, P, P]),
}

_lib = None


def load():
    """Load the in-tree library (raises if absent: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the CUDA library is the only implementation of this path)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    """Map C ABI status codes onto the reference exception classes."""
    if rc == SPLAT_OK:
        return
    msg = load().splat_last_error().decode(errors="replace")
    if rc == SPLAT_ERR_DIMENSION:
        raise DimensionError(msg)
    if rc == SPLAT_ERR_PARAMETER:
        raise ParameterError(msg)
    if rc == SPLAT_ERR_SCALE:
        raise UnsupportedScaleError(msg)
    raise RuntimeError(f"libsplat_b200 error {rc}: {msg}")


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)
