"""Wire formats against the reference's own files
(tests/golden/io.npz, written by splinesplat.io in make_golden.py).

CPU: the scene JSON document is byte-identical to the reference's and its
error cases raise the reference's exceptions.  GPU: GIMG dumps written here
have the reference's header and plane order; the reference's dump loads into
exactly its float32 values and upscales like the reference's re-loaded dump;
display encoding matches numpy bit for bit.
"""

import json
import struct

import numpy as np
import pytest

from conftest import golden, scene_of


def test_scene_json_is_byte_identical_to_reference(tmp_path):
    from paper_2503_14171_b200 import io as sio
    g = golden("io")
    sc = scene_of(g)
    path = tmp_path / "s.json"
    sio.save_scene(path, sc)
    assert path.read_bytes() == g["scene_json"].tobytes()
    back = sio.load_scene(path)
    for f in ("means", "log_scales", "rotations", "opacity_logits", "colors", "depths", "background"):
        assert np.array_equal(getattr(back, f), getattr(sc, f))
    assert tuple(back.reference_resolution) == tuple(sc.reference_resolution)


def test_scene_json_errors():
    from paper_2503_14171_b200 import io as sio
    from paper_2503_14171_b200.core import ParameterError
    doc = json.loads(golden("io")["scene_json"].tobytes())
    bad = dict(doc, version=2)
    with pytest.raises(ParameterError):
        sio.scene_from_dict(bad)
    bad = json.loads(json.dumps(doc))
    bad["gaussians"][3]["depth"] = float("nan")
    with pytest.raises(ParameterError):
        sio.scene_from_dict(bad)
    empty = dict(doc, gaussians=[])
    assert sio.scene_from_dict(empty).n == 0


def test_decode_display_matches_reference_formula():
    from paper_2503_14171_b200 import io as sio
    raw = np.arange(256, dtype=np.uint8)
    assert np.array_equal(sio.decode_display(raw), (raw.astype(np.float64) / 255.0) ** 2.2)


def test_gimg_header_errors():
    from paper_2503_14171_b200 import io as sio
    from paper_2503_14171_b200.core import ParameterError
    blob = golden("io")["gimg"].tobytes()
    with pytest.raises(ParameterError):
        sio.gradient_image_from_dump(b"GIMX" + blob[4:])
    with pytest.raises(ParameterError):
        sio.gradient_image_from_dump(blob[:-4])


@pytest.mark.gpu
def test_load_reference_dump_and_upscale():
    import torch
    from paper_2503_14171_b200 import io as sio
    import paper_2503_14171_b200 as P
    g = golden("io")
    blob = g["gimg"].tobytes()
    w, h = struct.unpack("<II", blob[4:12])
    img = sio.gradient_image_from_dump(blob)
    planes = np.frombuffer(blob[12:], dtype="<f4").reshape(16, h, w)
    got = img.numpy()
    for k, f in enumerate(("color", "d_dx", "d_dy", "d_dxdy")):
        assert np.array_equal(np.moveaxis(planes[3 * k:3 * k + 3], 0, 2), got[f].astype(np.float32))
    for k, f in enumerate(("alpha", "alpha_dx", "alpha_dy", "alpha_dxdy")):
        assert np.array_equal(planes[12 + k], got[f].astype(np.float32))
    assert int(got["contrib_count"].max()) == 0
    up = P.upscale_spline(img, 2.0).cpu().numpy()
    assert np.abs(up - g["up"]).max() < 1e-5
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_dump_matches_reference_layout_and_round_trips():
    from paper_2503_14171_b200 import io as sio
    import paper_2503_14171_b200 as P
    g = golden("io")
    sc = scene_of(g)
    w, h = int(g["out_w"]), int(g["out_h"])
    img = P.render_forward(sc, w, h)
    blob = sio.gradient_dump_bytes(img)
    ref = g["gimg"].tobytes()
    assert blob[:12] == ref[:12] and len(blob) == len(ref)
    a = np.frombuffer(blob[12:], dtype="<f4")
    b = np.frombuffer(ref[12:], dtype="<f4")
    assert np.abs(a.astype(np.float64) - b).max() < 1e-4
    back = sio.gradient_image_from_dump(blob)
    assert sio.gradient_dump_bytes(back) == blob


@pytest.mark.gpu
def test_backward_from_loaded_dump_rerenders():
    """A dump has no private float64 state: render_backward re-renders the view
    and gives the same gradients as from the live forward image."""
    import torch
    from paper_2503_14171_b200 import io as sio
    import paper_2503_14171_b200 as P
    g = golden("io")
    sc = scene_of(g)
    w, h = int(g["out_w"]), int(g["out_h"])
    fwd = P.render_forward(sc, w, h, train=True)
    loaded = sio.gradient_image_from_dump(sio.gradient_dump_bytes(fwd))
    rng = np.random.default_rng(1)
    adj = P.PixelAdjoint.of(*(rng.normal(size=(h, w, 3)) for _ in range(4)))
    a = P.render_backward(sc, fwd, adj)
    b = P.render_backward(sc, loaded, adj)
    for f in ("d_means", "d_log_scales", "d_rotations", "d_opacity_logits", "d_colors"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.gpu
def test_encode_display_matches_numpy():
    import torch
    from paper_2503_14171_b200 import io as sio
    g = golden("io")
    got = sio.encode_display(g["enc_in"])
    assert got.dtype == np.uint8
    assert np.array_equal(got, g["enc_out"])
    dev = sio.encode_display(torch.from_numpy(g["enc_in"]).cuda())
    assert dev.is_cuda and np.array_equal(dev.cpu().numpy(), g["enc_out"])
