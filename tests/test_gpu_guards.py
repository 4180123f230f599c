"""Out-of-bounds write detection without compute-sanitizer (closed on this pool):
every device buffer a kernel family writes -- frame workspace, GradientImage planes,
upscaled frames, adjoints, gradient buffers, loss workspace -- is placed between
canary regions that must be bit-for-bit intact after the run, on ragged sizes
(partial tiles, odd widths, 1-pixel images) where an off-by-one would land in a
canary.  The same tests run against the checked build (libsplat_b200_checked.so,
device-side SPLAT_DCHECK bounds and protocol checks) via SPLAT_B200_LIB."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = 4096            # canary bytes either side
CANARY = 0x5A


class Guarded:
    """A tensor view with canary bytes before and after it."""

    def __init__(self, shape, dtype):
        import torch
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        self.buf = torch.full((n + 2 * G,), CANARY, dtype=torch.uint8, device="cuda")
        self.n = n
        self.t = self.buf[G:G + n].view(dtype).view(shape)

    def intact(self):
        return bool((self.buf[:G] == CANARY).all()) and bool((self.buf[G + self.n:] == CANARY).all())


def guarded_image(w, h, train):
    import torch
    from paper_2503_14171_b200.raster_forward import GradientImage
    parts = {"planes": Guarded((h, w, 4, 3), torch.float32), "alphas": Guarded((4, h, w), torch.float32),
             "contrib_count": Guarded((h, w), torch.int32), "last": Guarded((h, w), torch.int32)}
    if train:
        parts["state"] = Guarded((h, w, 4), torch.float64)
    img = GradientImage(**{k: v.t for k, v in parts.items()})
    return img, parts


@pytest.mark.parametrize("w,h,train", [(97, 53, False), (97, 53, True), (1, 1, False), (16, 16, True),
                                       (250, 3, False), (33, 130, True)])
def test_forward_and_backward_write_only_their_buffers(w, h, train):
    import torch
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200.raster_backward import GradBuffer, PixelAdjoint, render_backward
    from paper_2503_14171_b200.raster_forward import Frame
    sc = P.synthetic_scene(4000, w, h, (0.5, 6.0), seed=w + h)
    ref = P.render_forward(sc, w, h, train=train)
    frame = Frame(sc.n, w, h, ref.frame.capacity, torch.device("cuda"), guard=G)
    img, parts = guarded_image(w, h, train)
    out = P.render_forward(sc, w, h, train=train, out=img, frame=frame, sync_check=False)
    torch.cuda.synchronize()
    assert frame.guards_intact(), "frame workspace canary overwritten"
    for k, g in parts.items():
        assert g.intact(), f"{k} canary overwritten"
    assert torch.equal(out.planes, ref.planes) and torch.equal(out.contrib_count, ref.contrib_count)
    if train:
        rng = np.random.default_rng(1)
        adj = PixelAdjoint.of(*(rng.normal(0, 1e-3, (h, w, 3)) for _ in range(4)))
        gb = GradBuffer(sc.n, torch.device("cuda"))
        gflat = Guarded(tuple(gb.flat.shape), torch.float32)
        gb.flat = gflat.t
        render_backward(sc, out, adj, out=gb)
        torch.cuda.synchronize()
        assert gflat.intact() and frame.guards_intact()
        refg = render_backward(sc, ref, adj)
        assert torch.equal(gb.grads().d_means, refg.d_means)


@pytest.mark.parametrize("w,h,factor", [(37, 23, 4.0), (38, 23, 2.0), (37, 23, 2.0), (5, 3, 2.5), (1, 1, 4.0),
                                        (130, 70, 4.0)])
def test_upscale_forward_and_backward_write_only_their_buffers(w, h, factor):
    import torch
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200.spline import output_size
    ow, oh = output_size(w, h, factor)
    src = Guarded((h, w, 4, 3), torch.float32)
    src.t.copy_(torch.rand((h, w, 4, 3), device="cuda"))
    img = P.GradientImage(planes=src.t, alphas=torch.zeros((4, h, w), device="cuda"),
                          contrib_count=torch.zeros((h, w), dtype=torch.int32, device="cuda"))
    out = Guarded((oh, ow, 3), torch.float32)
    P.upscale_spline(img, factor, out=out.t)
    dsrc = Guarded((h, w, 4, 3), torch.float32)
    adj = torch.randn((oh, ow, 3), device="cuda")
    P.upscale_backward(img, factor, adj, out=dsrc.t)
    torch.cuda.synchronize()
    assert src.intact() and out.intact() and dsrc.intact()
    assert torch.equal(out.t, P.upscale_spline(img, factor))
    assert torch.equal(dsrc.t, P.upscale_backward(img, factor, adj).planes)


@pytest.mark.parametrize("w,h", [(16, 16), (97, 61), (1920, 1080)])
def test_loss_writes_only_its_buffers(w, h):
    import torch
    from paper_2503_14171_b200 import fit
    pred, tgt = torch.rand((h, w, 3), device="cuda"), torch.rand((h, w, 3), device="cuda")
    adj = Guarded((h, w, 3), torch.float32)
    val = Guarded((2,), torch.float64)
    fit.loss_device(pred, tgt, 0.2, adj=adj.t, value=val.t, slot=7)
    torch.cuda.synchronize()
    assert adj.intact() and val.intact()
    v2, a2 = fit.loss_device(pred, tgt, 0.2, slot=8)
    assert torch.equal(adj.t, a2) and torch.equal(val.t, v2)


def test_abi_rejects_misaligned_buffers():
    """The bulk-copy (TMA) paths need aligned buffers: the C ABI refuses a frame workspace
    that is not 256-byte aligned and upscale planes / frames that are not 16-byte aligned
    (status 2 = ParameterError) instead of faulting."""
    import torch
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200 import _lib
    from paper_2503_14171_b200.core import ParameterError
    from paper_2503_14171_b200.device import to_device
    from paper_2503_14171_b200.raster_forward import Frame, make_view
    lib = _lib.load()
    sc = P.synthetic_scene(500, 64, 48, (0.5, 3.0), seed=2)
    ds = to_device(sc)
    fr = Frame(ds.n, 64, 48, 1 << 16, torch.device("cuda"))
    big = torch.empty(fr.nbytes + 256, dtype=torch.uint8, device="cuda")
    v = make_view(ds, 64, 48)
    rc = lib.splat_prepare_view(_lib.ptr(ds.const), ds.n, v, 64, 48, big.data_ptr() + 16, fr.nbytes, fr.capacity,
                                _lib.stream_ptr())
    assert rc == _lib.SPLAT_ERR_PARAMETER
    with pytest.raises(ParameterError):
        _lib.check(rc)
    src = torch.zeros(48 * 64 * 12 + 4, device="cuda")
    out = torch.zeros(96 * 128 * 3 + 4, device="cuda")
    from paper_2503_14171_b200.spline import upscale_plan
    plan = upscale_plan(64, 48, 128, 96, torch.device("cuda"))
    assert lib.splat_upscale_forward(src.data_ptr() + 4, 64, 48, out.data_ptr(), 128, 96, 1, _lib.ptr(plan),
                                     _lib.stream_ptr()) == _lib.SPLAT_ERR_PARAMETER
    assert lib.splat_upscale_forward(src.data_ptr(), 64, 48, out.data_ptr() + 4, 128, 96, 1, _lib.ptr(plan),
                                     _lib.stream_ptr()) == _lib.SPLAT_ERR_PARAMETER
    assert lib.splat_upscale_forward(src.data_ptr(), 64, 48, out.data_ptr(), 128, 96, 1, _lib.ptr(plan),
                                     _lib.stream_ptr()) == 0
