"""Quick timing probe of one C3/C2 view (development aid, not the bench)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2503_14171_b200 as P
from paper_2503_14171_b200.scenes import CONFIGS, synthetic_scene
from paper_2503_14171_b200 import _lib

def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

for cname in sys.argv[1:] or ["c2", "c3"]:
    c = CONFIGS[cname]
    t0 = time.time()
    sc = synthetic_scene(c.n, c.width, c.height, c.scale_range, seed=5)
    ds = P.device.to_device(sc) if hasattr(P, 'device') else None
    torch.cuda.synchronize()
    print(cname, "gen+upload+prepare", time.time() - t0)
    img = P.render_forward(sc, c.width, c.height)
    torch.cuda.synchronize()
    print(cname, "stats", img.stats)
    frame = img.frame
    lib = _lib.load()
    v = img.view
    st = _lib.stream_ptr()
    def fwd():
        _lib.check(lib.splat_render_forward(_lib.ptr(img.scene.const), img.scene.n, v, c.width, c.height, 0,
                   img.c_gimg(), _lib.ptr(frame.ws), frame.nbytes, frame.capacity, 0, st))
    def prep():
        _lib.check(lib.splat_prepare_view(_lib.ptr(img.scene.const), img.scene.n, v, c.width, c.height,
                   _lib.ptr(frame.ws), frame.nbytes, frame.capacity, 0, st))
    def binning():
        _lib.check(lib.splat_bin_tiles(img.scene.n, c.width, c.height, _lib.ptr(frame.ws), frame.nbytes, frame.capacity, 0, st))
    out = torch.empty((c.out_h, c.out_w, 3), device='cuda')
    def up():
        P.upscale_spline(img, c.factor, out=out)
    print(cname, "fwd ms", timeit(fwd), "prep ms", timeit(prep), "bin ms", timeit(binning), "up ms", timeit(up))
    ub = c.out_w * c.out_h * 12 + c.width * c.height * 48
    print(cname, "upscale GB/s", ub / (timeit(up) * 1e-3) / 1e9)
