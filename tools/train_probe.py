"""Stage timing of one C5 view-step (development aid)."""
import sys; sys.path.insert(0, '.')
import torch
import paper_2503_14171_b200 as P
from paper_2503_14171_b200 import fit
from paper_2503_14171_b200.scenes import CONFIGS, synthetic_scene, random_views
c = CONFIGS["c5"]
model = synthetic_scene(c.n, c.canvas_w, c.canvas_h, c.scale_range, seed=5)
tscene = synthetic_scene(c.n, c.canvas_w, c.canvas_h, c.scale_range, seed=7)
v = random_views(1, c.canvas_w, c.canvas_h, seed=13)[0]
W, H = c.out_size
tgt = P.render_forward(tscene, W, H, view=v).color.clamp(0, 1).contiguous()
ds = P.device.to_device(model)
ev = lambda: torch.cuda.Event(enable_timing=True)
gb = P.GradBuffer(ds.n, ds.device)
def one(report=False):
    e = [ev() for _ in range(8)]
    e[0].record(); fwd = P.render_forward(ds, c.width, c.height, view=v, train=True, sync_check=False)
    e[1].record(); pred = P.upscale_spline(fwd, 1.0, out_size=(W, H))
    e[2].record(); val, adj = fit.loss_device(pred, tgt, 0.2)
    e[3].record(); sadj = P.upscale_backward(fwd, 1.0, adj, out_size=(W, H))
    e[4].record(); P.render_backward(ds, fwd, P.PixelAdjoint.from_source(sadj), out=gb, accumulate=True, check_finite=False)
    e[5].record(); fit.adam_step(fit.scene_params(ds), fit.grads_dict(gb), st, lrs)
    e[6].record(); ds.refresh()
    e[7].record(); torch.cuda.synchronize()
    if report:
        names = ["fwd", "upscale", "loss", "up_bwd", "raster_bwd", "adam", "prepare"]
        print({n: round(e[i].elapsed_time(e[i+1])*1e3, 1) for i, n in enumerate(names)}, "us")
st = fit.AdamState.like(fit.scene_params(ds)); lrs = dict(fit.DEFAULT_LEARNING_RATES)
for i in range(3): one(i == 2)
img = P.render_forward(ds, c.width, c.height, view=v, train=True)
print("stats", img.stats)
