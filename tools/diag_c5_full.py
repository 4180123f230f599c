"""Diagnose a full-size C5 gradient mismatch: adjoint vs oracle adjoint, and the
rasterizer backward fed with the oracle's own adjoint."""
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_2503_14171_b200 as P
from paper_2503_14171_b200 import fit
from oracle import oracle as O
from paper_2503_14171_b200.scenes import CONFIGS, random_views, synthetic_scene, view_scene
from test_gpu_backward import FIELDS, rel_err
O.build()
c = CONFIGS["c5"]; W, H = c.out_size
sc = synthetic_scene(c.n, c.canvas_w, c.canvas_h, c.scale_range, seed=5)
tsc = synthetic_scene(c.n, c.canvas_w, c.canvas_h, c.scale_range, seed=7)
v = random_views(8, c.canvas_w, c.canvas_h, seed=13)[2]
tgt = P.render_forward(tsc, W, H, view=v).color.clamp(0, 1).contiguous()
img = P.render_forward(sc, c.width, c.height, view=v, train=True)
pred = P.upscale_spline(img, 4.0, out_size=(W, H))
_, adj = fit.loss_device(pred, tgt, 0.2)
sv = view_scene(sc, v)
ref_img = O.render_forward(sv, c.width, c.height)
ref_pred = O.upscale_spline(ref_img.color, ref_img.d_dx, ref_img.d_dy, ref_img.d_dxdy, 4.0, out_size=(W, H))
t64 = tgt.double().cpu().numpy()
_, ref_adj = O.loss(ref_pred, t64, 0.2)
a = adj.double().cpu().numpy()
print("pred err", np.abs(pred.double().cpu().numpy() - ref_pred).max())
d = np.abs(a - ref_adj); print("adj err max", d.max(), "scale", np.abs(ref_adj).max(), "n>1e-3*scale", int((d > 1e-3 * np.abs(ref_adj).max()).sum()))
flip = np.sign(pred.double().cpu().numpy() - t64) != np.sign(ref_pred - t64); print("sign flips", int(flip.sum()))
ref_sadj = O.upscale_backward(c.width, c.height, 4.0, ref_adj, out_size=(W, H))
ref = O.render_backward(sv, ref_img, ref_sadj)
# GPU backward with the oracle's adjoint
g1 = P.render_backward(sc, img, P.PixelAdjoint.of(*[np.asarray(x, np.float32) for x in ref_sadj])).numpy()
for f in FIELDS: print("oracle-adj", f, rel_err(g1[f], ref[f]))
sadj = P.upscale_backward(img, 4.0, adj, out_size=(W, H))
g2 = P.render_backward(sc, img, P.PixelAdjoint.from_source(sadj)).numpy()
for f in FIELDS: print("own-adj", f, rel_err(g2[f], ref[f]))
# the reference's sign(0) and near-zero differences: oracle with the GPU adjoint
ref2 = O.render_backward(sv, ref_img, O.upscale_backward(c.width, c.height, 4.0, a, out_size=(W, H)))
for f in FIELDS: print("oracle with GPU adj", f, rel_err(g2[f], ref2[f]))
