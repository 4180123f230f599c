import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch
import paper_2503_14171_b200 as P
from paper_2503_14171_b200 import fit
from conftest import golden, scene_of
from test_gpu_backward import FIELDS, rel_err
from oracle import oracle as O
g = golden("train_step"); sc = scene_of(g)
tgt = torch.from_numpy(g["target"]).float().cuda()
H, W = g["target"].shape[:2]; lw, lh = int(g["low_w"]), int(g["low_h"])
fwd = P.render_forward(sc, lw, lh, train=True)
pred = P.upscale_spline(fwd, 4.0, out_size=(W, H))
value, adj = fit.loss_device(pred, tgt, 0.2)
a = adj.double().cpu().numpy(); r = g["dpred"]
print("adj err max/absmax", np.abs(a-r).max()/np.abs(r).max(), "n sign-ish diffs", int((np.abs(a-r) > 1e-3*np.abs(r).max()).sum()))
for name, A in (("gpu_adj", adj), ("golden_adj", torch.from_numpy(r).float().cuda())):
    sadj = P.upscale_backward(fwd, 4.0, A, out_size=(W, H))
    gr = P.render_backward(sc, fwd, P.PixelAdjoint.from_source(sadj)).numpy()
    print(name, {f: f"{rel_err(gr[f], g[f]):.2e}" for f in FIELDS})
# oracle with fp32-rounded golden adjoint
ofwd = O.render_forward(sc, lw, lh)
for name, A in (("oracle_golden_adj", r), ("oracle_gpu_adj", a)):
    sadj = O.upscale_backward(lw, lh, 4.0, A, out_size=(W, H))
    og = O.render_backward(sc, ofwd, sadj)
    print(name, {f: f"{rel_err(og[f], g[f]):.2e}" for f in FIELDS})
