"""Accuracy of the loss adjoint and the train-step gradients vs the reference
goldens (run once per library build: compares SSIM statistic variants)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import golden, scene_of
from test_gpu_backward import FIELDS, rel_err
import paper_2503_14171_b200 as P
from paper_2503_14171_b200 import fit

g = golden("loss")
for lam, v, a in ((0.2, "v02", "a02"), (1.0, "v1", "a1")):
    value, adj = fit.loss(g["pred"], g["target"], lam)
    ref = g[a]
    print(f"loss lam={lam}: value err {abs(value - float(g[v])):.2e}  adjoint rel err "
          f"{np.abs(adj.double().cpu().numpy() - ref).max() / np.abs(ref).max():.2e}")
g = golden("train_step")
sc = scene_of(g)
tgt = torch.from_numpy(g["target"]).float().cuda()
H, W = g["target"].shape[:2]
lw, lh = int(g["low_w"]), int(g["low_h"])
fwd = P.render_forward(sc, lw, lh, train=True)
pred = P.upscale_spline(fwd, 4.0, out_size=(W, H))
value, adj = fit.loss_device(pred, tgt, 0.2)
sadj = P.upscale_backward(fwd, 4.0, adj, out_size=(W, H))
grads = P.render_backward(sc, fwd, P.PixelAdjoint.from_source(sadj)).numpy()
print("train-step grads rel err:", {f: f"{rel_err(grads[f], g[f]):.2e}" for f in FIELDS})
