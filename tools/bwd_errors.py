import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import paper_2503_14171_b200 as P
from conftest import golden, golden_names, scene_of
from test_gpu_backward import rel_err, FIELDS
for name in golden_names("bwd_"):
    g = golden(name); sc = scene_of(g)
    w, h = int(g["out_w"]), int(g["out_h"])
    img = P.render_forward(sc, w, h, train=True)
    gr = P.render_backward(sc, img, P.PixelAdjoint.of(g["w"], g["wx"], g["wy"], g["wxy"])).numpy()
    print(name, {f: f"{rel_err(gr[f], g[f]):.1e}" for f in FIELDS},
          'strict', {f: f"{np.max(np.abs(gr[f]-g[f])/np.maximum(np.abs(g[f]),1e-6)):.1e}" for f in FIELDS})
