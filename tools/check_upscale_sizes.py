import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2503_14171_b200 as P
from oracle import oracle as O
for (w, h) in [(960, 540), (1080, 540), (960, 1200), (1080, 1200), (200, 1200), (1080, 64)]:
    rng = np.random.default_rng(w * 1000 + h)
    planes = [rng.uniform(0, 1, (h, w, 3))] + [rng.normal(0, 0.3, (h, w, 3)) for _ in range(3)]
    img = P.GradientImage.from_planes(*planes)
    f32 = [np.asarray(x, dtype=np.float32).astype(np.float64) for x in planes]
    ref = O.upscale_spline(*f32, 2.0, clamp=False)
    for rep in range(3):
        got = P.upscale_spline(img, 2.0, clamp=False).cpu().numpy()
        d = np.abs(got - ref)
        bad = np.argwhere(d > 1e-4)
        print(w, h, rep, d.max(), len(bad), (bad[:, 0].min(), bad[:, 0].max(), bad[:, 1].min(), bad[:, 1].max()) if len(bad) else "")
