"""Pipeline rate when every view is the same (so a timing-only build that reuses a
frame's first tile lists renders the same work): stage marginal costs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_14171_b200.pipeline import ViewPipeline
from paper_2503_14171_b200.scenes import CONFIGS, random_views, synthetic_scene
c = CONFIGS["c3"]
sc = synthetic_scene(c.n, c.width, c.height, c.scale_range, seed=5)
v = random_views(16, c.width, c.height, seed=11)[7]
views = [v] * 256
pipe = ViewPipeline(sc, c.width, c.height, factor=c.factor, slots=4, views_for_capacity=[v])
pipe.render(views[:16]); pipe.join(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); pipe.render(views); pipe.join(); e1.record(); torch.cuda.synchronize()
lib = os.path.basename(os.environ.get("SPLAT_B200_LIB", "libsplat_b200.so"))
print(f"{lib}: {len(views) / (e0.elapsed_time(e1) / 1e3):.1f} frames/s (one view x {len(views)})")
