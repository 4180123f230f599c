"""Host-side cost of ViewPipeline.render: wall time to enqueue a batch small enough for the
launch queues (16 C3 views), per-view ABI calls vs the batched splat_render_views."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_14171_b200.pipeline import ViewPipeline
from paper_2503_14171_b200.scenes import CONFIGS, random_views, synthetic_scene
c = CONFIGS["c3"]
sc = synthetic_scene(c.n, c.width, c.height, c.scale_range, seed=5)
views = random_views(1024, c.width, c.height, seed=11)
pipe = ViewPipeline(sc, c.width, c.height, factor=c.factor, slots=4, views_for_capacity=views[:64])
for batched in (False, True, False, True):
    ViewPipeline.BATCHED = batched
    pipe.render(views[:16]); pipe.join(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe.render(views[:16])
    t1 = time.perf_counter()
    pipe.join(); torch.cuda.synchronize()
    print(f"batched={batched}: enqueue {1e6 * (t1 - t0) / 16:.1f} us/view (16 views, queue not full)")
