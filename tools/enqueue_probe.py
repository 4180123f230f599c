"""Host-side cost of ViewPipeline.render: wall time to enqueue the C3 batch vs device time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_14171_b200.pipeline import ViewPipeline
from paper_2503_14171_b200.scenes import CONFIGS, random_views, synthetic_scene
c = CONFIGS["c3"]
sc = synthetic_scene(c.n, c.width, c.height, c.scale_range, seed=5)
views = random_views(1024, c.width, c.height, seed=11)
pipe = ViewPipeline(sc, c.width, c.height, factor=c.factor, slots=4, views_for_capacity=views[:64])
pipe.render(views[:64]); torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter()
    pipe.render(views)
    t1 = time.perf_counter()
    pipe.join(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"enqueue {1e3*(t1-t0):.1f} ms ({1e6*(t1-t0)/len(views):.1f} us/view), total {1e3*(t2-t0):.1f} ms")
