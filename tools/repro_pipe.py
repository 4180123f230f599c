import sys; sys.path.insert(0,'.')
import torch
import paper_2503_14171_b200 as P
from paper_2503_14171_b200.pipeline import ViewPipeline
sc = P.synthetic_scene(30000, 320, 180, (0.5, 2.5), seed=5)
views = P.random_views(5, 320, 180, seed=2)
print("calibrating", flush=True)
pipe = ViewPipeline(sc, 320, 180, factor=4.0, slots=1, views_for_capacity=views)
print("cap", pipe.capacity, flush=True)
outs = pipe.render(views, keep=True); torch.cuda.synchronize(); print("ok")
