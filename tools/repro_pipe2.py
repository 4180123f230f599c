import sys; sys.path.insert(0,'.')
import torch
import paper_2503_14171_b200 as P
from paper_2503_14171_b200.pipeline import ViewPipeline
sc = P.synthetic_scene(30000, 320, 180, (0.5, 2.5), seed=5)
views = P.random_views(5, 320, 180, seed=2)
for slots in (1, 3):
    print("slots", slots, flush=True)
    pipe = ViewPipeline(sc, 320, 180, factor=4.0, slots=slots, views_for_capacity=views)
    torch.cuda.synchronize(); print("calibrated", pipe.capacity, flush=True)
    outs = pipe.render(views, keep=True)
    pipe.join()
    torch.cuda.synchronize(); print("rendered", flush=True)
    pipe.check()
    for v, got in zip(views, outs):
        ref = P.upscale_spline(P.render_forward(sc, 320, 180, view=v), 4.0)
        torch.cuda.synchronize()
        print(torch.equal(got, ref), flush=True)
