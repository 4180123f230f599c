"""Work statistics of the forward rasterizer (build with -DRASTER_STATS=1):
chunks, blend steps, group-list entries, lane evaluations vs contributors."""
import os, sys
import torch
sys.path.insert(0, '.')
import paper_2503_14171_b200 as P
from paper_2503_14171_b200.scenes import CONFIGS, random_views, synthetic_scene

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
sc = synthetic_scene(c.n, c.width, c.height, c.scale_range, seed=5)
v = random_views(1, c.width, c.height, seed=11)[0]
img = P.render_forward(sc, c.width, c.height, view=v)
ctr = img.frame.counters()
ctr[8:].zero_()
img = P.render_forward(sc, c.width, c.height, view=v, out=img, sync_check=False)
torch.cuda.synchronize()
ctr = img.frame.counters().cpu().numpy().view("uint64")
chunks, steps, entries, evals, dead, conlanes = (int(x) for x in ctr[4:10])
K = int(img.contrib_count.sum(dtype=torch.int64))
print(f"chunks {chunks}  steps {steps} ({steps / chunks:.2f}/chunk)  group entries {entries} "
      f"({entries / max(steps, 1):.2f} of 4 groups busy per step)")
print(f"lane-steps {steps * 32}  lane evals {evals} ({evals / (steps * 32):.1%} of lane-steps)  "
      f"contributors K {K} ({K / evals:.1%} of evals, {K / (steps * 32):.1%} of lane-steps)")
print(f"steps with evaluations but no contributor: {dead} ({dead / max(steps, 1):.1%} of steps); "
      f"contributing lanes per live step {conlanes / max(steps - dead, 1):.1f}")
