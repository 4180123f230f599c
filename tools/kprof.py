"""Per-kernel device times of the C3 single-view path via torch.profiler (CUPTI
activity records: no replay, no cache flush — unlike ncu's per-launch list)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2503_14171_b200 as P
from paper_2503_14171_b200.scenes import CONFIGS, synthetic_scene, random_views

cname = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
c = CONFIGS[cname]
sc = synthetic_scene(c.n, c.width, c.height, c.scale_range, seed=5)
views = random_views(reps, c.width, c.height, seed=1)
img = P.render_forward(sc, c.width, c.height, view=views[0])
out = torch.empty((int(c.height * c.factor + 0.5), int(c.width * c.factor + 0.5), 3), device="cuda")
for v in views[:3]:
    img = P.render_forward(sc, c.width, c.height, view=v, out=img, sync_check=False)
    P.upscale_spline(img, c.factor, out=out)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for v in views:
        img = P.render_forward(sc, c.width, c.height, view=v, out=img, sync_check=False)
        P.upscale_spline(img, c.factor, out=out)
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    k = e.name[:90]
    t, n = agg.get(k, (0.0, 0))
    agg[k] = (t + e.device_time, n + 1)   # us
tot = sum(t for t, _ in agg.values())
print(f"{'us/view':>9} {'n':>4} {'share':>6}  kernel")
for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{t / reps:9.2f} {n:4d} {100 * t / tot:5.1f}%  {k}")
print(f"{tot / reps:9.2f} total us/view")
