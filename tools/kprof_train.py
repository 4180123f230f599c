"""Per-kernel device times of the C5 training step via torch.profiler (CUPTI)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2503_14171_b200 import fit
from paper_2503_14171_b200.raster_forward import render_forward
from paper_2503_14171_b200.scenes import CONFIGS, random_views, synthetic_scene

vpr = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
streams = int(sys.argv[3]) if len(sys.argv) > 3 else 2
c = CONFIGS["c5"]
model = synthetic_scene(c.n, c.canvas_w, c.canvas_h, c.scale_range, seed=5)
target = synthetic_scene(c.n, c.canvas_w, c.canvas_h, c.scale_range, seed=7)
views = random_views(vpr, c.canvas_w, c.canvas_h, seed=13)
W, H = c.out_size
targets = [render_forward(target, W, H, view=v).color.clamp(0.0, 1.0).contiguous() for v in views]
tr = fit.ViewTrainer(model, (c.width, c.height), (W, H), views, targets, ssim_weight=0.2, streams=streams)
for _ in range(2):
    tr.step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        tr.step()
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    k = e.name[:90]
    t, n = agg.get(k, (0.0, 0))
    agg[k] = (t + e.device_time, n + 1)
nv = vpr * steps
tot = sum(t for t, _ in agg.values())
print(f"{'us/view':>9} {'n':>4} {'share':>6}  kernel")
for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{t / nv:9.2f} {n:4d} {100 * t / tot:5.1f}%  {k}")
print(f"{tot / nv:9.2f} total kernel us/view-step")
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
for _ in range(steps):
    tr.step()
s1.record()
torch.cuda.synchronize()
print(f"streams {streams}: {s0.elapsed_time(s1) * 1e3 / nv:9.2f} wall us/view-step")
