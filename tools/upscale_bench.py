"""Steady-state upscaler throughput (bench.upscale_steady_state) for the C2, C3, C4
shapes; run per variant library with SPLAT_B200_LIB=... to compare kernel shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import upscale_steady_state  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6546.9
torch.cuda.set_device(0)
lib = os.path.basename(os.environ.get("SPLAT_B200_LIB", "libsplat_b200.so"))
for name, (w, h, f) in {"c3": (960, 540, 4), "c4": (1080, 1200, 2), "c2": (960, 540, 2)}.items():
    for nbuf in (1, 4):
        us, by, k = upscale_steady_state(w, h, f * w, f * h, nbuf=nbuf)
        print(f"{lib:28s} {name} nbuf={nbuf} {k:22s} {us:7.2f} us  {by / us / 1e3:7.1f} GB/s  "
              f"{by / us / 1e3 / peak:5.3f} of peak", flush=True)
