#!/usr/bin/env python
"""Benchmark: upscaled 4K frames/s (x4 spline upscale) on a 1024-view batch.

Workload (BASELINE.json configs[2], SURVEY.md 8(d) "C3"): synthetic 1M-splat
scene, 960x540 render with analytic gradients, x4 gradient-aware spline
upscale to 3840x2160, 1024 seeded camera views sharded over the ranks (one
process per GPU, no data-path collective; strong scaling of the fixed batch).
A step renders + upscales every view of this rank's shard.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
        torchrun --nproc-per-node N bench.py --gpus N ...

Without torchrun, ``--gpus N`` (N > 1) launches the N ranks itself through
torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1); under
torchrun, a WORLD_SIZE different from --gpus is refused.

Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "upscaled frames/s (4K output, ×4) & output Mpix/s at 1/2/4/8 B200 vs CPU ref"
WORKLOADS = {
    "c3": "c3: synthetic 1M-Gaussian scene, 960x540 render with analytic gradients, "
          "x4 gradient-aware spline upscale to 3840x2160, 1024-view batch sharded over ranks",
    "c2": "c2: synthetic 200k-Gaussian scene, 960x540 render with analytic gradients, "
          "x2 gradient-aware spline upscale to 1920x1080",
    "c4": "c4: synthetic 3M-Gaussian scene, stereo frames of two 1080x1200 eyes (disparity pan), "
          "x2 gradient-aware spline upscale to 2160x2400 per eye",
}
FP32_LANES_PER_SM = 128
NUM_SMS = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c2", "c3", "c4"],
                    help="render workload (BASELINE.json configs; c3 is the headline)")
    ap.add_argument("--views", type=int, default=None, help="views in the batch (default: 1024; c4: 64 frames)")
    ap.add_argument("--slots", type=int, default=8, help="concurrent view streams in the timed region (4 -> 8: C3 +1%%, C2 +3%%)")
    ap.add_argument("--kernel-views", type=int, default=64,
                    help="views of the single-stream per-kernel timing pass (roofline)")
    ap.add_argument("--workload", default="render", choices=["render", "train"],
                    help="render: C3 frames/s (headline); train: C5 upscale-aware training step")
    ap.add_argument("--train-views", type=int, default=4, help="views per rank per training step (C5)")
    ap.add_argument("--train-streams", type=int, default=4, help="C5 views in flight per rank (ViewTrainer streams)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="C3 only: skip the C2 / C4 / C5 measurements appended as extra_configs")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: tests with several ranks on one GPU)")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="map ranks onto the visible GPUs modulo their count (multi-rank tests on one GPU; "
                         "never a timing configuration)")
    ap.add_argument("--shard-log", default=None,
                    help="each rank writes the batch indices of its shard to <path>.<rank> (tests)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch/shard only: join the (gloo) group, write --shard-log, exit (no GPU; tests)")
    return ap.parse_args()


def maybe_spawn(args) -> None:
    """--gpus N without a torchrun environment: launch the N ranks through
    torch.distributed.run and exit with its status.  Under torchrun the world
    size must equal --gpus (a line whose n_gpus differs from --gpus is never printed)."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if int(env_world) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}: refusing a mismatched run")
        return
    if args.gpus <= 1 or args.impl == "reference":   # the reference arm runs on rank 0 alone
        return
    from paper_2503_14171_b200.distributed import free_port
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    sys.exit(subprocess.call(cmd, env=env))


def setup_rank(args):
    """(rank, world, device) of this process; joins the process group for N > 1."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world != max(args.gpus, 1):
        sys.exit(f"bench.py: --gpus {args.gpus} but world size {world}")
    ndev = torch.cuda.device_count()
    if ndev < 1:
        sys.exit("bench.py: no CUDA device visible")
    if args.shared_gpu:
        dev = local % ndev
    elif local >= ndev:
        sys.exit(f"bench.py: rank {rank} needs GPU {local} but only {ndev} are visible "
                 "(--gpus must not exceed the GPU count)")
    else:
        dev = local
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(args.dist_backend)
    return rank, world, dev


def dry_run(args) -> None:
    """The launch and sharding logic of the render path without a GPU: every rank
    joins a gloo group, computes its shard of the batch, logs it, and checks that
    the whole job covers the batch exactly once."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world != max(args.gpus, 1):
        sys.exit(f"bench.py: --gpus {args.gpus} but world size {world}")
    if world > 1:
        dist.init_process_group("gloo")
    nframes = args.views // views_per_frame(args)
    lo, hi = frame_shard(nframes, views_per_frame(args), rank, world)
    if args.shard_log:
        with open(f"{args.shard_log}.{rank}", "w") as f:
            json.dump({"rank": rank, "world": world, "lo": lo, "hi": hi}, f)
    from paper_2503_14171_b200 import distributed as D
    total = D.total_items(hi - lo)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "views": total}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def upscale_steady_state(W: int, H: int, OW: int, OH: int, nbuf: int = 4, launches: int = 48):
    """Per-launch time of splat_upscale_forward in steady state: back-to-back launches
    rotating over `nbuf` distinct source images and output frames, so each launch's
    working set (48 B per source + 12 B per output pixel) was evicted from the 126 MB L2
    since its last use and the write-back of earlier frames is paid inside the window.
    Returns (us per launch, algorithmic bytes per launch, kernel name)."""
    import torch
    from paper_2503_14171_b200 import _lib
    from paper_2503_14171_b200.spline import upscale_plan
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    gen = torch.Generator(device=dev).manual_seed(0)
    srcs = [torch.rand((H, W, 4, 3), device=dev, generator=gen) for _ in range(nbuf)]
    outs = [torch.empty((OH, OW, 3), device=dev) for _ in range(nbuf)]
    plan = upscale_plan(W, H, OW, OH, dev)
    st = _lib.stream_ptr()

    def launch(k):
        _lib.check(lib.splat_upscale_forward(_lib.ptr(srcs[k % nbuf]), W, H, _lib.ptr(outs[k % nbuf]), OW, OH,
                                             1, _lib.ptr(plan), st))

    for k in range(2 * nbuf):
        launch(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(launches):
        launch(k)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / launches
    if OW == 4 * W and OH == 4 * H:
        name = "upscale_x4_kernel"
    elif OW == 2 * W and OH == 2 * H:
        name = "upscale_x2_kernel" if OW % 4 == 0 else "upscale_int_kernel<2>"
    else:
        name = "upscale_fwd_kernel"
    del srcs, outs
    return us, 12.0 * OW * OH + 48.0 * W * H, name


def frame_shard(nframes: int, vpf: int, rank: int, world: int):
    """[lo, hi) view indices of this rank: a contiguous, balanced run of whole frames
    (both eyes of a stereo frame stay on one rank)."""
    from paper_2503_14171_b200.distributed import shard_bounds
    lo, hi = shard_bounds(nframes, rank, world)
    return lo * vpf, hi * vpf


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def metric_of(args):
    if args.config == "c3":
        return METRIC
    c = bench_config(args)
    what = "stereo frames/s (2 eyes" if args.config == "c4" else "upscaled frames/s ("
    return f"{what}{', ' if args.config == 'c4' else ''}{c.out_w}x{c.out_h} output, ×{c.factor:g}) at 1 B200 vs CPU ref"


def bench_config(args):
    from paper_2503_14171_b200.scenes import CONFIGS
    return CONFIGS[args.config]


def views_per_frame(args):
    return 2 if args.config == "c4" else 1


def config_dict(args, world, views_per_rank):
    c = bench_config(args)
    d = {"workload": WORKLOADS[args.config], "n_splats": c.n, "render": [c.width, c.height],
         "output": [c.out_w, c.out_h], "factor": c.factor, "views": args.views,
         "views_per_rank": views_per_rank, "parallelism": f"view-shard x{world}",
         "l2": "no explicit flush: each view streams ~250 MB (pack, pairs, planes, 99.5 MB output) "
               "through the 126 MB L2" if args.config == "c3" else
               "no explicit flush: per-view working set (pack, pairs, planes, output) exceeds the 126 MB L2"}
    if views_per_frame(args) > 1:
        d["views_per_frame"] = views_per_frame(args)
    return d


# ---------------------------------------------------------------------------
# CPU reference (oracle port) timing
# ---------------------------------------------------------------------------

def cpu_reference_view(scene, view, c):
    """One view through the CPU oracle (render + upscale); seconds."""
    from oracle import oracle as O
    from paper_2503_14171_b200.scenes import view_scene
    t0 = time.perf_counter()
    img = O.render_forward(view_scene(scene, view), c.width, c.height)
    O.upscale_spline(img.color, img.d_dx, img.d_dy, img.d_dxdy, c.factor)
    return time.perf_counter() - t0


def make_workload(args):
    from paper_2503_14171_b200.scenes import random_views, stereo_views, synthetic_scene
    c = bench_config(args)
    scene = synthetic_scene(c.n, c.width, c.height, c.scale_range, seed=5)
    if args.config == "c4":
        views = stereo_views(args.views, c.width, c.height, seed=11)
    else:
        views = random_views(args.views, c.width, c.height, seed=11)
    return scene, views


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    c = bench_config(args)
    scene, views = make_workload(args)
    cores = O.default_threads()
    for i in range(min(args.warmup, 1)):
        cpu_reference_view(scene, views[i], c)
    times = [cpu_reference_view(scene, views[i % len(views)], c) for i in range(args.steps)]
    per_view = sum(times) / len(times)
    value = 1.0 / (per_view * views_per_frame(args))
    sample = (f"1 view of the {args.config.upper()} batch per step (views 0..{args.steps - 1}), "
              f"per-view time x {len(views)} views extrapolated")
    line = {"impl": "reference", "metric": metric_of(args), "value": value, "unit": "frames/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": min(args.warmup, 1),
            "ms_per_step": per_view * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, 1, len(views)),
            "mpix_per_s": value * views_per_frame(args) * c.out_w * c.out_h / 1e6,
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "note": "reference CPU path = the float64 C/numpy oracle port of splinesplat (the reference "
                    "is a Python/numba package that cannot be shipped to the GPU box)"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.path = tempfile.mktemp(prefix="clocks_", suffix=".csv")
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for row in open(self.path):
            p = [x.strip() for x in row.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        busy = [s for s in sm if s > 0.5 * mx] or sm
        busy.sort()
        return {"sm_mhz": busy[len(busy) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def train_workload(views_per_rank, world):
    from paper_2503_14171_b200.scenes import CONFIGS, random_views, synthetic_scene
    c = CONFIGS["c5"]
    model = synthetic_scene(c.n, c.canvas_w, c.canvas_h, c.scale_range, seed=5)
    target = synthetic_scene(c.n, c.canvas_w, c.canvas_h, c.scale_range, seed=7)
    views = random_views(views_per_rank * world, c.canvas_w, c.canvas_h, seed=13)
    return c, model, target, views


TRAIN_METRIC = "upscale-aware training view-steps/s (C5: 1M splats, 480x270 render, x4 to 1920x1080, L1+SSIM)"


def train_config(c, world, vpr, streams=2):
    return {"workload": "c5: 1M-splat model (seed 5) fit to a 1M-splat target scene (seed 7); per view: "
                        "480x270 render with analytic gradients, x4 spline upscale to 1920x1080, "
                        "L1+SSIM (lambda 0.2) loss, backward through upscaler and rasterizer; "
                        "grads all-reduced over ranks, then Adam",
            "n_splats": c.n, "render": [c.width, c.height], "output": list(c.out_size),
            "views_per_rank": vpr, "views_in_flight": streams,
            "parallelism": f"view-DP x{world} + NCCL all_reduce(SUM) of the 9N fp32 rank-order gradient terms"}


def cpu_reference_train_view(model, target_img, view, c):
    """One C5 view-step through the CPU oracle: fwd, upscale, loss, upscale bwd, raster bwd (seconds)."""
    from oracle import oracle as O
    from paper_2503_14171_b200.scenes import view_scene
    t0 = time.perf_counter()
    sc = view_scene(model, view)
    fwd = O.render_forward(sc, c.width, c.height)
    pred = O.upscale_spline(fwd.color, fwd.d_dx, fwd.d_dy, fwd.d_dxdy, c.factor, out_size=c.out_size)
    _, dpred = O.loss(pred, target_img, 0.2)
    sadj = O.upscale_backward(c.width, c.height, c.factor, dpred, out_size=c.out_size)
    O.render_backward(sc, fwd, sadj)
    return time.perf_counter() - t0


def train_line(args, rank, world, local):
    """C5 upscale-aware training step (view-DP + NCCL all-reduce); rank 0 gets the JSON dict."""
    import torch
    import torch.distributed as dist
    from paper_2503_14171_b200 import _lib, distributed as D, fit
    from paper_2503_14171_b200.raster_forward import render_forward

    lib = _lib.load()
    vpr = args.train_views
    c, model, target_scene, views = train_workload(vpr, world)
    mine = D.shard(views, rank, world)
    W, H = c.out_size
    targets = [render_forward(target_scene, W, H, view=v).color.clamp(0.0, 1.0).contiguous() for v in mine]
    trainer = fit.ViewTrainer(model, (c.width, c.height), (W, H), mine, targets, ssim_weight=0.2,
                              streams=args.train_streams)
    for _ in range(args.warmup):
        trainer.step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = lib.splat_kernel_launches()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(args.steps):
        vals = trainer.step()
    s1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = lib.splat_kernel_launches() - l0
    trainer.check()
    ms = D.max_over_ranks(s0.elapsed_time(s1) / args.steps, device="cuda")
    total_views = D.total_items(len(mine), device="cuda")
    value = total_views / (ms / 1e3)
    # e2e: every step's targets streamed from pinned host memory (uploaded one step ahead on a
    # copy stream, overlapping the previous step), losses read back every step
    host_t = [t.cpu().pin_memory() for t in targets]
    h2d = sum(t.numel() * t.element_size() for t in host_t)
    ksteps = 20   # steady state: the first step's upload (not overlapped) is a one-off pipeline fill
    # per-step losses come back through a pinned double buffer: step k's read completes
    # while step k+1 is already queued, so the host never starves the device
    lbuf = [torch.empty_like(trainer.values, device="cpu").pin_memory() for _ in range(2)]
    lev = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize()
    e0 = time.perf_counter()
    trainer.prefetch_targets(host_t)
    for k in range(ksteps):
        vals = trainer.step()
        if k + 1 < ksteps:
            trainer.prefetch_targets(host_t)
        lbuf[k % 2].copy_(vals, non_blocking=True)
        lev[k % 2].record()
        if k > 0:
            lev[(k - 1) % 2].synchronize()
            losses = lbuf[(k - 1) % 2].clone()
    lev[(ksteps - 1) % 2].synchronize()
    losses = lbuf[(ksteps - 1) % 2].clone()
    torch.cuda.synchronize()
    ems = D.max_over_ranks((time.perf_counter() - e0) / ksteps * 1e3, device="cuda")
    clk = clocks.stop()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        O.build()
        tgt0 = targets[0].double().cpu().numpy()
        tcpu = cpu_reference_train_view(model, tgt0, mine[0], c)
        cpu = {"value": 1.0 / tcpu, "unit": "view-steps/s", "cores": O.default_threads(), "kind": "port",
               "sample": "1 C5 view-step (fwd, x4 upscale, L1+SSIM, upscale bwd, raster bwd) through the oracle"}
    # roofline of the dominant kernel (the rasterizer backward): one view at a time on one
    # stream, CUDA events around render_backward, algorithmic FLOPs per SURVEY 8(d)
    roof = None
    if rank == 0:
        from paper_2503_14171_b200.raster_backward import PixelAdjoint, render_backward
        from paper_2503_14171_b200.spline import upscale_backward, upscale_spline
        tr_ds = trainer.ds
        tms, flops = 0.0, 0.0
        for v, tgt in zip(mine, targets):
            fwd = render_forward(tr_ds, c.width, c.height, view=v, train=True)
            pred = upscale_spline(fwd, 1.0, out_size=(W, H))
            _, adj_img = fit.loss_device(pred, tgt, 0.2)
            adj = PixelAdjoint.from_source(upscale_backward(fwd, 1.0, adj_img, out_size=(W, H)))
            K = float(fwd.contrib_count.sum(dtype=torch.int64))
            bb = fwd.frame.bboxes().to(torch.int64)
            E = float(((bb[:, 1] - bb[:, 0]) * (bb[:, 3] - bb[:, 2]))[fwd.frame.touched() > 0].sum())
            gbuf = trainer.grads   # scratch use after the timed steps
            render_backward(tr_ds, fwd, adj, out=gbuf, check_finite=False)   # warm (workspace allocation)
            # the same ABI call with its arguments prepared, so the events bracket device work only
            fr = fwd.frame
            nb = lib.splat_backward_workspace_bytes(tr_ds.n, fr.capacity)
            bws = torch.empty(nb, dtype=torch.uint8, device="cuda")
            cargs = (_lib.ptr(tr_ds.const), tr_ds.c_scene(), fwd.view, c.width, c.height, fwd.c_gimg(),
                     _lib.ptr(adj.planes), _lib.ptr(fr.ws), fr.nbytes, fr.capacity, _lib.ptr(bws), nb,
                     _lib.ptr(gbuf.flat), 0, _lib.stream_ptr())
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(lib.splat_render_backward(*cargs))
            e1.record()
            torch.cuda.synchronize()
            tms += e0.elapsed_time(e1)
            flops += c.width * c.height * 27.0 + 13.0 * E + 360.0 * K
        sm_mhz = (clk or {}).get("sm_mhz") or 1335.0
        peak = NUM_SMS * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12
        ach = flops / (tms * 1e-3) / 1e12
        roof = {"kernel": "raster_bwd2_kernel + reduce_pairs2_kernel + chain_kernel (splat_render_backward, per view)",
                "bound": "fp32", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "measured": f"CUDA events around the splat_render_backward call, {len(mine)} views one at a time",
                "algorithmic": {"formula": "27P + 13E + 360K (SURVEY 8d backward; E = bbox-tested upper bound)",
                                "flops_per_view": flops / len(mine)},
                "traffic": json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get("raster_bwd2_kernel")
                if os.path.exists(os.path.join(ROOT, "profiles", "ncu_traffic.json")) else None,
                "ms_per_view": tms / len(mine)}
    if rank == 0:
        line = {"metric": TRAIN_METRIC, "value": value, "unit": "view-steps/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": train_config(c, world, vpr, args.train_streams), "gpu_launches": int(launches),
                "loss_last_step": [float(x) for x in losses[:, 0]],
                "roofline": roof,
                "cpu_baseline": cpu,
                "e2e": {"value": total_views / (ems / 1e3), "unit": "view-steps/s", "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(vals.numel() * 8), "steps": ksteps},
                "clocks": clk}
        return line
    return None


def render_line(args, rank, world, local):
    """Render + upscale a view batch (C2/C3/C4); rank 0 gets the JSON dict."""
    import torch
    import torch.distributed as dist

    import numpy as np
    from paper_2503_14171_b200 import _lib, distributed as D
    from paper_2503_14171_b200.device import DeviceScene
    from paper_2503_14171_b200.pipeline import ViewPipeline

    lib = _lib.load()
    c = bench_config(args)
    W, H, F = c.width, c.height, c.factor
    OW, OH = c.out_w, c.out_h
    vpf = views_per_frame(args)
    scene, views = make_workload(args)
    nframes = len(views) // vpf
    lo, hi = frame_shard(nframes, vpf, rank, world)
    mine = views[lo:hi]
    if args.shard_log:
        with open(f"{args.shard_log}.{rank}", "w") as f:
            json.dump({"rank": rank, "world": world, "device": local, "lo": lo, "hi": hi,
                       "views": [[v.zoom, v.ox, v.oy] for v in mine]}, f)
    # pinned host buffers (e2e ring, scene upload) on the GPU's own NUMA node
    numa = D.numa_node_of(local)
    cpus = D.bind_host_to_numa(numa) if world > 1 else None

    pipe = ViewPipeline(scene, W, H, factor=F, slots=args.slots, views_for_capacity=mine)

    # untimed: algorithmic work per view (K = sum contrib_count, E = sum valid bbox areas)
    sample = mine[: min(16, len(mine))]
    from paper_2503_14171_b200.raster_forward import render_forward
    K = E = 0.0
    for v in sample:
        img = render_forward(pipe.scene, W, H, view=v)
        K += float(img.contrib_count.sum(dtype=torch.int64))
        bb = img.frame.bboxes().to(torch.int64)
        area = (bb[:, 1] - bb[:, 0]) * (bb[:, 3] - bb[:, 2])
        E += float(area[img.frame.touched() > 0].sum())
        del img
    K /= len(sample)
    E /= len(sample)
    P = W * H
    raster_flops = 27.0 * P + 13.0 * E + 69.0 * K
    up_bytes = 12.0 * OW * OH + 48.0 * P

    for _ in range(args.warmup):
        pipe.render(mine)
    torch.cuda.synchronize()
    pipe.check()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.splat_kernel_launches()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(args.steps):
        pipe.fork()
        pipe.render(mine)
        pipe.join()
    end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = lib.splat_kernel_launches() - launches0
    ms = start.elapsed_time(end) / args.steps
    pipe.check()
    # per-kernel timing pass (roofline): the same views on ONE stream with CUDA events
    # around every stage, so each kernel's duration is measured without overlap
    kpipe = ViewPipeline(pipe.scene, W, H, factor=F, slots=1, capacity=pipe.capacity)
    kviews = mine[: max(1, min(args.kernel_views, len(mine)))]
    kpipe.render(kviews)
    torch.cuda.synchronize()
    kpipe.enable_stage_timing(True)
    kpipe.render(kviews)
    torch.cuda.synchronize()
    kpipe.check()
    stage = kpipe.stage_times_ms()
    clk = clocks.stop()
    del kpipe
    ms_max = D.max_over_ranks(ms, device="cuda")
    total_views = D.total_items(len(mine), device="cuda")   # views rendered by the whole job
    value = total_views / vpf / (ms_max / 1e3)

    # ---- e2e through the public API with host buffers -------------------------------------
    e2e = None
    if not args.no_e2e:
        host = {f: torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).pin_memory()
                for f in ("means", "log_scales", "rotations", "opacity_logits", "colors", "depths")}
        h2d = sum(v.numel() * v.element_size() for v in host.values())
        ring = [torch.empty((OH, OW, 3), dtype=torch.float32).pin_memory() for _ in range(4)]
        d2h = len(mine) * OH * OW * 3 * 4

        def e2e_step():
            dev = {k: v.to("cuda", non_blocking=True) for k, v in host.items()}
            ds = DeviceScene(**dev, background=tuple(scene.background),
                             reference_resolution=tuple(scene.reference_resolution)).prepare()
            p2 = ViewPipeline(ds, W, H, factor=F, slots=args.slots, capacity=pipe.capacity)
            p2.render(mine, host_out=ring)
            p2.join()
            return p2

        e2e_step()
        torch.cuda.synchronize()
        ksteps = max(1, min(args.steps, 2))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(ksteps):
            p2 = e2e_step()
        s1.record()
        torch.cuda.synchronize()
        p2.check()
        ems = s0.elapsed_time(s1) / ksteps
        wall = (time.perf_counter() - t0) / ksteps * 1e3
        et = D.max_over_ranks(max(ems, wall), device="cuda")
        e2e = {"value": total_views / vpf / (et / 1e3), "unit": "frames/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": ksteps, "api": "DeviceScene upload + prepare, ViewPipeline.render(host_out=pinned ring)"}

    # ---- roofline ------------------------------------------------------------------------------
    sm_mhz = (clk or {}).get("sm_mhz") or 1335.0
    fp32_peak = NUM_SMS * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak, hbm_src = float(peaks["hbm_gbs"]), "measured"
    except Exception:
        hbm_peak, hbm_src = 6650.0, "fallback"
    traffic = {}
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        pass
    util = {}
    try:
        util = json.load(open(os.path.join(ROOT, "profiles", "ncu_util.json")))
    except Exception:
        pass
    roof = None
    roof_up = None
    roof_issue = None
    if stage:
        r_ms = stage["raster"]
        roof = {"kernel": "raster_fwd_kernel (splat_rasterize with the fix-up deferred; per view)", "bound": "fp32",
                "measured": f"CUDA events around the raster kernel on its stream, single-stream pass over "
                            f"{len(kviews)} views (the exact fix-up is timed as its own stage)",
                "achieved": raster_flops / (r_ms * 1e-3) / 1e12,
                "peak": fp32_peak, "unit": "TFLOP/s", "frac": raster_flops / (r_ms * 1e-3) / 1e12 / fp32_peak,
                "traffic": traffic.get("raster_fwd_kernel"),
                "algorithmic": {"flops_per_view": raster_flops, "K_contrib_per_view": K,
                                "E_bbox_evals_per_view": E, "formula": "27P + 13E + 69K (SURVEY 8d)"},
                "peak_source": f"148 SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz (median SM clock in run)",
                "ncu_utilisation": util.get("raster_fwd_kernel"),
                "note": "the SURVEY 8(d) FLOP count omits the certified-decision arithmetic, culling and "
                        "blend bookkeeping; the kernel is issue-bound (see ncu_utilisation, roofline_issue)"}
        inst = (util.get("raster_fwd_kernel") or {}).get("inst_executed") if args.config == "c3" else None
        if inst:   # the bound the kernel actually meets: warp-instruction issue (4 schedulers per SM)
            issue_peak = NUM_SMS * 4 * sm_mhz * 1e6
            roof_issue = {"kernel": "raster_fwd_kernel", "bound": "issue", "unit": "G warp-instructions/s",
                          "achieved": inst / (r_ms * 1e-3) / 1e9, "peak": issue_peak / 1e9,
                          "frac": inst / (r_ms * 1e-3) / issue_peak, "instructions_per_launch": inst,
                          "source": "smsp__inst_executed.sum of one C3 launch (profiles/r02/ncu_summary.txt) over "
                                    "the stage time measured here; peak = 148 SM x 4 schedulers x 1 issue/clock"}
    if rank == 0:
        # steady state: back-to-back launches over 4 distinct sources and frames (working set
        # 4 x 124 MB at C3/C4 >> the 126 MB L2), so each frame's write-back is paid in the window
        u_us, u_bytes, u_name = upscale_steady_state(W, H, OW, OH, nbuf=4, launches=48)
        roof_up = {"kernel": u_name, "bound": "hbm",
                   "measured": "CUDA events around 48 back-to-back launches rotating over 4 distinct source "
                               "images and output frames (L2 flushed by the working set)",
                   "us_per_launch": u_us, "achieved": u_bytes / (u_us * 1e-6) / 1e9, "peak": hbm_peak,
                   "unit": "GB/s", "frac": u_bytes / (u_us * 1e-6) / 1e9 / hbm_peak,
                   "traffic": traffic.get(u_name), "algorithmic_bytes": u_bytes, "peak_source": hbm_src,
                   "in_pipeline_stage_us": stage.get("upscale", 0.0) * 1e3 if stage else None}

    # ---- CPU baseline (rank 0, N=1 only) ---------------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        O.build()
        tcpu = cpu_reference_view(scene, mine[0], c)
        cpu = {"value": 1.0 / (tcpu * vpf), "unit": "frames/s", "cores": O.default_threads(), "kind": "port",
               "sample": f"1 view of the {args.config.upper()} batch through the float64 oracle "
                         f"(render + x{F:g} upscale), x{vpf} views per frame"}

    cfg = config_dict(args, world, len(mine))
    if world > 1:
        cfg["host_numa"] = {"node": numa, "cpus": len(cpus) if cpus else None,
                            "note": "rank 0's pinned host ring is allocated on its GPU's NUMA node"}
        cfg["backend"] = args.dist_backend
    if rank == 0:
        line = {"metric": metric_of(args), "value": value, "unit": "frames/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": cfg,
                "mpix_per_s": value * vpf * OW * OH / 1e6,
                "stage_ms_per_view": stage, "gpu_launches": int(launches),
                "roofline": roof, "roofline_upscale": roof_up, "roofline_issue": roof_issue,
                "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clk}
        return line
    return None


def main():
    args = parse()
    maybe_spawn(args)
    if args.views is None:
        args.views = {"c2": 256, "c3": 1024, "c4": 64}[args.config]
    if args.impl == "reference":
        run_reference(args)
        return
    if args.dry_run:
        dry_run(args)
        return
    import torch.distributed as dist
    rank, world, local = setup_rank(args)
    if args.workload == "train":
        line = train_line(args, rank, world, local)
    else:
        line = render_line(args, rank, world, local)
        if args.config == "c3" and not args.no_extras:
            extras = run_extras(args, rank, world, local)
            if rank == 0:
                line["extra_configs"] = extras
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


EXTRA_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "mpix_per_s", "stage_ms_per_view", "gpu_launches", "roofline", "roofline_upscale", "e2e",
              "cpu_baseline", "loss_last_step", "clocks")


def run_extras(args, rank, world, local):
    """The other BASELINE.json configurations, measured after (outside) the C3 timed region
    by the same code paths: C2 and C4 renders (x2) and the C5 training step."""
    import copy
    import torch
    extras = {}
    for cfg, views in (("c2", 256), ("c4", 64)):
        a = copy.copy(args)
        a.config, a.views, a.kernel_views, a.shard_log = cfg, views, 16, None
        a.steps, a.no_cpu_baseline = max(3, min(args.steps, 10)), True
        ln = render_line(a, rank, world, local)
        torch.cuda.empty_cache()
        if rank == 0:
            extras[cfg] = {k: ln.get(k) for k in EXTRA_KEYS if k in ln}
    a = copy.copy(args)
    a.workload, a.steps, a.warmup = "train", 5, 3
    ln = train_line(a, rank, world, local)
    torch.cuda.empty_cache()
    if rank == 0:
        extras["c5_train"] = {k: ln.get(k) for k in EXTRA_KEYS if k in ln}
    return extras


if __name__ == "__main__":
    main()
