"""The N>1 paths run for real, as two processes on the one GPU of the test box
(gloo group over CUDA tensors; correctness only, never timing):

* bench.py --gpus 2 launches its own ranks, renders the C3 batch sharded by view
  (disjoint shards whose union is the batch) through the real pipeline and e2e
  path, and reports n_gpus = 2 with the whole job's view count;
* ViewTrainer.step inside a real process group: the all-reduced step equals the
  single-process step over all views (float32 summation order only) and the
  oracle's sum of per-view gradients (1e-3 relative, SURVEY 8(e);
  reference: raster_backward.py:116-124, fit.py:188-223);
* three ranks' view shards render bitwise what one process renders for the batch.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from test_gpu_backward import FIELDS, rel_err

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_render_disjoint_shards(tmp_path):
    log = str(tmp_path / "shard")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--shared-gpu",
                        "--dist-backend", "gloo", "--views", "10", "--kernel-views", "2", "--steps", "1",
                        "--warmup", "3", "--no-cpu-baseline", "--shard-log", log],
                       capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["views"] == 10
    shards = [json.load(open(f"{log}.{k}")) for k in range(2)]
    assert [s["rank"] for s in shards] == [0, 1] and all(s["world"] == 2 for s in shards)
    assert (shards[0]["lo"], shards[0]["hi"], shards[1]["lo"], shards[1]["hi"]) == (0, 5, 5, 10)
    from paper_2503_14171_b200.scenes import random_views
    views = [[v.zoom, v.ox, v.oy] for v in random_views(10, 960, 540, seed=11)]
    assert shards[0]["views"] + shards[1]["views"] == views
    # the job's frame count: whole views of both ranks over the max-over-ranks time
    assert abs(line["value"] - 10 / (line["ms_per_step"] / 1e3)) <= 1e-6 * line["value"]


def _problem():
    from paper_2503_14171_b200.scenes import random_views, synthetic_scene
    model = synthetic_scene(2000, 96, 64, (2.0, 6.0), seed=5)
    tsc = synthetic_scene(2000, 96, 64, (2.0, 6.0), seed=7)
    return model, tsc, random_views(4, 96, 64, seed=3)


def _trainer_rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2503_14171_b200 as P
        from paper_2503_14171_b200 import distributed as D, fit
        model, tsc, views = _problem()
        mine = D.shard(views, rank, world)
        tg = [P.render_forward(tsc, 96, 64, view=v).color.clamp(0, 1).contiguous() for v in mine]
        tr = fit.ViewTrainer(model, (24, 16), (96, 64), mine, tg)
        tr.step()
        torch.cuda.synchronize()
        grads = tr.grads.grads().numpy()
        params = {k: v.double().cpu().numpy() for k, v in fit.scene_params(tr.ds).items()}
        q.put((rank, grads, params))
    except Exception as e:   # surface the failure in the parent
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


def test_view_trainer_step_in_a_real_process_group(oracle):
    import torch
    import torch.multiprocessing as mp
    import paper_2503_14171_b200 as P
    from paper_2503_14171_b200 import fit
    from paper_2503_14171_b200.distributed import free_port
    from paper_2503_14171_b200.scenes import view_scene
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_trainer_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[2] is not None, r[1]
    (_, g0, p0), (_, g1, p1) = res
    # every replica applied the identical update
    for f in FIELDS:
        assert np.array_equal(g0[f], g1[f]), f
    for k in p0:
        assert np.array_equal(p0[k], p1[k]), k
    # == the single-process step over all four views (float32 order only)
    model, tsc, views = _problem()
    tg = [P.render_forward(tsc, 96, 64, view=v).color.clamp(0, 1).contiguous() for v in views]
    full = fit.ViewTrainer(model.copy(), (24, 16), (96, 64), views, tg)
    full.step()
    one = full.grads.grads().numpy()
    for f in FIELDS:
        assert np.abs(g0[f] - one[f]).max() <= 1e-5 * np.abs(one[f]).max(), f
    # == the oracle's sum over views (the reference's per-view gradients, summed)
    ref = None
    for v, t in zip(views, tg):
        sv = view_scene(model, v)
        fwd = oracle.render_forward(sv, 24, 16)
        pred = oracle.upscale_spline(fwd.color, fwd.d_dx, fwd.d_dy, fwd.d_dxdy, 4.0, out_size=(96, 64))
        _, dpred = oracle.loss(pred, t.double().cpu().numpy(), 0.2)
        sadj = oracle.upscale_backward(24, 16, 4.0, dpred, out_size=(96, 64))
        gv = oracle.render_backward(sv, fwd, sadj)
        ref = gv if ref is None else {f: ref[f] + gv[f] for f in FIELDS}
    for f in FIELDS:
        assert rel_err(g0[f], ref[f]) < 1e-3, (f, rel_err(g0[f], ref[f]))
    torch.cuda.synchronize()


def _render_rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_14171_b200 import distributed as D
        from paper_2503_14171_b200.pipeline import render_upscale_views
        from paper_2503_14171_b200.scenes import random_views, synthetic_scene
        sc = synthetic_scene(30000, 320, 180, (0.5, 2.5), seed=5)
        views = random_views(9, 320, 180, seed=4)
        lo, hi = D.shard_bounds(len(views), rank, world)
        out = render_upscale_views(sc, 320, 180, views[lo:hi], factor=4.0, slots=3)
        q.put((rank, lo, out.cpu().numpy()))
    except Exception as e:
        q.put((rank, -1, repr(e)))
    finally:
        dist.destroy_process_group()


def test_view_sharded_render_is_invariant_to_world_size():
    """The reference's output never depends on its worker count (raster_forward.py:181-186,
    pkg/tests/test_raster_forward.py:200-207); here: the frames three ranks render for their
    shards of a 9-view batch are bitwise the single-process batch."""
    import torch
    import torch.multiprocessing as mp
    from paper_2503_14171_b200.distributed import free_port
    from paper_2503_14171_b200.pipeline import render_upscale_views
    from paper_2503_14171_b200.scenes import random_views, synthetic_scene
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_render_rank, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[1] >= 0, r[2]
    sharded = np.concatenate([r[2] for r in res])
    sc = synthetic_scene(30000, 320, 180, (0.5, 2.5), seed=5)
    whole = render_upscale_views(sc, 320, 180, random_views(9, 320, 180, seed=4), factor=4.0, slots=3)
    torch.cuda.synchronize()
    assert sharded.shape == tuple(whole.shape)
    assert np.array_equal(sharded, whole.cpu().numpy())
