"""Multi-process host logic of the N>1 path on CPU (gloo, world_size 2):
view sharding, the gradient all-reduce of the training step, and the
max-over-ranks timing.  The GPU kernels are not involved (no GPU here)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_14171_b200 import distributed as D


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            spans = [D.shard_bounds(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        views = list(range(10))
        mine = D.shard(views, rank, world)
        # each rank's "gradient" = a deterministic function of its views
        flat = torch.zeros(11 * 5, dtype=torch.float32)
        for v in mine:
            flat += torch.arange(flat.numel(), dtype=torch.float32) * (v + 1)
        D.allreduce_grads(flat)
        t = D.max_over_ranks(1.0 + rank)
        total = D.total_items(len(mine))
        out.put((rank, mine, flat.numpy().copy(), t, total))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_views_and_allreduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, v0, g0, t0, n0), (r1, v1, g1, t1, n1) = res
    assert v0 + v1 == list(range(10)) and not set(v0) & set(v1)
    expect = np.arange(55, dtype=np.float32) * sum(v + 1 for v in range(10))
    assert np.array_equal(g0, expect) and np.array_equal(g1, expect)   # identical update everywhere
    assert t0 == t1 == 2.0
    assert n0 == n1 == 10


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, env=None, timeout=300):
    import subprocess
    import sys
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                          text=True, env=e, timeout=timeout, cwd=ROOT)


@pytest.mark.parametrize("world,config,views", [(2, "c3", 1024), (3, "c3", 1024), (3, "c4", 64)])
def test_bench_gpus_n_spawns_n_ranks_and_shards_the_batch(tmp_path, world, config, views):
    """`bench.py --gpus N` outside torchrun launches N ranks itself; their shards
    are disjoint, contiguous, balanced whole frames covering the batch once."""
    log = str(tmp_path / "shard")
    r = _bench(["--gpus", str(world), "--dry-run", "--config", config, "--views", str(views),
                "--shard-log", log])
    assert r.returncode == 0, r.stderr[-2000:]
    import json
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == world and line["views"] == views
    spans = sorted(tuple(json.load(open(f"{log}.{k}"))[x] for x in ("lo", "hi")) for k in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == views
    assert all(b == c for (_, b), (c, _) in zip(spans, spans[1:]))
    vpf = 2 if config == "c4" else 1
    sizes = [(b - a) // vpf for a, b in spans]
    assert all((b - a) % vpf == 0 for a, b in spans) and max(sizes) - min(sizes) <= 1


def test_bench_refuses_a_world_size_other_than_gpus():
    r = _bench(["--gpus", "2", "--dry-run"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "refusing" in r.stderr
    assert not any(ln.startswith("{") for ln in r.stdout.splitlines())
