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
