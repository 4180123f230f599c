"""Multi-GPU plumbing: one process per GPU (torchrun), view sharding, and the
single collective of the training path.

* Inference (configs 2-4): camera views are independent, so a batch is split
  into contiguous per-rank shards and rendered with no data-path collective
  (SURVEY.md 8(e)); only the timing uses a barrier and a MAX reduction.
* Training (config 5): view data-parallel.  Each rank accumulates the float32
  gradients of its views into one flat buffer; ``allreduce_grads`` sums them
  over the group (NCCL over NVLink on the B200 box, gloo in the CPU tests) so
  every rank applies the identical Adam update to its parameter replica.

The functions here are device-agnostic so the host logic is tested with gloo
on CPU (tests/test_distributed.py).
"""

from __future__ import annotations

import os
import socket

import torch
import torch.distributed as dist


def env_rank_world():
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard_bounds(n_items: int, rank: int, world: int):
    """Contiguous [lo, hi) of rank's share; sizes differ by at most one."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("invalid rank/world")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard(items, rank: int, world: int):
    lo, hi = shard_bounds(len(items), rank, world)
    return list(items[lo:hi])


def allreduce_grads(flat: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-rank gradient buffers in place (the training path's only collective)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


def max_over_ranks(value: float, device=None, group=None) -> float:
    """MAX of a per-rank scalar (step times are reported as the slowest rank's)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def total_items(n_local: int, device=None, group=None) -> int:
    """SUM of per-rank item counts (views rendered by the whole job)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return int(n_local)
    t = torch.tensor([int(n_local)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def free_port() -> int:
    """An unused TCP port on 127.0.0.1 for a local rendezvous."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def numa_node_of(device: int) -> int | None:
    """NUMA node the GPU hangs off (sysfs), or None when unknown / single-node."""
    try:
        p = torch.cuda.get_device_properties(device)
        path = f"/sys/bus/pci/devices/{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0/numa_node"
        node = int(open(path).read().strip())
        return node if node >= 0 else None
    except Exception:
        return None


def bind_host_to_numa(node: int | None) -> list | None:
    """Restrict this process's CPUs to ``node`` so pinned host buffers allocated
    afterwards are first-touched (hence placed) on the GPU's own NUMA node.
    Returns the CPU list, or None if nothing was changed."""
    if node is None:
        return None
    try:
        spec = open(f"/sys/devices/system/node/node{node}/cpulist").read().strip()
        cpus = []
        for part in spec.split(","):
            lo, _, hi = part.partition("-")
            cpus.extend(range(int(lo), int(hi or lo) + 1))
        cpus = [c for c in cpus if c in os.sched_getaffinity(0)]
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        return cpus
    except Exception:
        return None
