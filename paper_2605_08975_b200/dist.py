"""Multi-GPU sharding of the action-generation path.

The path shards only across independent units: the trajectories (lanes) of
one scene given its prefix, and independent scenes.  There is no cross-lane
reduction anywhere in the path (attention, LayerNorm and GEMM rows are per
lane), so the only exchanges are

* one prefix-KV broadcast per scene from the rank that produced the reasoning
  (ncclBroadcast over NVLink/NVSwitch, 302 MB bf16 at Alpamayo width), and
* one gather of the per-rank action / trajectory slices (512 B + 768 B per
  trajectory).

Lane slices keep GLOBAL lane indices, so the per-lane noise seed
``action_init_seed + lane * stride`` (pipeline.cpp:415-424) and therefore the
result are identical on 1 and G GPUs.

Plumbing is torch.distributed (NCCL on GPUs, gloo on CPU for the tests); the
compute is the C-ABI library.
"""
from __future__ import annotations

from typing import Callable


def even_split(total: int, world: int, rank: int) -> tuple[int, int]:
    """(first index, count) of rank's contiguous share of `total` units."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(total, world)
    count = base + (1 if rank < rem else 0)
    first = rank * base + min(rank, rem)
    return first, count


def lane_slice(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """(lane0, n_local) of one scene's trajectories on this rank."""
    return even_split(n_total, world, rank)


def scene_slice(num_scenes: int, world: int, rank: int) -> range:
    """Scenes this rank denoises in a batched (config-5) run."""
    first, count = even_split(num_scenes, world, rank)
    return range(first, first + count)


def broadcast_prefix(prefix, root: int = 0, group=None) -> None:
    """One collective per scene: the prefix KV (a torch tensor, device or
    host) from the producing rank to every rank, in place."""
    import torch.distributed as dist

    dist.broadcast(prefix, root, group=group)


def gather_lanes(local, n_total: int, group=None):
    """All-gather per-rank lane slices [n_local, ...] into [n_total, ...]
    ordered by global lane index (uneven slices padded for the collective)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = [even_split(n_total, world, r)[1] for r in range(world)]
    width = max(counts)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


def run_scene(compute: Callable[[int, int], "object"], prefix, n_total: int, root: int = 0,
              produce: Callable[[object], None] | None = None, group=None):
    """One sharded scene: the root produces the prefix (``produce(prefix)``),
    it is broadcast, every rank computes its lane slice with
    ``compute(lane0, n_local) -> tensor [n_local, ...]`` and the slices are
    gathered on every rank.  Returns the full [n_total, ...] tensor."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if produce is not None and rank == root:
        produce(prefix)
    broadcast_prefix(prefix, root, group)
    lane0, n_local = lane_slice(n_total, world, rank)
    local = compute(lane0, n_local)
    return gather_lanes(local, n_total, group)
