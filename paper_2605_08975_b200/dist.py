"""Multi-GPU sharding of the action-generation path.

The path shards only across independent units: the trajectories (lanes) of
one scene given its prefix, and independent scenes.  There is no cross-lane
reduction anywhere in the path (attention, LayerNorm and GEMM rows are per
lane), so the only exchanges are

* one prefix-KV broadcast per scene from the rank that produced the reasoning
  (ncclBroadcast over NVLink/NVSwitch, 302 MB bf16 at Alpamayo width), and
* one gather of the per-rank action / trajectory slices (512 B + 768 B per
  trajectory).

Batched scenes (config 5, ``run_scenes``) shard whole scenes round-robin; the
producing rank sends each scene's prefix to its owner (NCCL point-to-point
over NVLink) on a side stream, so the transfer of the next scene overlaps the
denoising of the current one, and the results are gathered once at the end.

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


def scene_owner(scene: int, world: int) -> int:
    """Round-robin scene placement of a batched run: the producer streams the
    scenes in order and every rank receives one scene per round."""
    return scene % world


def owned_scenes(num_scenes: int, world: int, rank: int) -> list[int]:
    return [s for s in range(num_scenes) if scene_owner(s, world) == rank]


def run_scenes(num_scenes: int, compute: Callable[[int, object], object],
               produce: Callable[[int, object], None], make_buf: Callable[[], object],
               root: int = 0, group=None, side_stream=None):
    """Config 5: ``num_scenes`` independent scenes sharded round-robin over the
    ranks (``scene_owner``).  The root produces every scene's prefix
    (``produce(scene, buf)``) and sends it to the scene's owner (its own scenes
    stay local); each rank receives its next scene's prefix into the spare half
    of a double buffer while it denoises the current one
    (``compute(scene, buf) -> tensor [n, ...]``).  On GPUs the root's
    production and sends run on ``side_stream`` so they never wait behind its
    own denoising.  Returns ``(results [num_scenes, n, ...] on every rank,
    own scene list)``."""
    import contextlib

    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = owned_scenes(num_scenes, world, rank)
    side = (torch.cuda.stream(side_stream) if side_stream is not None
            else contextlib.nullcontext())
    outs = []
    if rank == root:
        # send buffers in flight, oldest first; one is reused only after its send completed
        from collections import deque
        inflight: deque = deque()
        max_inflight = 2 * max(1, world - 1)
        own_bufs = [make_buf(), make_buf()]
        own_events = {}
        ready = {}
        used = {}  # own buffer index -> event after the compute that read it

        def produce_round(k: int) -> None:
            for s in range(k * world, min(num_scenes, (k + 1) * world)):
                dst = scene_owner(s, world)
                with side:
                    if dst == root:
                        bi = (s // world) % 2
                        if bi in used:  # the compute two rounds back still reads it
                            side_stream.wait_event(used.pop(bi))
                        buf = own_bufs[bi]
                        produce(s, buf)
                        if side_stream is not None:
                            ev = torch.cuda.Event()
                            ev.record(side_stream)
                            own_events[s] = ev
                        ready[s] = buf
                        continue
                    if len(inflight) < max_inflight:
                        buf = make_buf()
                    else:
                        buf, work = inflight.popleft()
                        work.wait()
                    produce(s, buf)
                    inflight.append((buf, dist.isend(buf, dst, group=group)))

        rounds = (num_scenes + world - 1) // world
        produce_round(0)
        for k in range(rounds):
            if k + 1 < rounds:
                produce_round(k + 1)  # next round's transfers overlap this round's denoise
            for s in mine:
                if s // world == k:
                    if s in own_events:
                        torch.cuda.current_stream().wait_event(own_events.pop(s))
                    outs.append(compute(s, ready.pop(s)))
                    if side_stream is not None:
                        ev = torch.cuda.Event()
                        ev.record(torch.cuda.current_stream())
                        used[(s // world) % 2] = ev
        for _, w in inflight:
            w.wait()
    else:
        bufs = [make_buf(), make_buf()]
        pending = None
        if mine:
            pending = dist.irecv(bufs[0], root, group=group)
        for i, s in enumerate(mine):
            work = pending
            if i + 1 < len(mine):
                pending = dist.irecv(bufs[(i + 1) % 2], root, group=group)
            work.wait()
            outs.append(compute(s, bufs[i % 2]))
    local = torch.stack(outs) if outs else None
    # gather every rank's scenes, padded to the largest share, back in scene order
    share = (num_scenes + world - 1) // world
    if local is None:
        raise ValueError("every rank needs at least one scene (num_scenes >= world)")
    pad = torch.zeros((share,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    full = torch.empty((num_scenes,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    for r in range(world):
        for j, s in enumerate(owned_scenes(num_scenes, world, r)):
            full[s] = bufs[r][j]
    return full, mine
