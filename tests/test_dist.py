"""Multi-process (world_size 2, gloo, CPU) tests of the sharded scene path.

The plumbing under test is paper_2605_08975_b200.dist (slice planning, the
prefix broadcast, the lane gather).  On CPU the per-rank compute stands in
with the oracle restatement (test infrastructure) on the rank's global lanes;
the GPU path runs the same plumbing over NCCL with the C-ABI compute.
"""
import os
import socket

import numpy as np
import pytest

from paper_2605_08975_b200 import dist as pdist


def test_even_split_covers_everything():
    for total in (0, 1, 5, 6, 16, 64):
        for world in (1, 2, 3, 4, 8):
            got = [pdist.even_split(total, world, r) for r in range(world)]
            assert sum(c for _, c in got) == total
            nxt = 0
            for first, count in got:
                assert first == nxt
                nxt += count
    assert list(pdist.scene_slice(64, 8, 3)) == list(range(24, 32))
    assert pdist.lane_slice(6, 4, 3) == (5, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from oracle.oracle import Cfg, Port

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port_ = Port()
    cfg = Cfg.make(vision_blocks=1, decoder_blocks=2, hidden_dim=16, action_hidden_dim=8,
                   kv_dim=8, heads=2, vocab_size=128, weight_seed=77, diffusion_iters=3)
    w = port_.weights(cfg)
    r, n_total = 12, 5
    prefix = torch.zeros(2 * 2 * r * 8, dtype=torch.float32)

    def produce(buf):  # the reasoning stage lives on the root only
        buf.copy_(torch.from_numpy(port_.synthetic_prefix(4242, 2, r, 8).ravel()))

    def compute(lane0, n_local):
        pre = prefix.numpy().reshape(2, 2, r, 8)
        acts = port_.refine(cfg, w, pre, port_.noise(2, 1, n_local, lane0))
        return torch.from_numpy(acts)

    full = pdist.run_scene(compute, prefix, n_total, root=0, produce=produce)
    if rank == 0:
        np.save(os.path.join(out_dir, "sharded.npy"), full.numpy())
        ref = port_.refine(cfg, w, port_.synthetic_prefix(4242, 2, r, 8), port_.noise(2, 1, n_total))
        np.save(os.path.join(out_dir, "single.npy"), ref)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_scene_matches_single_process(tmp_path):
    import torch.multiprocessing as mp

    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    a = np.load(tmp_path / "sharded.npy")
    b = np.load(tmp_path / "single.npy")
    assert a.shape == (5, 64, 2)
    np.testing.assert_array_equal(a, b)  # global lane seeds: bit-identical


def _scenes_worker(rank, world, port, out_dir, num_scenes):
    import torch
    import torch.distributed as dist

    from oracle.oracle import Cfg, Port

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port_ = Port()
    cfg = Cfg.make(vision_blocks=1, decoder_blocks=2, hidden_dim=16, action_hidden_dim=8,
                   kv_dim=8, heads=2, vocab_size=128, weight_seed=77, diffusion_iters=2)
    w = port_.weights(cfg)
    r, n = 10, 3
    computed = []

    def produce(s, buf):  # only the root produces prefixes (the reasoning stage)
        assert rank == 0
        buf.copy_(torch.from_numpy(port_.synthetic_prefix(4242 + 1000 * s, 2, r, 8).ravel()))

    def compute(s, buf):
        computed.append(s)
        pre = buf.numpy().reshape(2, 2, r, 8)
        return torch.from_numpy(port_.refine(cfg, w, pre, port_.noise(2, 1, n)))

    full, mine = pdist.run_scenes(num_scenes, compute, produce,
                                  lambda: torch.zeros(2 * 2 * r * 8, dtype=torch.float32))
    assert computed == mine == pdist.owned_scenes(num_scenes, world, rank)
    if rank == 0:
        np.save(os.path.join(out_dir, "scenes.npy"), full.numpy())
        ref = np.stack([port_.refine(cfg, w, port_.synthetic_prefix(4242 + 1000 * s, 2, r, 8),
                                     port_.noise(2, 1, n)) for s in range(num_scenes)])
        np.save(os.path.join(out_dir, "scenes_ref.npy"), ref)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,num_scenes", [(2, 5), (3, 7)])
def test_batched_scenes_sharded_match_single_process(tmp_path, world, num_scenes):
    """Config 5 plumbing: scenes round-robin over ranks, the root sends each
    prefix point-to-point to the owner, results gathered in scene order."""
    import torch.multiprocessing as mp

    mp.spawn(_scenes_worker, args=(world, _free_port(), str(tmp_path), num_scenes), nprocs=world,
             join=True)
    a = np.load(tmp_path / "scenes.npy")
    b = np.load(tmp_path / "scenes_ref.npy")
    assert a.shape == (num_scenes, 3, 64, 2)
    np.testing.assert_array_equal(a, b)


def test_scene_owner_round_robin():
    assert [pdist.scene_owner(s, 4) for s in range(6)] == [0, 1, 2, 3, 0, 1]
    assert pdist.owned_scenes(64, 8, 3) == list(range(3, 64, 8))
