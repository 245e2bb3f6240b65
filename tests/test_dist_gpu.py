"""The sharded paths with the LIBRARY as each rank's compute, on the GPU box
(one B200): NCCL at world size 1 (the scene broadcast + lane gather and the
batched-scene runner exercise the NCCL collectives and the library together)
and two ranks sharing the GPU over gloo (a real cross-process run_scenes with
the root sending prefixes point-to-point).  Results must equal the
single-process library call bitwise (global lane seeds; deterministic kernels).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

R = 256


def _cfg(dtype="bf16"):
    import paper_2605_08975_b200 as alpa
    return alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=2,
                            action_hidden_dim=256, kv_dim=128, heads=2, diffusion_iters=2,
                            dtype=dtype)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _direct(scene_seeds, n, dtype="bf16"):
    import paper_2605_08975_b200 as alpa
    out = []
    with alpa.ActionGenerator(_cfg(dtype)) as g:
        for seed in scene_seeds:
            g.bind_prefix_synthetic(seed, R)
            out.append(g.run_action_generation(alpa.InferenceRequest(num_trajectories=n, v0=5.0)))
    return out


def _nccl_world1(rank, port, out_dir):
    import torch
    import torch.distributed as dist

    import paper_2605_08975_b200 as alpa
    from paper_2605_08975_b200 import dist as pdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    g = alpa.ActionGenerator(_cfg())
    g.set_stream(stream.cuda_stream)
    n = 5
    req = alpa.InferenceRequest(num_trajectories=n, v0=5.0)
    noise = torch.from_numpy(alpa.host_noise(2, 1, n)).to(dev)
    per = g.prefix_bytes(R)

    def make_buf():
        return torch.empty(per // 2, dtype=torch.bfloat16, device=dev)

    def produce(s, buf):
        g.synthesize_prefix(buf.data_ptr(), 4242 + 1000 * s, R)

    def compute(s, buf):
        g.bind_prefix_device(buf.data_ptr(), 1, R)
        a = torch.empty((n, 64, 2), dtype=torch.float32, device=dev)
        t = torch.empty((n, 64, 3), dtype=torch.float32, device=dev)
        g.generate_device(req, noise.data_ptr(), a.data_ptr(), t.data_ptr())
        return torch.cat([a.reshape(n, -1), t.reshape(n, -1)], dim=1)

    prefix = make_buf()

    def lanes(lane0, n_local):
        g.bind_prefix_device(prefix.data_ptr(), 1, R)
        return compute(0, prefix)

    one = pdist.run_scene(lanes, prefix, n, root=0, produce=lambda b: produce(0, b))
    many, mine = pdist.run_scenes(3, compute, produce, make_buf, side_stream=torch.cuda.Stream(dev))
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, "one.npy"), one.cpu().numpy())
    np.save(os.path.join(out_dir, "many.npy"), many.cpu().numpy())
    g.close()
    dist.destroy_process_group()


def _split(res):
    return np.concatenate([res.actions.reshape(res.actions.shape[0], -1),
                           res.trajectories.reshape(res.trajectories.shape[0], -1)], axis=1)


def test_nccl_world1_library_scene_paths(tmp_path):
    import torch.multiprocessing as mp

    mp.spawn(_nccl_world1, args=(_free_port(), str(tmp_path)), nprocs=1, join=True)
    ref = [_split(r) for r in _direct([4242 + 1000 * s for s in range(3)], 5)]
    np.testing.assert_array_equal(np.load(tmp_path / "one.npy"), ref[0])
    np.testing.assert_array_equal(np.load(tmp_path / "many.npy"), np.stack(ref))


def _gloo_two_ranks(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import paper_2605_08975_b200 as alpa
    from paper_2605_08975_b200 import dist as pdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = alpa.ActionGenerator(_cfg())  # both ranks on cuda:0, separate contexts
    n = 4
    per = g.prefix_bytes(R)
    req = alpa.InferenceRequest(num_trajectories=n, v0=5.0)
    staging = torch.empty(per // 2, dtype=torch.bfloat16, device="cuda")

    def make_buf():  # gloo point-to-point moves host tensors
        return torch.empty(per // 2, dtype=torch.bfloat16)

    def produce(s, buf):
        assert rank == 0
        g.synthesize_prefix(staging.data_ptr(), 4242 + 1000 * s, R)
        torch.cuda.synchronize()
        buf.copy_(staging.cpu())

    def compute(s, buf):
        staging.copy_(buf.cuda())
        torch.cuda.synchronize()
        g.bind_prefix_device(staging.data_ptr(), 1, R)
        return torch.from_numpy(_split(g.run_action_generation(req)))

    full, mine = pdist.run_scenes(5, compute, produce, make_buf)
    assert mine == pdist.owned_scenes(5, world, rank)
    if rank == 0:
        np.save(os.path.join(out_dir, "gloo.npy"), full.numpy())
    dist.barrier()
    g.close()
    dist.destroy_process_group()


def test_two_ranks_share_gpu_batched_scenes(tmp_path):
    import torch.multiprocessing as mp

    mp.spawn(_gloo_two_ranks, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    ref = np.stack([_split(r) for r in _direct([4242 + 1000 * s for s in range(5)], 4)])
    np.testing.assert_array_equal(np.load(tmp_path / "gloo.npy"), ref)


def _gloo_two_ranks_lanes(rank, world, port, out_dir, dtype):
    import torch
    import torch.distributed as dist

    import paper_2605_08975_b200 as alpa
    from paper_2605_08975_b200 import dist as pdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = alpa.ActionGenerator(_cfg(dtype))
    n_total = 7
    per = g.prefix_bytes(R)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    staging = torch.empty(per // staging_esize(dtype), dtype=tdt, device="cuda")
    prefix = torch.empty(per // staging_esize(dtype), dtype=tdt)  # gloo moves host tensors

    def produce(buf):
        g.synthesize_prefix(staging.data_ptr(), 4242, R)
        torch.cuda.synchronize()
        buf.copy_(staging.cpu())

    def compute(lane0, n_local):
        staging.copy_(prefix.cuda())
        torch.cuda.synchronize()
        g.bind_prefix_device(staging.data_ptr(), 1, R)
        res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=n_local, lane0=lane0, v0=5.0))
        return torch.from_numpy(_split(res))

    full = pdist.run_scene(compute, prefix, n_total, root=0, produce=produce)
    if rank == 0:
        np.save(os.path.join(out_dir, "lanes.npy"), full.numpy())
    dist.barrier()
    g.close()
    dist.destroy_process_group()


def staging_esize(dtype):
    return 2 if dtype == "bf16" else 4


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_two_ranks_share_gpu_lane_sharded_scene(tmp_path, dtype):
    """One scene's lanes split over two processes (4 + 3 of 7, global lane
    seeds): the prefix broadcast from the producing rank, the library on each
    slice, the gather.  fp32 path: equal to one process computing all 7 lanes
    bitwise.  bf16 path: the persistent kernel's split-K / KV-split plan
    depends on the lane count (the reduction order with it), so a slice is
    equal within the bf16 bar, not bitwise."""
    import torch.multiprocessing as mp

    mp.spawn(_gloo_two_ranks_lanes, args=(2, _free_port(), str(tmp_path), dtype), nprocs=2, join=True)
    got = np.load(tmp_path / "lanes.npy")
    ref = _split(_direct([4242], 7, dtype)[0])
    if dtype == "f32":
        np.testing.assert_array_equal(got, ref)
    else:
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 2e-2
