"""Dev tool: ms/scene of one (N, K) point at the bench shape (env knobs apply).
    python tools/sweep_point.py N K"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_08975_b200 as alpa  # noqa: E402

n, K = int(sys.argv[1]), int(sys.argv[2])
cfg = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=36,
                       action_hidden_dim=2048, kv_dim=1024, heads=8, diffusion_iters=K, dtype="bf16")
g = alpa.ActionGenerator(cfg)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
g.set_stream(stream.cuda_stream)
g.bind_prefix_synthetic(4242, 2048)
req = alpa.InferenceRequest(num_trajectories=n, diffusion_iters=K, v0=5.0)
noise = torch.from_numpy(alpa.host_noise(2, 1, n)).cuda()
a = torch.empty((n, 64, 2), device="cuda")
t = torch.empty((n, 64, 3), device="cuda")
for _ in range(3):
    g.generate_device(req, noise.data_ptr(), a.data_ptr(), t.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(stream)
for _ in range(5):
    g.generate_device(req, noise.data_ptr(), a.data_ptr(), t.data_ptr())
e1.record(stream)
torch.cuda.synchronize()
print(f"N={n} K={K} {os.environ.get('ALPA_MK_SPLITS', '')} {os.environ.get('ALPA_MK_TN', '')}: "
      f"{e0.elapsed_time(e1) / 5:.3f} ms/scene finite={bool(torch.isfinite(a).all())}")
