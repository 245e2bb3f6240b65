"""Dev tool: build a config-2-width context and run scenes (for ncu captures).

    python tools/run_iteration.py [--blocks 2] [--scenes 1] [--eager] [--n 6]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08975_b200 as alpa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--blocks", type=int, default=2)
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--scenes", type=int, default=1)
ap.add_argument("--n", type=int, default=6)
ap.add_argument("--r", type=int, default=2048)
ap.add_argument("--eager", action="store_true")
a = ap.parse_args()
cfg = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=a.blocks,
                       action_hidden_dim=2048, kv_dim=1024, heads=8, diffusion_iters=a.iters,
                       dtype="bf16")
g = alpa.ActionGenerator(cfg)
g.bind_prefix_synthetic(4242, a.r)
req = alpa.InferenceRequest(num_trajectories=a.n, v0=5.0,
                            executor="eager" if a.eager else "graph")
for _ in range(a.scenes):
    res = g.run_action_generation(req)
print("ok", res.stats, float(abs(res.actions).mean()))
