import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2605_08975_b200 as alpa
from oracle.oracle import Port, Cfg
port = Port()
r = int(sys.argv[1]); B=1
m = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=B, action_hidden_dim=256, kv_dim=128, heads=1, diffusion_iters=1, dtype="bf16")
oc = Cfg.make(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=B, action_hidden_dim=256, kv_dim=128, heads=1, diffusion_iters=1)
pre = port.synthetic_prefix(7, B, r, 128)
exp = port.refine(oc, port.weights(oc), pre, port.noise(2, 1, 2))
g = alpa.ActionGenerator(m); g.bind_prefix(pre)
res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=2, v0=5.0, executor="eager"))
print("r", r, "splits", os.environ.get("ALPA_ATTN_SPLITS"), "relL2", np.linalg.norm(res.actions-exp)/np.linalg.norm(exp), flush=True)
