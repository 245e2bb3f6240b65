"""Dev tool: one small bf16 config through the default path (hang / parity triage).
    python tools/small_bf16.py [ah kv heads r n B K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_08975_b200 as alpa  # noqa: E402
from oracle.oracle import Cfg, Port  # noqa: E402

a = [int(v) for v in sys.argv[1:]] or [256, 128, 2, 100, 6, 2, 3]
ah, kv, heads, r, n, B, K = a
port = Port()
m = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=B, action_hidden_dim=ah,
                     kv_dim=kv, heads=heads, diffusion_iters=K, dtype="bf16")
oc = Cfg.make(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=B, action_hidden_dim=ah, kv_dim=kv,
              heads=heads, diffusion_iters=K)
pre = port.synthetic_prefix(7, B, r, kv)
with alpa.ActionGenerator(m) as g:
    g.bind_prefix(pre)
    res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=n, v0=5.0, executor="eager"))
exp = port.refine(oc, port.weights(oc), pre, port.noise(2, 1, n))
print("ok rel-L2", float(np.linalg.norm(res.actions - exp) / np.linalg.norm(exp)))
