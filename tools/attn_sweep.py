"""Dev tool: attention kernel time vs KV splits / prefix length (eager, CUDA events)."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import paper_2605_08975_b200 as alpa
    r = int(sys.argv[1]); n = int(sys.argv[2])
    cfg = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=1,
                           action_hidden_dim=2048, kv_dim=1024, heads=8, diffusion_iters=1, dtype="bf16")
    g = alpa.ActionGenerator(cfg)
    g.bind_prefix_synthetic(4242, r)
    req = alpa.InferenceRequest(num_trajectories=n, v0=5.0)
    g.profile(req, 1)
    best = min((p for p in g.profile(req, 3) if p["name"] == "attention"), key=lambda p: p["total_ms"])
    print(json.dumps({"r": r, "n": n, "splits": os.environ.get("ALPA_ATTN_SPLITS"), "us": best["total_ms"] / best["launches"] * 1e3}))
else:
    for r in (512, 2048):
        for s in ("1", "2", "3", "6", "8"):
            env = dict(os.environ, ALPA_ATTN_SPLITS=s)
            out = subprocess.run([sys.executable, __file__, str(r), "6"], env=env, capture_output=True, text=True, timeout=60)
            print(out.stdout.strip() or out.stderr[-300:])
