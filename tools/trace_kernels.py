"""Dev tool: per-CTA phase timeline (globaltimer) of the attention kernel and of
the last GEMM of an eager iteration (trace build: make -C paper_2605_08975_b200 trace)."""
import ctypes as C, os, sys
import numpy as np
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["ALPA_LIB"] = os.path.join(HERE, "paper_2605_08975_b200/build_trace/libalpa_trace.so")
os.environ.setdefault("ALPA_PDL", "0")
sys.path.insert(0, HERE)
import paper_2605_08975_b200 as alpa
L = alpa.lib()
r = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
cfg = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=1,
                       action_hidden_dim=2048, kv_dim=1024, heads=8, diffusion_iters=1, dtype="bf16")
g = alpa.ActionGenerator(cfg)
g.bind_prefix_synthetic(4242, r)
req = alpa.InferenceRequest(num_trajectories=6, v0=5.0, executor="eager")
g.run_action_generation(req)
L.alpa_debug_trace_clear()
g.run_action_generation(req)
buf = np.zeros((4096, 8), np.uint64)
L.alpa_debug_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 4096)
for name, base, labels in (("attention", 0, ["start", "setup", "q_loaded", "S0_ready", "softmax_done", "combine", "stored", "end"]),
                           ("gemm(last)", 2048, ["start", "setup", "first_stage", "mma_done", "staged", "cluster1", "stored", "end"])):
    blk = buf[base:base + 2048]
    blk = blk[blk[:, 0] > 0].astype(np.int64)
    if not len(blk):
        continue
    t0 = blk[:, 0].min()
    rel = (blk - t0) / 1000.0
    rel[blk == 0] = np.nan
    print(f"{name}: {len(blk)} CTAs, span {(np.nanmax(rel)):.1f} us")
    for i, lab in enumerate(labels):
        col = rel[:, i]
        print(f"   {lab:13s} min {np.nanmin(col):7.2f}  med {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f}")
