"""Dev tool: per-op critical-path timeline of the persistent iteration kernel.

    ALPA_MK_TRACE=1 python tools/mk_trace.py [--blocks 4] [--n 6]

Prints, per op of the last profiled iteration, event times (us) relative to the
previous op's completion: median and max over CTAs that processed an item.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

os.environ.setdefault("ALPA_MK_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08975_b200 as alpa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--blocks", type=int, default=4)
ap.add_argument("--n", type=int, default=6)
ap.add_argument("--r", type=int, default=2048)
ap.add_argument("--dump", default="", help="save the raw per-CTA trace (npz)")
ap.add_argument("--extra", action="store_true", help="split finalisation / attention merge sub-phases")
a = ap.parse_args()
cfg = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=a.blocks,
                       action_hidden_dim=2048, kv_dim=1024, heads=8, diffusion_iters=2, dtype="bf16")
g = alpa.ActionGenerator(cfg)
g.bind_prefix_synthetic(4242, a.r)
req = alpa.InferenceRequest(num_trajectories=a.n, v0=5.0)
try:
    g.run_action_generation(req)
except alpa.InternalError as e:  # debug flags may produce garbage actions
    print('note:', e)
prof = g.profile(req, iters=2)
L = alpa.lib()
L.alpa_debug_mk_trace.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int64,
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
buf = np.zeros(4 << 20, np.uint64)
nops, grid = C.c_int64(), C.c_int64()
rc = L.alpa_debug_mk_trace(g._h, buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size,
                           C.byref(nops), C.byref(grid))
assert rc == 0, rc
NS = 128  # mk::TR_NSLOT
tr = buf[: nops.value * grid.value * NS].reshape(nops.value, grid.value, NS).astype(np.int64)
if a.dump:
    np.savez_compressed(a.dump, trace=tr)
names = [p["name"][5:] for p in prof if p["name"].startswith("span:")]
spans = {p["name"][5:]: p for p in prof if p["name"].startswith("span:")}
ev = ["dep", "mma1", "acc", "acc9", "loop", "loop9", "bar", "drain", "meet", "fix", "pub"]
order = [0, 2, 3, 12, 10, 13, 11, 7, 4, 8, 5]
if a.extra:
    ev = ["dep", "mma0", "sm0", "smx", "mma1", "acc", "loop", "merge", "meet", "fixin", "fixv0", "fixc0", "fixc1", "fixc2", "fixed", "store", "stats",
          "fix", "fence", "pub"]
    order = [0, 1, 25, 26, 2, 3, 10, 22, 4, 23, 24, 16, 17, 18, 19, 20, 21, 8, 9, 5]
t0 = tr[tr > 0].min()
prev_done = t0
tags = []
# op tags in plan order: encode, enc1, enc2, (qkv, attn, o, mlp1, mlp2)*B, head
tags = ["encode", "gemm_enc_mlp1", "gemm_enc_mlp2"] + \
    ["gemm_qkv", "attention", "gemm_o", "gemm_mlp1", "gemm_mlp2"] * a.blocks + ["head_update"]
print(f"{'op':16s} " + " ".join(f"{e:>11s}" for e in ev) + "   span")
for o in range(nops.value):
    row = tr[o]
    act = row[:, 5] > 0
    out = []
    for k in order:
        v = row[act, k]
        v = v[v > 0]
        if len(v):
            rel = (v - prev_done) / 1000.0
            out.append(f"{np.median(rel):5.1f}/{rel.max():5.1f}")
        else:
            out.append(" " * 11)
    done = row[act, 5].max() if act.any() else prev_done
    print(f"{tags[o] if o < len(tags) else o:16s} " + " ".join(out) + f"  {(done - prev_done) / 1000:6.1f}")
    prev_done = done
