"""Dev tool: run a small bf16 config with the soft watchdog + trace and print,
per op, which CTAs published (ALPA_MK_DEBUG=1 ALPA_MK_TRACE=1)."""
import ctypes as C, os, sys
import numpy as np
os.environ["ALPA_MK_DEBUG"] = "1"
os.environ["ALPA_MK_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08975_b200 as alpa
from oracle.oracle import Port
port = Port()
kv = int(sys.argv[1]) if len(sys.argv) > 1 else 128
m = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=1, action_hidden_dim=256,
                     kv_dim=kv, heads=2, diffusion_iters=1, dtype="bf16")
g = alpa.ActionGenerator(m)
g.bind_prefix(port.synthetic_prefix(7, 1, 100, kv))
req = alpa.InferenceRequest(num_trajectories=6, v0=5.0)
prof = g.profile(req, iters=1)
L = alpa.lib()
L.alpa_debug_mk_trace.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
buf = np.zeros(1 << 22, np.uint64)
nops, grid = C.c_int64(), C.c_int64()
print("trace rc", L.alpa_debug_mk_trace(g._h, buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size, C.byref(nops), C.byref(grid)))
tr = buf[: nops.value * grid.value * 16].reshape(nops.value, grid.value, 16)
for o in range(nops.value):
    pub = np.nonzero(tr[o, :, 5])[0]
    acc = np.nonzero(tr[o, :, 3])[0]
    mma = np.nonzero(tr[o, :, 2])[0]
    print(f"op {o}: published {list(pub)[:40]}  acc {list(acc)[:40]}  mma1 {list(mma)[:40]}")
