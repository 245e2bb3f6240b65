"""Dev tool: GEMM MMA-thread accounting per op of one block (clock64 stamps of the
traced twin): first stage landed -> last MMA issued, the part spent waiting for
landed stages, k-blocks, cycles per k-block issued.
    python tools/gemm_clk.py trace.npz [block]"""
import sys
import numpy as np

tr = np.load(sys.argv[1])["trace"]
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for k, name in [(0, "qkv"), (2, "o"), (3, "mlp1"), (4, "mlp2")]:
    r = tr[3 + 5 * blk + k].astype(np.int64)
    r = r[r[:, 64] > 0]
    span = r[:, 65] - r[:, 64]
    wait = r[:, 66]
    kb = r[:, 67]
    print(f"{name:5s} items {len(r):3d}  k-blocks {int(np.median(kb)):3d}  mainloop {np.median(span):7.0f} cyc  "
          f"waiting {np.median(wait):7.0f}  busy/k-block {np.median((span - wait) / np.maximum(kb - 1, 1)):6.0f}")
