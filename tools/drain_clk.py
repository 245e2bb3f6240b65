"""Dev tool: GEMM epilogue drain phases per op of one block (clock64, traced twin):
cycles after the accumulator is ready for chunk c (16 tokens of the warp half):
TMEM data in registers / values staged / half barrier passed / TMA store issued.
    python tools/drain_clk.py trace.npz [block]"""
import sys
import numpy as np

tr = np.load(sys.argv[1])["trace"]
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for k, name in [(0, "qkv"), (2, "o"), (3, "mlp1")]:
    r = tr[3 + 5 * blk + k].astype(np.int64)
    r = r[r[:, 68] > 0]
    base = r[:, 68]
    out = []
    for c in range(4):
        ph = []
        for q in range(4):
            v = r[:, 72 + 4 * c + q]
            ok = v > 0
            ph.append(np.median(v[ok] - base[ok]) if ok.any() else float("nan"))
        out.append("/".join(f"{x:5.0f}" for x in ph))
    print(f"{name:5s} drain end {np.median(r[:, 69] - base):6.0f}  chunks (ld/staged/bar/store): " + "  ".join(out))
