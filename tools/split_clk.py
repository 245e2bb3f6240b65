"""Dev tool: split-K finalisation phases of MLP2 in one block (clock64, traced twin):
cycles after the partials of the other splits' rows were issued (drain done):
rendezvous passed / fix (own TMEM + 3 L2 partials -> fp32 staging) / fp32 rows stored /
row pass + bf16 copy stored / published.
    python tools/split_clk.py trace.npz [block]"""
import sys
import numpy as np

tr = np.load(sys.argv[1])["trace"]
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 2
r = tr[3 + 5 * blk + 4].astype(np.int64)
r = r[r[:, 90] > 0]
b = r[:, 90]
names = [("meet", 91), ("fixed", 92), ("e stored", 93), ("x stored", 94), ("published", 95)]
print("mlp2 split finalisation, cycles after the partial drain: " +
      "  ".join(f"{n} {np.median(r[:, i] - b):6.0f}" for n, i in names))
print("accumulator ready -> partial drain done:", np.median(r[:, 90] - r[:, 68]) if (r[:, 68] > 0).any() else "n/a")
