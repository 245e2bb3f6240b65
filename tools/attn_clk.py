"""Dev tool: cycle-precise attention pipeline of one block (clock64 stamps of the
traced twin, tools/mk_trace.py --dump): median cycles after the item's Q landed.
    python tools/attn_clk.py trace.npz [block]"""
import sys
import numpy as np

tr = np.load(sys.argv[1])["trace"]
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 2
row = tr[3 + 5 * blk + 1].astype(np.int64)
r = row[row[:, 64] > 0]


def med(i):
    v = r[:, i]
    ok = v > 0
    return np.median(v[ok] - r[ok, 64]) if ok.any() else float("nan")


names = [("K/V seen", 65), ("S issued", 71), ("PV issued", 83), ("S ready", 89), ("S read", 95), ("exps", 101), ("P slot", 107),
         ("P pub", 113)]
print("block " + "".join(f"{n:>11s}" for n, _ in names))
for j in range(6):
    print(f"{j:5d} " + "".join(f"{med(i + j)   :11.0f}" for _, i in names))
print(f"all MMAs done {med(119):.0f}  merge+partials stored {med(120):.0f}  (cycles)")
