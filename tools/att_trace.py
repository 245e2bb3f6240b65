"""Dev tool: per-64-key-block event times of attention items from a
tools/mk_trace.py --dump npz (us relative to the previous op's completion).
    python tools/att_trace.py trace.npz [op_index]"""
import sys
import numpy as np

tr = np.load(sys.argv[1])["trace"]
o = int(sys.argv[2]) if len(sys.argv) > 2 else 9
prev = tr[o - 1][:, 5]
t_prev = prev[prev > 0].max()
row = tr[o]
act = row[:, 5] > 0
names = {0: "dep", 6: "pre", 2: "mma1", 3: "acc", 25: "sm0", 26: "smx", 22: "merge", 4: "meet", 5: "pub"}
for j in range(5):
    names[37 + j] = f"L{j}"
    names[42 + j] = f"F{j}"
    names[32 + j] = f"S{j}"
    names[27 + j] = f"SM{j}"
order = [6, 0] + [37, 42, 32, 27] * 0
for j in range(6):
    names[48 + j] = ["sxS", "sxRd", "sxExp", "sxPf", "sxSt", "sxArr"][j]
cols = [6, 0, 37, 38, 39, 40, 41, 42, 43, 44, 45, 46, 32, 33, 34, 35, 36, 25, 27, 28, 29, 30, 31, 26, 2, 3, 22, 4, 5, 48, 49, 50, 51, 52, 53]
for k in cols:
    v = row[act, k]
    v = v[v > 0]
    if len(v):
        rel = (v - t_prev) / 1000.0
        print(f"{names[k]:>6s}  med {np.median(rel):6.2f}  min {rel.min():6.2f}  max {rel.max():6.2f}  n={len(v)}")
