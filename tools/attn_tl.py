"""Dev tool: per-block attention timeline of one block (trace npz from tools/quick.sh)."""
import sys
import numpy as np
tr = np.load(sys.argv[1])['trace']
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 2
base = 3 + 5 * blk
prev = tr[base][:, 5].max()  # qkv done
row = tr[base + 1]
act = row[:, 5] > 0
cols = [('dep', 0), ('mma0', 1), ('sm0', 25)] + [(f'L{j}', 37 + j) for j in range(5)] + \
       [(f'F{j}', 42 + j) for j in range(5)] + [(f'S{j}', 32 + j) for j in range(5)] + [(f'P{j}', 27 + j) for j in range(5)] + \
       [('smx', 26), ('acc', 3), ('merge', 22), ('meet', 4), ('fix', 8), ('pub', 5)]
for nm, i in cols:
    v = row[act, i]
    v = (v[v > 0] - prev) / 1000
    if len(v):
        print(f"{nm:6s} med {np.median(v):6.2f} max {v.max():6.2f} min {v.min():6.2f}")
