"""Summarize an ncu launch list (gpu__time_duration.sum) by kernel: count, total, share."""
import csv
import re
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.DictReader(lines))
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(CUtensorMap_st.*|\(.*", "", r["Kernel Name"]).replace("void ", "")
    name = f"{name} grid{r['Grid Size']}"
    agg[name][0] += 1
    agg[name][1] += float(r["Metric Value"]) / 1000.0
tot = sum(v[1] for v in agg.values())
print("| kernel (grid) | launches | total us | share |")
print("|---|---|---|---|")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f}% |")
print(f"\n{len(rows)} launches, {tot:.1f} us of kernel time (cold-cache, serialised by ncu)")
