"""Dev tool: per-source-line warp-stall samples from an ncu report's source page.
    ncu -i rep --page source --csv --print-source cuda,sass > mix.csv
    python tools/ncu_lines.py mix.csv [top] [line_lo line_hi]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rng = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else None
hdr = None
fname, line, src = "", 0, ""
agg = collections.defaultdict(lambda: collections.Counter())
srcs = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0] and r[0].isdigit():
        line = int(r[0])
        srcs[(fname, line)] = ",".join(r[1:len(r) - len(hdr) + 2]) if len(r) > len(hdr) else r[1]
        continue
    if len(r) == len(hdr) and r[2].startswith("0x"):
        c = agg[(fname, line)]
        for k in range(4, len(hdr)):
            name = hdr[k]
            if name.startswith("stall_") and "Not Issued" not in name or name == "Warp Stall Sampling (All Samples)":
                try:
                    c[name] += int(r[k])
                except ValueError:
                    pass
tot = sum(c["Warp Stall Sampling (All Samples)"] for c in agg.values())
items = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])
if rng:
    items = sorted([kv for kv in agg.items() if rng[0] <= kv[0][1] <= rng[1] and kv[0][0] == "mk.cuh"])
print(f"total samples {tot}")
for (f, l), c in items[:top] if not rng else items:
    s = c["Warp Stall Sampling (All Samples)"]
    if s == 0:
        continue
    rs = sorted(((v, k[6:]) for k, v in c.items() if k.startswith("stall_")), reverse=True)[:3]
    print(f"{f}:{l:5d} {s:7d} {100.0 * s / tot:5.1f}%  " + " ".join(f"{k}={100.0 * v / s:.0f}%" for v, k in rs) +
          f"   | {srcs.get((f, l), '')[:70].strip()}")
