"""Dev tool: SASS bytes of the persistent kernel per source line (I-cache budget).

    python tools/sass_size.py [--tn 192] [--hd 128] [--top 30]
"""
import argparse
import collections
import os
import re
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--tn", type=int, default=192)
ap.add_argument("--hd", type=int, default=128)
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--tr", action="store_true", help="the instrumented twin")
a = ap.parse_args()
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "mk.sm_100a.cubin",
                    os.path.join(ROOT, "paper_2605_08975_b200", "libalpa_action.so")], cwd=d, check=True,
                   capture_output=True)
    txt = subprocess.run(["nvdisasm", "-gi", os.path.join(d, "mk.sm_100a.cubin")], capture_output=True,
                         text=True, check=True).stdout
name = f"_ZN4alpa2mk11iter_kernelILi{a.tn}ELi{a.hd}ELb{int(a.tr)}EEEvNS0_6ParamsE"
beg = txt.index(f".text.{name}:")
end = txt.find("\n.text.", beg + 10)
body = txt[beg:end if end > 0 else None].split("\n")
src = {}
cur = None
cnt = collections.Counter()
total = 0
for l in body:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    if re.search(r"/\*[0-9a-f]{4,}\*/", l):
        total += 16
        if cur:
            cnt[cur] += 16
print(f"{name}: {total} B")
for (f, ln), c in cnt.most_common(a.top):
    if f not in src:
        src[f] = open(f).read().split("\n") if os.path.exists(f) else []
    s = src[f][ln - 1].strip()[:80] if ln - 1 < len(src[f]) else ""
    print(f"{c:6d} {os.path.basename(f)}:{ln:<5d} {s}")
