"""Attribute an ncu SASS source-page export (--page source --csv --print-source sass) to CUDA
source lines, using nvdisasm -gi line info of the same cubin.
usage: sass_lines.py <ncu_sass.csv> <nvdisasm -gi output> <function-substring> [top]"""
import csv
import re
import sys
from collections import defaultdict

csv_path, dis_path, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(dis_path).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and fn in l)
loc = {}
cur = "?"
fresh = True  # the first marker after an instruction is the innermost frame
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if fresh:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            m2 = re.search(r'inlined at "([^"]+)", line (\d+)', l)
            if m2:
                cur += f" <- {m2.group(1).split('/')[-1]}:{m2.group(2)}"
            fresh = False
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,6})\*/", l)
    if m:
        loc[int(m.group(1), 16)] = cur
        fresh = True
rows = list(csv.reader(open(csv_path)))
h = rows[1]
data = rows[2:]
ia, iss, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
base = int(data[0][ia], 16)
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
for r in data:
    off = int(r[ia], 16) - base
    key = loc.get(off, "?")
    a = agg[key]
    a[0] += float(r[iss] or 0)
    a[1] += float(r[iex] or 0)
    for c in stall_cols:
        a[2][c] += float(r[h.index(c)] or 0)
tot = sum(a[0] for a in agg.values())
print(f"total samples {tot:.0f}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    st = sorted(a[2].items(), key=lambda kv: -kv[1])[:3]
    print(f"{a[0]:6.0f} {100*a[0]/tot:5.1f}% inst {a[1]:9.0f}  {k[:70]:70s} " + " ".join(f"{s[6:]}={v:.0f}" for s, v in st))
