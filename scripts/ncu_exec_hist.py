"""How much distinct code a kernel walks, by how often a warp runs it: from `ncu --page source --csv
--print-source sass` (src.csv) and the warp count of the launch.
    python scripts/ncu_exec_hist.py src.csv <warps in the launch>"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
W = float(sys.argv[2])
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
names = ["hot (>= 8 per warp)", "2-8 per warp", "about once per warp (0.5-2)", "0.05-0.5", "< 0.05"]
lines = Counter()
ins = Counter()
ops = {n: Counter() for n in names}
for r in data:
    e = int(r[ix["Instructions Executed"]] or 0)
    if e == 0:
        continue
    x = e / W
    k = names[0] if x >= 8 else names[1] if x >= 2 else names[2] if x >= 0.5 else names[3] if x >= 0.05 else names[4]
    lines[k] += 1
    ins[k] += e
    src = r[ix["Source"]].strip()
    ops[k][re.sub(r"^@!?U?P\w+\s+", "", src).split()[0]] += 1
tot = sum(ins.values())
print("kernel SASS lines", len(data), "executed lines", sum(lines.values()), "warps", int(W))
for k in names:
    print(f"{k:30s} lines {lines[k]:6d}  {lines[k] * 16 / 1024:7.1f} KB  exec share {100 * ins[k] / tot:5.1f} %   "
          f"per warp {ins[k] / W:8.0f}   top: {ops[k].most_common(8)}")
