"""Instruction mix per kernel (and of its hottest loop) from cuobjdump -sass output."""
import re
import subprocess
import sys
from collections import Counter

path = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ins = []
    for l in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    loops = []
    for addr, txt in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d\s*,\s*)?(?:`\()?\.?L?_?x?_?\w*?\s*0x([0-9a-f]+)", txt)
        if m and int(m.group(1), 16) < addr:
            tgt = int(m.group(1), 16)
            body = [t for a, t in ins if tgt <= a <= addr]
            loops.append(body)
    print(name, "total", len(ins))
    for body in sorted(loops, key=len, reverse=True)[:2]:
        c = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body)
        print("  loop", len(body), c.most_common(16))
