"""Find loops (backward branches) in a cuobjdump -sass listing and print the opcode mix of each
loop body that contains MUFU (the step loops).   python scripts/sass_loops.py file.sass"""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\()?\.?L?_?x?[_0-9]*\)?\s*0x([0-9a-f]+)|BRA\s+0x([0-9a-f]+)", t)
    if not m:
        continue
    tgt = int(m.group(1) or m.group(2), 16)
    if tgt >= a or tgt not in addr_idx:
        continue
    body = [x[1] for x in ins[addr_idx[tgt]:i + 1]]
    ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", b).split()[0] for b in body)
    nmufu = sum(v for k, v in ops.items() if k.startswith("MUFU"))
    if nmufu < 4:
        continue
    print(f"loop {tgt:#x}..{a:#x}: {len(body)} instrs, MUFU {nmufu}")
    print("   " + ", ".join(f"{k} {v}" for k, v in ops.most_common(18)))
