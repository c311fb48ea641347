"""Per-CUDA-source-line totals from `ncu --page source --csv --print-source cuda`: executed
warp-instructions and stall samples per line, sorted; python scripts/ncu_cuda_lines.py f.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
out = []
cur_file = ""
for r in rows[hi + 1:]:
    if len(r) < len(hdr):
        if r and r[0].strip().startswith("/"):
            cur_file = r[0].strip()
        continue
    try:
        ex = int(r[ix["Instructions Executed"]] or 0)
        sm = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    out.append((ex, sm, r[0], r[ix["Source"]].strip()[:110]))
tot = sum(o[0] for o in out) or 1
tots = sum(o[1] for o in out) or 1
print("total executed", tot, "samples", tots)
for ex, sm, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * ex / tot:6.2f}% ex {100 * sm / tots:6.2f}% smp  L{ln}: {src}")
