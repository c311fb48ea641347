"""Summaries of an `ncu --page source --csv --print-source sass` export (profiles/r02_ncu_*_source.txt):
per-opcode shares of executed warp-instructions and of stall samples, stall reasons, and code
regions in 0x800-byte buckets.

    ncu -i prof.ncu-rep --page source --csv --print-source sass > src.csv
    python scripts/ncu_source_mix.py src.csv
"""
import csv
import re
import sys
from collections import Counter


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    return {h: i for i, h in enumerate(hdr)}, rows[2:], hdr


def opcode_mix(ix, data):
    tot_e = tot_s = 0
    ops, samp = Counter(), Counter()
    for r in data:
        try:
            ex = int(r[ix["Instructions Executed"]])
            s = int(r[ix["Warp Stall Sampling (All Samples)"]])
        except ValueError:
            continue
        src = r[ix["Source"]].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0] if src else "?"
        ops[op] += ex
        samp[op] += s
        tot_e += ex
        tot_s += s
    print("total warp-instr executed", tot_e, "samples", tot_s)
    for op, c in ops.most_common(45):
        print(f"{op:28s} {c / tot_e * 100:6.2f}%  samples {samp[op] / tot_s * 100:6.2f}%")


def stall_reasons(ix, data, hdr):
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = Counter()
    for r in data:
        for c in cols:
            try:
                tot[c] += int(r[ix[c]])
            except ValueError:
                pass
    s = sum(tot.values())
    for c, v in tot.most_common(14):
        print(f"{c:28s} {v / s:.3f}")


def regions(ix, data):
    base = int(data[0][0], 16)
    buckets = {}
    for r in data:
        a = int(r[0], 16) - base
        ex = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        d = buckets.setdefault(a // 0x800, [0, 0])
        d[0] += ex
        d[1] += s
    te = sum(v[0] for v in buckets.values())
    ts = sum(v[1] for v in buckets.values())
    for b in sorted(buckets):
        e, s = buckets[b]
        if e / te > 0.003 or s / ts > 0.003:
            print(f"{b * 0x800:#8x} exec {e / te * 100:5.1f}% samp {s / ts * 100:5.1f}%")


if __name__ == "__main__":
    ix, data, hdr = load(sys.argv[1])
    opcode_mix(ix, data)
    print()
    stall_reasons(ix, data, hdr)
    print()
    regions(ix, data)
