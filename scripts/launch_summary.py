"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: launches and device
time per kernel, in launch order segments (consecutive runs of the same grid shape).

    python scripts/launch_summary.py launches.csv
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
tot = OrderedDict()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0]
    key = (name, r[ix["Grid Size"]], r[ix["Block Size"]])
    unit = r[ix["Metric Unit"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    v = v / 1e3 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1e3
    d = tot.setdefault(key, [0, 0.0])
    d[0] += 1
    d[1] += v
print(f"{'kernel':28s} {'grid':>10s} {'block':>8s} {'launches':>8s} {'total us':>12s} {'avg us':>10s}")
for (name, g, b), (n, us) in tot.items():
    print(f"{name:28s} {g:>10s} {b:>8s} {n:8d} {us:12.1f} {us / n:10.1f}")
