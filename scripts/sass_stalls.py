"""Summarise an `ncu --page source --csv` SASS dump: instruction mix and stall samples per opcode.

    python scripts/sass_stalls.py dump.csv
"""
import sys

import pandas as pd

df = pd.read_csv(sys.argv[1], skiprows=1)
df = df[df["Address"].astype(str).str.startswith("0x") | df["Address"].astype(str).str.isnumeric()]
num = lambda c: pd.to_numeric(df[c], errors="coerce").fillna(0)
df["op"] = df["Source"].astype(str).str.strip().str.replace(r"^@!?U?P\w+\s+", "", regex=True).str.split().str[0]
df["samples"] = num("Warp Stall Sampling (All Samples)")
df["exec"] = num("Instructions Executed")
cols = [c for c in df.columns if c.startswith("stall_") and "Not Issued" not in c]
for c in cols:
    df[c] = num(c)
g = df.groupby("op").agg({"exec": "sum", "samples": "sum", **{c: "sum" for c in cols}})
g = g.sort_values("samples", ascending=False)
tot_e, tot_s = g["exec"].sum(), g["samples"].sum()
print(f"total warp-instructions {tot_e:.3e}, stall samples {tot_s:.0f}")
print("stall reasons (share of samples):")
print((g[cols].sum() / tot_s).sort_values(ascending=False).head(12).round(3).to_string())
print("\nper opcode: exec share, sample share, top stalls")
for op, r in g.head(25).iterrows():
    top = r[cols].sort_values(ascending=False).head(3)
    print(f"{op:12s} exec {r['exec'] / tot_e:6.3f}  samples {r['samples'] / tot_s:6.3f}  " +
          " ".join(f"{k[6:]}={v / max(r['samples'], 1):.2f}" for k, v in top.items()))
