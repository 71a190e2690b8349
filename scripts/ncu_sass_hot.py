"""Aggregate an ncu source page (SASS) by stall reason / opcode (developer tool).

    ncu -i rep --page source --csv --print-source sass --kernel-id ::regex:NAME:K | python scripts/ncu_sass_hot.py
"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(sys.stdin))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
keys = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = defaultdict(float)
by_op = defaultdict(lambda: defaultdict(float))
top = []
for r in data:
    op = r[idx["Source"]].strip()
    opc = re.sub(r"^@!?U?P\w+\s+", "", op).split(" ")[0]
    s = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    top.append((s, op[:90]))
    for k in keys:
        v = float(r[idx[k]] or 0)
        tot[k] += v
        by_op[opc][k] += v
S = sum(tot.values())
print("total samples", S)
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {k:24s} {v / S * 100:5.1f}%")
print("by opcode (share of all samples; top stall)")
for opc, d in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
    s = sum(d.values())
    k, v = max(d.items(), key=lambda kv: kv[1])
    print(f"  {opc:14s} {s / S * 100:5.1f}%   {k} {v / S * 100:4.1f}%")
print("hottest instructions")
for s, op in sorted(top, reverse=True)[:25]:
    print(f"  {s / S * 100:5.2f}%  {op}")
