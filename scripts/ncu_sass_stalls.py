"""Warp-stall samples of an ncu SASS source page, by opcode and hottest instructions (developer tool).

    ncu -i rep --page source --csv --print-source sass [--launch-skip k --launch-count 1] | python scripts/ncu_sass_stalls.py
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(sys.stdin))
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ins = [r for r in rows if r and r[0].startswith("0x") and len(r) == len(hdr)]
S = lambda r: float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
tot = sum(S(r) for r in ins)
by_op = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
for r in ins:
    op = r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]
    op = op.split(".")[0]
    d = by_op[op]
    d[0] += S(r)
    d[1] += float(r[ix["Instructions Executed"]] or 0)
    for k in stalls:
        d[2][k[6:]] += float(r[ix[k]] or 0)
print(f"total samples {tot:.0f}, instructions {len(ins)}")
for op, (s, ie, st) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:18]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{op:10s} {s / tot * 100:5.1f}%  exec {ie / 1e6:9.1f}M  " + " ".join(f"{k}:{v / tot * 100:.1f}" for k, v in top))
agg = defaultdict(float)
for r in ins:
    for k in stalls:
        agg[k[6:]] += float(r[ix[k]] or 0)
print("all: " + " ".join(f"{k}:{v / tot * 100:.1f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
