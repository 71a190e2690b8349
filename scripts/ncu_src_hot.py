"""Top CUDA source lines of an ncu source page (cuda,sass view) by warp-stall samples (developer tool).

    ncu -i rep --page source --csv --print-source cuda,sass | python scripts/ncu_src_hot.py [N]
"""
import csv
import sys

N = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rows = list(csv.reader(sys.stdin))
hdr = next(r for r in rows if r and r[0] == "Line No")
idx = {}
for i, h in enumerate(hdr):
    idx.setdefault(h, i)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
lines = [r for r in rows if r and r[0].isdigit() and len(r) == len(hdr)]
tot = sum(float(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in lines)
print(f"total samples {tot:.0f}")
agg = {}
for r in lines:
    s = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    st = sorted(((float(r[idx[k]] or 0), k[6:]) for k in stalls), reverse=True)[:2]
    agg[int(r[0])] = (s, r[1].strip(), st, float(r[idx["Instructions Executed"]] or 0))
for ln, (s, src, st, ie) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    tops = " ".join(f"{k}:{v / tot * 100:.1f}" for v, k in st)
    print(f"{s / tot * 100:5.2f}%  L{ln:<5d} inst {ie / 1e6:8.1f}M  [{tops}]  {src[:110]}")
