"""Summarise an ncu --page source --print-source sass CSV: hottest SASS
instructions by warp-stall samples, with their dominant stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[key] or 0) for d in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(float(d[h] or 0) for d in data) for h in stalls}
print("total samples", tot)
print("stalls:", sorted(((round(100 * v / tot, 1), h) for h, v in agg.items() if v), reverse=True)[:8])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for d in sorted(data, key=lambda d: -float(d[key] or 0))[:n]:
    s = float(d[key] or 0)
    top = sorted(((float(d[h] or 0), h) for h in stalls), reverse=True)[:2]
    print(f"{100*s/tot:5.1f}% {d['Address']:>6} {d['Source'][:60]:60} exe={d['Instructions Executed']:>10} "
          + " ".join(f"{h[6:]}={int(v)}" for v, h in top if v))
