"""Hottest CUDA source lines of an `ncu --page source --csv --print-source cuda,sass`
export: warp-stall samples aggregated per source line (inlined intrinsics are
attributed to their header), with executed instructions and average active
threads.  python scripts/ncu_lines.py export.csv [top_n]"""
import csv
import os
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, hdr = None, None
lines = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 11 or not r[0]:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = float(r[4] or 0)
        ex = float(r[7] or 0)
        tix = float(r[8] or 0) if r[8] not in ("-", "") else 0.0
        th = tix / ex if ex else 0.0  # average active threads per executed instruction
    except ValueError:
        continue
    lines.append((s, fname, r[0], r[1].strip()[:90], ex, th))
tot = sum(x[0] for x in lines)
print(f"total samples {tot:.0f}")
by_file = {}
for s, f, *_ in lines:
    by_file[f] = by_file.get(f, 0) + s
print("by file:", ", ".join(f"{f} {100 * v / tot:.1f}%" for f, v in
                            sorted(by_file.items(), key=lambda x: -x[1])))
for s, f, ln, src, ex, th in sorted(lines, key=lambda x: -x[0])[:n]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5} exec={ex:>12.0f} thr={th:5.1f}  {src}")
