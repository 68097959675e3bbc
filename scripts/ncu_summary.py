"""Summarise ncu reports / launch lists into markdown for profiles/.

    python scripts/ncu_summary.py report.ncu-rep [--top 25] > profiles/x.md
    python scripts/ncu_summary.py --launches launches.csv > profiles/y.md
"""

import argparse
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread",
    "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem",
    "Theoretical Occupancy", "Achieved Occupancy", "Executed Ipc Active", "Issue Slots Busy",
    "SM Busy", "Warp Cycles Per Issued Instruction", "No Eligible",
    "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size",
    "Block Size",
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed.sum", "smsp__inst_executed.sum"]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def details(rep):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "details", "--csv"]))))
    h = rows[0]
    out = defaultdict(dict)
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (d["ID"], d["Kernel Name"])
        if d["Metric Name"] in METRICS:
            out[key][d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    return out


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    h = rows[0]
    out = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        out[(d["ID"], d["Kernel Name"])] = {m: d.get(m) for m in RAW if m in d}
    return out


def hot_sass(rep, top):
    rows = list(csv.reader(io.StringIO(
        ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    hdr, data, seen = None, [], 0
    for r in rows:  # one section per kernel; keep the first
        if r and r[0] == "Address":
            seen += 1
            if seen > 1:
                break
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    if not data:
        return []
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(d[key] or 0) for d in data) or 1.0
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {h: sum(float(d[h] or 0) for d in data) for h in stalls}
    lines = ["stall mix: " + ", ".join(f"{h[6:]} {100 * v / tot:.1f}%" for v, h in
                                       sorted(((v, h) for h, v in agg.items() if v),
                                              reverse=True)[:6])]
    for d in sorted(data, key=lambda d: -float(d[key] or 0))[:top]:
        s = float(d[key] or 0)
        lines.append(f"{100 * s / tot:5.1f}%  {d['Source'][:70]:70s} exec={d['Instructions Executed']}")
    return lines


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        ms = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:90]
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values()) or 1.0
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{n}` | {c} | {v:.3f} | {100 * v / tot:.1f}% |")
    print(f"\ntotal {tot:.3f} ms over {sum(c for c, _ in agg.values())} launches "
          "(ncu-serialised, cold cache: compare shares, not absolutes)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--launches")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    if a.launches:
        launches(a.launches)
        return
    det = details(a.report)
    rw = raw(a.report)
    for key, m in det.items():
        print(f"### launch {key[0]}: `{key[1][:120]}`\n")
        for name in METRICS:
            if name in m:
                print(f"- {name}: {m[name]}")
        for name, v in (rw.get(key) or {}).items():
            print(f"- {name}: {v}")
        print()
    print("### hottest SASS (first profiled kernel, warp-stall samples)\n```")
    for ln in hot_sass(a.report, a.top):
        print(ln)
    print("```")


if __name__ == "__main__":
    sys.exit(main())
