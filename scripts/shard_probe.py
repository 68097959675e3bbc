"""Time single shards of a big run (estimate the whole run from a slice).

    python scripts/shard_probe.py --workload rmat22 --k 7 --algo orient \
        --scheme vertex --world 16 --ranks 0 7 15

Each listed rank's root range (kc_shard_ranges, cost-balanced) is counted
alone with device_count_raw; one JSON line per shard with its device ms,
visits and raw limbs.  With KC_TIMING=1 the library prints per-launch times.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import paper_2104_13209_b200 as kc  # noqa: E402
from paper_2104_13209_b200.orientation import rank_and_orient  # noqa: E402
from paper_2104_13209_b200.scheduler import device_count_raw, finalize  # noqa: E402
from paper_2104_13209_b200.shard import shard_ranges  # noqa: E402

from explore import cached_edges  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="rmat22")
    ap.add_argument("--k", type=int, default=7)
    ap.add_argument("--algo", default="orient")
    ap.add_argument("--scheme", default="vertex")
    ap.add_argument("--criterion", default="degeneracy")
    ap.add_argument("--world", type=int, default=16)
    ap.add_argument("--ranks", type=int, nargs="+", default=[0])
    ap.add_argument("--range", type=int, nargs=2, default=None,
                    help="explicit [lo, hi) of make_tasks order instead of shard ranks")
    a = ap.parse_args()
    g = kc.from_edges(cached_edges(a.workload))
    cfg = kc.RunConfig(k=a.k, algorithm=a.algo, scheme=a.scheme, criterion=a.criterion)
    t = time.perf_counter()
    og = rank_and_orient(g, a.criterion)
    orient_s = time.perf_counter() - t
    ranges = shard_ranges(og, cfg, a.world)
    print(json.dumps({"workload": a.workload, "n": g.n, "m": g.m, "d_max": og.d_max,
                      "orient_s": round(orient_s, 3), "world": a.world,
                      "ranges": ranges}), flush=True)
    todo = [(r, ranges[r]) for r in a.ranks] if a.range is None else [(-1, tuple(a.range))]
    for r, (lo, hi) in todo:
        t = time.perf_counter()
        raw = device_count_raw(og, cfg, lo, hi)
        if raw.hist is not None:
            h = np.asarray(raw.hist)
            bad = [(int(i), int(j), int(h[i, j])) for i, j in np.argwhere(h) if j > i]
            if bad:  # a leaf cannot have more pivots than path vertices
                print(json.dumps({"bad_hist_bins": bad[:20], "n_bad": len(bad)}), flush=True)
        try:
            count, _ = finalize(raw, cfg, g.n, g.m)
        except OverflowError as e:
            count = f"OverflowError: {e}"
        print(json.dumps({"rank": r, "lo": lo, "hi": hi, "algo": a.algo, "scheme": a.scheme,
                          "k": a.k, "count": str(count),
                          "wall_s": round(time.perf_counter() - t, 3),
                          "kernel_ms": raw.count_ms, "visits": int(raw.visits),
                          "limbs": [int(x) for x in raw.limbs], "word_ops": int(raw.word_ops),
                          "hist_sum": int(np.asarray(raw.hist, dtype=np.uint64).sum()) if raw.hist is not None else 0}),
              flush=True)


if __name__ == "__main__":
    main()
