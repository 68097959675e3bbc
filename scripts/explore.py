"""Measure run_count over the BASELINE.json configs (one JSON line per run).

    python scripts/explore.py --workload rmat18 --k 4 7 --algo orient pivot \
        --scheme vertex edge --criterion degeneracy [--oracle-workers 0]

Graphs come from paper_2104_13209_b200.synth (seeded); edges are cached as
.npy under $KC_GRAPH_CACHE (default ./_graphs) so repeated subprocesses skip
generation.  Timings: orient_ms / count_ms are host wall times around the
device calls (each ends in a stream sync); device_ms are CUDA-event times.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2104_13209_b200 as kc  # noqa: E402
from paper_2104_13209_b200 import synth  # noqa: E402


def cached_edges(name):
    d = os.environ.get("KC_GRAPH_CACHE", "_graphs")
    os.makedirs(d, exist_ok=True)
    p = os.path.join(d, f"{name}.npy")
    if os.path.exists(p):
        return np.load(p)
    e = synth.workload(name)
    np.save(p, e)
    return e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="er2000")
    ap.add_argument("--k", type=int, nargs="+", default=[4])
    ap.add_argument("--algo", nargs="+", default=["orient"])
    ap.add_argument("--scheme", nargs="+", default=["vertex"])
    ap.add_argument("--criterion", nargs="+", default=["degree"])
    ap.add_argument("--group", type=int, nargs="+", default=[0])
    ap.add_argument("--all-k", action="store_true")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--oracle-workers", type=int, default=0,
                    help="also run the C oracle with this many threads (0 = skip)")
    a = ap.parse_args()
    t = time.perf_counter()
    edges = cached_edges(a.workload)
    gen_s = time.perf_counter() - t
    t = time.perf_counter()
    g = kc.from_edges(edges)
    print(json.dumps({"workload": a.workload, "n": g.n, "m": g.m, "gen_s": round(gen_s, 2),
                      "from_edges_s": round(time.perf_counter() - t, 3),
                      "build_ms": g.build_ms, "d_max_und": g.max_degree()}), flush=True)
    for crit in a.criterion:
        for algo in a.algo:
            for scheme in a.scheme:
                for k in a.k:
                    for gs in a.group:
                        cfg = kc.RunConfig(k=k, algorithm=algo, scheme=scheme, criterion=crit,
                                           all_k=a.all_k, group_size=gs)
                        best = None
                        for _ in range(a.reps):
                            rep = kc.run_count(g, cfg)
                            tot = rep.orient_ms + rep.count_ms
                            if best is None or tot < best[0]:
                                best = (tot, rep)
                        tot, rep = best
                        out = {"workload": a.workload, "k": k, "algo": algo, "scheme": scheme,
                               "criterion": crit, "group": gs, "all_k": a.all_k,
                               "count": str(rep.count), "orient_ms": round(rep.orient_ms, 3),
                               "count_ms": round(rep.count_ms, 3), "device_ms": rep.device_ms,
                               "cliques_per_s": rep.count / (tot / 1e3) if tot else None,
                               "d_max": rep.d_max, "degeneracy": rep.degeneracy,
                               "visits": rep.load.total,
                               "normalized_max": round(rep.load.normalized_max, 3),
                               "counters": rep.counters}
                        if a.all_k and rep.counts:
                            out["counts"] = {str(kk): str(v) for kk, v in rep.counts.items()}
                        if a.oracle_workers:
                            import oracle
                            og = oracle.from_edges(edges)
                            t0 = time.perf_counter()
                            o = oracle.run_count(og, k, algo, scheme, crit, a.oracle_workers,
                                                 all_k=a.all_k)
                            out["oracle_s"] = round(time.perf_counter() - t0, 3)
                            out["oracle_match"] = o.count == rep.count
                        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
