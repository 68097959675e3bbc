"""Full-graph oracle counts at the BASELINE.json sizes (test infrastructure).

    python tests/golden/make_scale_goldens.py rmat18:4:orient:vertex:degeneracy [...]

Each argument is ``workload:k:algorithm:scheme:criterion[:all]``.  The C
restatement of the reference (oracle/kc_oracle.c, pinned to the reference's
own fixtures by tests/test_oracle_golden.py) runs the WHOLE graph with every
host core -- no sampling -- on the seeded synthetic workload
(paper_2104_13209_b200.synth.workload), under the reference's own sequential
heap order for ``degeneracy`` (orientation.py:81-113).  The record keeps the
count, the visits (the reference's ``load.total``), the wall time, the thread
count and the host CPU model, and is merged into tests/golden/scale.json.
The GPU tests and bench.py compare against these records (the GPU box never
re-runs the long ones).
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import oracle  # noqa: E402
from paper_2104_13209_b200 import synth  # noqa: E402

OUT = os.path.join(HERE, "scale.json")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def load() -> list:
    if os.path.exists(OUT):
        with open(OUT) as f:
            return json.load(f)
    return []


def save(recs: list) -> None:
    with open(OUT, "w") as f:
        json.dump(recs, f, indent=1)
        f.write("\n")


def key(r) -> tuple:
    return (r["workload"], r["k"], r["algorithm"], r["scheme"], r["criterion"], r["all_k"])


def run(spec: str, workers: int) -> dict:
    parts = spec.split(":")
    wl, k, algo, scheme, crit = parts[0], int(parts[1]), parts[2], parts[3], parts[4]
    all_k = len(parts) > 5 and parts[5] == "all"
    edges = synth.workload(wl)
    t0 = time.perf_counter()
    g = oracle.from_edges(edges)
    build_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    rank, degen = oracle.compute_rank(g, crit)
    og = oracle.orient(g, rank, degen)
    orient_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    rep = oracle.run_count(g, k, algo, scheme, crit, workers=workers, all_k=all_k, rank=rank)
    count_s = time.perf_counter() - t0
    rec = {"workload": wl, "k": k, "algorithm": algo, "scheme": scheme, "criterion": crit,
           "all_k": all_k, "n": g.n, "m": g.m, "d_max": og.d_max, "degeneracy": degen,
           "edges_digest": synth.edges_digest(edges), "count": str(rep.count),
           "visits": rep.visits, "oracle_build_s": round(build_s, 2),
           "oracle_orient_s": round(orient_s, 2), "oracle_count_s": round(count_s, 2),
           "workers": workers, "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
           "recipe": "tests/golden/make_scale_goldens.py " + spec,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    if all_k and rep.counts:
        rec["counts"] = {str(kk): str(v) for kk, v in rep.counts.items()}
    return rec


def main(argv) -> int:
    workers = int(os.environ.get("ORACLE_WORKERS", os.cpu_count() or 1))
    oracle.build()
    for spec in argv:
        rec = run(spec, workers)
        recs = [r for r in load() if key(r) != key(rec)]
        recs.append(rec)
        recs.sort(key=lambda r: (r["workload"], r["k"], r["algorithm"], r["scheme"],
                                 r["criterion"]))
        save(recs)
        print(json.dumps(rec), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
