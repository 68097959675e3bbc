"""Exact heap order on the device vs the oracle's heap (rank array equality)
and its cost next to the bulk peel.  python scripts/exact_order_check.py rmat16 rmat18 ..."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2104_13209_b200 as kc  # noqa: E402
from paper_2104_13209_b200 import synth  # noqa: E402

for wl in sys.argv[1:]:
    e = synth.workload(wl)
    g = kc.from_edges(e)
    out = {"workload": wl, "n": g.n}
    for crit in ("degeneracy_exact", "degeneracy"):
        ms = []
        for _ in range(3):
            r = kc.compute_rank(g, crit)
            ms.append(r.rank_ms)
        out[crit + "_rank_ms"] = sorted(ms)
    r = kc.compute_rank(g, "degeneracy_exact")
    if g.n <= 3_000_000 and os.environ.get("CHECK", "1") == "1":
        o = oracle.from_edges(e)
        t0 = time.perf_counter()
        want, deg = oracle.compute_rank(o, "degeneracy")
        out["oracle_rank_s"] = round(time.perf_counter() - t0, 2)
        out["rank_equal"] = bool(np.array_equal(r.rank, want))
        out["degeneracy"] = (r.degeneracy, deg)
    print(json.dumps(out), flush=True)
