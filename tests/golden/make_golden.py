"""Generate golden fixtures by running the REFERENCE package itself.

Run in the dev container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies ``/root/reference/pkg/src/kcliques`` to a temp dir (numba's
``cache=True`` would otherwise write into the read-only tree), imports it, and
writes small JSON fixtures next to this script.  The fixtures pin both the
C oracle (tests/test_oracle_golden.py, CPU) and the CUDA path
(tests/test_gpu_parity.py, GPU box) -- /root/reference itself is never read
at test time.
"""

from __future__ import annotations

import itertools
import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from paper_2104_13209_b200 import synth  # noqa: E402

REF_SRC = "/root/reference/pkg/src/kcliques"


def import_reference():
    tmp = tempfile.mkdtemp(prefix="kc_ref_")
    shutil.copytree(REF_SRC, os.path.join(tmp, "kcliques"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "numba_cache"))
    sys.path.insert(0, tmp)
    import kcliques  # noqa: PLC0415

    return kcliques


CONFIGS = list(itertools.product(("orient", "pivot"), ("vertex", "edge"), ("degree", "degeneracy")))


def gnp_edges(n, p, seed):
    # tests/conftest.py:65-73 of the reference
    rng = np.random.default_rng(seed)
    pairs = np.array(list(itertools.combinations(range(n), 2)), dtype=np.int64)
    kept = pairs[rng.random(len(pairs)) < p]
    if kept.shape[0] == 0:
        kept = pairs[:1]
    return kept


def complete_edges(n):
    return np.array(list(itertools.combinations(range(n), 2)), dtype=np.int64)


def petersen_edges():
    pairs = []
    for i in range(5):
        pairs += [(i, (i + 1) % 5), (i, i + 5), (5 + i, 5 + (i + 2) % 5)]
    return np.array(pairs, dtype=np.int64)


def graph_record(kc, name, edges, ks, with_arrays=True, allk=True, workers=2):
    g = kc.from_edges(edges)
    rec = {"name": name, "n": g.n, "m": g.m, "d_max_undirected": g.max_degree(),
           "edges_digest": synth.edges_digest(edges)}
    if with_arrays:
        rec["edges"] = np.asarray(edges).tolist()
        rec["row_ptr"] = g.row_ptr.tolist()
        rec["col"] = g.col.tolist()
        rec["coo_src"] = g.coo_src.tolist()
        rec["orig_ids"] = g.orig_ids.tolist()
    for crit in ("degree", "degeneracy"):
        r = kc.compute_rank(g, crit)
        og = kc.orient(g, r)
        rec[f"d_max_{crit}"] = og.d_max
        if crit == "degeneracy":
            rec["degeneracy"] = r.degeneracy
        if with_arrays:
            rec[f"rank_{crit}"] = r.rank.tolist()
    runs = []
    for k in ks:
        for algo, scheme, crit in CONFIGS:
            if isinstance(ks, dict) and (algo, scheme, crit) not in ks[k]:
                continue
            rep = kc.run_count(g, kc.RunConfig(k=k, algorithm=algo, scheme=scheme, criterion=crit,
                                               workers=workers))
            runs.append({"k": k, "algorithm": algo, "scheme": scheme, "criterion": crit,
                         "count": str(rep.count), "visits": rep.load.total, "d_max": rep.d_max})
    rec["runs"] = runs
    if allk:
        rec["all_k"] = []
        for scheme in ("vertex", "edge"):
            for crit in ("degree", "degeneracy"):
                rep = kc.run_count(g, kc.RunConfig(k=3, algorithm="pivot", scheme=scheme,
                                                   criterion=crit, workers=workers, all_k=True))
                rec["all_k"].append({"scheme": scheme, "criterion": crit,
                                     "counts": {str(k): str(v) for k, v in rep.counts.items()},
                                     "visits": rep.load.total})
    return rec


def small_suite(kc):
    cases = []
    for n in (3, 5, 8, 12):
        cases.append(graph_record(kc, f"K{n}", complete_edges(n), ks=range(3, n + 2)))
    cases.append(graph_record(kc, "petersen", petersen_edges(), ks=(3, 4, 5)))
    cases.append(graph_record(kc, "C7", np.array([(i, (i + 1) % 7) for i in range(7)]), ks=(3, 4)))
    cases.append(graph_record(kc, "K3,5", np.array([(i, 3 + j) for i in range(3) for j in range(5)]),
                              ks=(3, 4)))
    cases.append(graph_record(kc, "path6", np.array([(i, i + 1) for i in range(5)]), ks=(3, 4)))
    # reference tests/test_acceptance.py:99-126 style: seeded random small graphs
    rng = np.random.default_rng(2024)
    for i in range(24):
        n = int(rng.integers(4, 31))
        p = (0.1, 0.3, 0.5, 0.8)[i % 4]
        pairs = complete_edges(n)
        e = pairs[rng.random(len(pairs)) < p]
        if e.shape[0] == 0:
            e = pairs[:1]
        cases.append(graph_record(kc, f"rand{i}_n{n}_p{p}", e, ks=(3, 4, 5, 6)))
    for seed in (1, 2, 3):
        cases.append(graph_record(kc, f"gnp60_{seed}", gnp_edges(60, 0.3, seed), ks=(3, 4, 5, 6, 7)))
    # multi-word rows (reference tests/test_scheduler.py:119-122), 128-bit
    cases.append(graph_record(kc, "K70", complete_edges(70),
                              ks={4: CONFIGS, 6: [("pivot", "vertex", "degree")]},
                              with_arrays=False, allk=False))
    return cases


def extraction_suite(kc):
    out = []
    for name, edges, crit in (("gnp30_1", gnp_edges(30, 0.3, 1), "degree"),
                              ("gnp30_2", gnp_edges(30, 0.5, 2), "degeneracy"),
                              ("K70", complete_edges(70), "degree")):
        g = kc.from_edges(edges)
        og = kc.orient(g, kc.compute_rank(g, crit))
        tasks = []
        for scheme in ("vertex", "edge"):
            n_tasks = og.n if scheme == "vertex" else og.m_dir
            for task in range(0, n_tasks, max(1, n_tasks // 12)):
                for directed in (True, False):
                    S = (kc.extract_vertex_induced if scheme == "vertex" else kc.extract_edge_induced)(
                        og, task, directed=directed)
                    d = S.local_count
                    words = S.words[:d, : S.words_per_row]
                    tasks.append({"scheme": scheme, "task": task, "directed": directed, "d": d,
                                  "l2g": S.local_to_global[:d].tolist(),
                                  "words": [str(int(x)) for x in words.ravel()]})
                    if d and scheme == "vertex" and task % 3 == 0:
                        for t in range(0, min(d, 6) + 1):
                            if directed:
                                st = kc.NodeCounter()
                                c = kc.count_tcliques_orient(S, t, stats=st)
                                tasks[-1].setdefault("orient", []).append([t, str(c), st.visited])
                            else:
                                st = kc.NodeCounter()
                                c = kc.count_tcliques_pivot(S, t, stats=st)
                                tasks[-1].setdefault("pivot", []).append([t, str(c), st.visited])
                        if not directed:
                            st = kc.NodeCounter()
                            allt = kc.count_tcliques_pivot_all_t(S, stats=st)
                            tasks[-1]["pivot_all"] = [[str(x) for x in allt], st.visited]
        out.append({"name": name, "criterion": crit, "edges": edges.tolist(), "tasks": tasks})
    return out


def medium_suite(kc):
    """Synthetic workloads from paper_2104_13209_b200.synth at sizes the
    reference finishes in seconds (BASELINE.json configs, scaled)."""
    out = []
    plan = [
        ("er2000", synth.erdos_renyi(2000, 0.01, seed=0),
         [(4, "orient", "vertex", "degree"), (3, "orient", "vertex", "degree"),
          (4, "pivot", "edge", "degeneracy"), (5, "orient", "edge", "degeneracy")], True),
        ("rmat10", synth.rmat(10, 16, seed=1),
         [(k, a, s, c) for k in (3, 4, 5, 7) for a, s, c in CONFIGS], True),
        ("rmat12", synth.rmat(12, 16, seed=1),
         [(k, a, s, c) for k in (4, 7) for a, s, c in CONFIGS] +
         [(10, "pivot", "edge", "degeneracy"), (10, "pivot", "vertex", "degree"),
          (10, "orient", "vertex", "degeneracy")], True),
        ("rmat14", synth.rmat(14, 16, seed=1),
         [(4, "orient", "vertex", "degree"), (4, "orient", "vertex", "degeneracy"),
          (4, "orient", "edge", "degeneracy"), (7, "orient", "vertex", "degeneracy"),
          (7, "pivot", "edge", "degeneracy"), (7, "pivot", "vertex", "degeneracy"),
          (10, "pivot", "edge", "degeneracy"), (10, "pivot", "vertex", "degeneracy")], True),
        ("planted", synth.planted_cliques(), [(4, "orient", "vertex", "degree"),
                                              (10, "pivot", "edge", "degeneracy")], True),
        ("planted_small", synth.planted_cliques(n=5000, n_cliques=10, size_lo=30, size_hi=60, seed=5),
         [(4, "orient", "vertex", "degree"), (6, "orient", "edge", "degeneracy"),
          (12, "pivot", "edge", "degeneracy")], True),
    ]
    for name, edges, runs, allk in plan:
        g = kc.from_edges(edges)
        rec = {"name": name, "n": g.n, "m": g.m, "d_max_undirected": g.max_degree(),
               "edges_digest": synth.edges_digest(edges), "runs": []}
        for crit in ("degree", "degeneracy"):
            r = kc.compute_rank(g, crit)
            rec[f"d_max_{crit}"] = kc.orient(g, r).d_max
            if crit == "degeneracy":
                rec["degeneracy"] = r.degeneracy
        for k, algo, scheme, crit in runs:
            rep = kc.run_count(g, kc.RunConfig(k=k, algorithm=algo, scheme=scheme, criterion=crit,
                                               workers=os.cpu_count() or 1))
            rec["runs"].append({"k": k, "algorithm": algo, "scheme": scheme, "criterion": crit,
                                "count": str(rep.count), "visits": rep.load.total,
                                "d_max": rep.d_max})
            print(name, k, algo, scheme, crit, rep.count, rep.load.total, flush=True)
        if allk:
            rec["all_k"] = []
            for scheme in ("vertex", "edge"):
                rep = kc.run_count(g, kc.RunConfig(k=3, algorithm="pivot", scheme=scheme,
                                                   criterion="degeneracy",
                                                   workers=os.cpu_count() or 1, all_k=True))
                rec["all_k"].append({"scheme": scheme, "criterion": "degeneracy",
                                     "counts": {str(k): str(v) for k, v in rep.counts.items()},
                                     "visits": rep.load.total})
        out.append(rec)
    return out


def normalize_suite(kc):
    """Reference load_edge_list (graph.py:67-109) on raw edge-list texts with
    loops, repeats in both orders, comments and blank lines."""
    rng = np.random.default_rng(93)
    texts = ["", "# only a comment\n", "7 7\n", "3 1\n1 3\n2 2\n5 0\n2 2\n7 7\n",
             "1 2\n\n# c\n2 1 # tail\n1 2\n"]
    for trial in range(10):
        hi = (40, 300, 5000, 1 << 40)[trial % 4]
        m = int(rng.integers(1, 400))
        raw = rng.integers(0, hi, size=(m, 2))
        loops = rng.random(m) < 0.1
        raw[loops, 1] = raw[loops, 0]
        dup = rng.integers(0, m, size=m // 4)
        raw = np.concatenate([raw, raw[dup][:, ::-1]])
        texts.append("".join(f"{a} {b}\n" for a, b in raw.tolist()))
    out = []
    for i, text in enumerate(texts):
        el = kc.load_edge_list(text)
        out.append({"name": f"norm{i}", "text": text, "edges": el.edges.tolist(),
                    "n_self_loops": el.n_self_loops, "n_duplicates": el.n_duplicates,
                    "loop_ids": el.loop_ids.tolist()})
    return out


def main():
    kc = import_reference()
    with open(os.path.join(HERE, "normalize.json"), "w") as f:
        json.dump(normalize_suite(kc), f)
    if "--normalize-only" in sys.argv:
        return
    with open(os.path.join(HERE, "small.json"), "w") as f:
        json.dump(small_suite(kc), f)
    with open(os.path.join(HERE, "extract.json"), "w") as f:
        json.dump(extraction_suite(kc), f)
    with open(os.path.join(HERE, "medium.json"), "w") as f:
        json.dump(medium_suite(kc), f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
