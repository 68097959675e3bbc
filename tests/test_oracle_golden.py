"""CPU: pin the C oracle (oracle/kc_oracle.c) to the reference.

The fixtures in tests/golden/ were produced by running the reference package
itself (tests/golden/make_golden.py); the known answers below are the
reference tests' own (cited per test).  Nothing here needs a GPU.
"""

import itertools
import math
import os

import numpy as np
import pytest

from conftest import complete_edges, cycle_edges, gnp_edges, load_golden, petersen_edges

CONFIGS = list(itertools.product(("orient", "pivot"), ("vertex", "edge"), ("degree", "degeneracy")))
WORKERS = min(8, os.cpu_count() or 1)


def _edges(rec):
    return np.array(rec["edges"], dtype=np.int64).reshape(-1, 2)


SMALL = load_golden("small.json")
SMALL_WITH_ARRAYS = [r for r in SMALL if "edges" in r]


@pytest.mark.parametrize("rec", SMALL_WITH_ARRAYS, ids=lambda r: r["name"])
def test_csr_rank_orient_match_reference(oracle, rec):
    """graph.py:162-200 and orientation.py:116-153 array for array."""
    g = oracle.from_edges(_edges(rec))
    assert (g.n, g.m) == (rec["n"], rec["m"])
    assert g.row_ptr.tolist() == rec["row_ptr"]
    assert g.col.tolist() == rec["col"]
    assert g.coo_src.tolist() == rec["coo_src"]
    assert g.orig_ids.tolist() == rec["orig_ids"]
    for crit in ("degree", "degeneracy"):
        rank, degen = oracle.compute_rank(g, crit)
        assert rank.tolist() == rec[f"rank_{crit}"], crit
        og = oracle.orient(g, rank, degen)
        assert og.d_max == rec[f"d_max_{crit}"]
        if crit == "degeneracy":
            assert degen == rec["degeneracy"]


@pytest.mark.parametrize("rec", SMALL_WITH_ARRAYS, ids=lambda r: r["name"])
def test_counts_and_visits_match_reference(oracle, rec):
    """scheduler.py:296-338 count and load.total for every run in the fixture."""
    g = oracle.from_edges(_edges(rec))
    for run in rec["runs"]:
        rep = oracle.run_count(g, run["k"], run["algorithm"], run["scheme"], run["criterion"],
                               workers=2)
        assert str(rep.count) == run["count"], run
        assert rep.visits == run["visits"], run
    for run in rec.get("all_k", []):
        rep = oracle.run_count(g, 3, "pivot", run["scheme"], run["criterion"], workers=2,
                               all_k=True)
        assert {str(k): str(v) for k, v in rep.counts.items()} == run["counts"]
        assert rep.visits == run["visits"]


def test_k70_multiword_rows_match_reference(oracle):
    rec = next(r for r in SMALL if r["name"] == "K70")
    g = oracle.from_edges(complete_edges(70))
    for run in rec["runs"]:
        rep = oracle.run_count(g, run["k"], run["algorithm"], run["scheme"], run["criterion"],
                               workers=WORKERS)
        assert str(rep.count) == run["count"]
        assert rep.visits == run["visits"]


@pytest.mark.parametrize("rec", load_golden("extract.json"), ids=lambda r: r["name"])
def test_extraction_and_engines_match_reference(oracle, rec):
    """bitgraph.py:125-152 bitmaps and engine_orient/engine_pivot single-matrix counts."""
    g = oracle.from_edges(_edges(rec))
    rank, degen = oracle.compute_rank(g, rec["criterion"])
    og = oracle.orient(g, rank, degen)
    for task in rec["tasks"]:
        l2g, words = oracle.extract(og, task["scheme"], task["task"], task["directed"])
        assert len(l2g) == task["d"]
        assert l2g.tolist() == task["l2g"]
        assert [str(int(x)) for x in words.ravel()] == task["words"]
        d = task["d"]
        for t, cnt, vis in task.get("orient", []):
            c, v, _ = oracle.count_bitgraph(words, d, t, "orient")
            assert (str(c), v) == (cnt, vis)
        for t, cnt, vis in task.get("pivot", []):
            c, v, _ = oracle.count_bitgraph(words, d, t, "pivot")
            assert (str(c), v) == (cnt, vis)
        if "pivot_all" in task:
            allt, vis = task["pivot_all"]
            c, v, _ = oracle.count_bitgraph(words, d, 0, "pivot_all")
            assert [str(x) for x in c[:len(allt)]] == allt
            assert v == vis


MEDIUM = load_golden("medium.json")


@pytest.mark.parametrize("name", ["er2000", "rmat10", "rmat12", "planted_small"])
def test_medium_synthetic_match_reference(oracle, name):
    from paper_2104_13209_b200 import synth

    rec = next(r for r in MEDIUM if r["name"] == name)
    edges = {"er2000": lambda: synth.erdos_renyi(2000, 0.01, seed=0),
             "rmat10": lambda: synth.rmat(10, 16, seed=1),
             "rmat12": lambda: synth.rmat(12, 16, seed=1),
             "planted_small": lambda: synth.planted_cliques(n=5000, n_cliques=10, size_lo=30,
                                                            size_hi=60, seed=5)}[name]()
    assert synth.edges_digest(edges) == rec["edges_digest"]
    g = oracle.from_edges(edges)
    assert (g.n, g.m) == (rec["n"], rec["m"])
    for run in rec["runs"]:
        rep = oracle.run_count(g, run["k"], run["algorithm"], run["scheme"], run["criterion"],
                               workers=WORKERS)
        assert str(rep.count) == run["count"], run
        assert rep.visits == run["visits"], run
        assert rep.d_max == run["d_max"]
    for run in rec.get("all_k", []):
        rep = oracle.run_count(g, 3, "pivot", run["scheme"], run["criterion"], workers=WORKERS,
                               all_k=True)
        assert {str(k): str(v) for k, v in rep.counts.items()} == run["counts"]


# ---- the reference tests' own known answers --------------------------------
def test_closed_forms_complete_graphs(oracle):
    """tests/test_acceptance.py:147-159, tests/test_engine_orient.py:77-82."""
    for n in (5, 9, 13):
        g = oracle.from_edges(complete_edges(n))
        for k in range(1, n + 2):
            for algo, scheme, crit in CONFIGS:
                rep = oracle.run_count(g, k, algo, scheme, crit)
                assert rep.count == math.comb(n, k), (n, k, algo, scheme, crit)


def test_zero_clique_graphs(oracle):
    """tests/test_acceptance.py:160-164: Petersen, C7, K_{3,5} have no triangles."""
    bip = np.array([(i, 3 + j) for i in range(3) for j in range(5)], dtype=np.int64)
    for e in (petersen_edges(), cycle_edges(7), bip):
        g = oracle.from_edges(e)
        for algo, scheme, crit in CONFIGS:
            assert oracle.run_count(g, 3, algo, scheme, crit).count == 0


def test_beyond_64_bits_and_overflow(oracle):
    """tests/test_scheduler.py:106-116: K75 k=37 > 2^64; K140 k=70 overflows 2^128."""
    g = oracle.from_edges(complete_edges(75))
    rep = oracle.run_count(g, 37, "pivot", "vertex", "degree")
    assert rep.count == math.comb(75, 37) and rep.count > 2**64
    g = oracle.from_edges(complete_edges(140))
    with pytest.raises(OverflowError):
        oracle.run_count(g, 70, "pivot", "vertex", "degree")


def test_binomial_128_bit_boundary(oracle):
    """tests/test_engine_pivot.py:61-67: C(131,65) fits, C(132,66) is flagged."""
    lo, hi, big = oracle.binomial_table(132)
    assert not big[131, 65]
    assert int(lo[131, 65]) | (int(hi[131, 65]) << 64) == math.comb(131, 65)
    assert big[132, 66]


def test_random_sweep_against_brute_force(oracle):
    """tests/test_acceptance.py:99-126 (reduced): every config equals a brute-force count."""
    rng = np.random.default_rng(2024)
    for i in range(30):
        n = int(rng.integers(4, 16))
        p = (0.1, 0.3, 0.5, 0.8)[i % 4]
        e = gnp_edges(n, p, int(rng.integers(1 << 30)))
        adj = np.zeros((n, n), dtype=bool)
        adj[e[:, 0], e[:, 1]] = adj[e[:, 1], e[:, 0]] = True
        g = oracle.from_edges(e)
        ids = g.orig_ids.tolist()
        for k in (3, 4, 5):
            brute = sum(1 for c in itertools.combinations(ids, k)
                        if all(adj[a, b] for a, b in itertools.combinations(c, 2)))
            for algo, scheme, crit in CONFIGS:
                assert oracle.run_count(g, k, algo, scheme, crit).count == brute


def test_visits_independent_of_worker_count(oracle):
    """tests/test_scheduler.py:55-66: count and visits identical for 1/2/8 workers."""
    g = oracle.from_edges(gnp_edges(60, 0.3, 7))
    for algo, scheme, crit in CONFIGS:
        base = oracle.run_count(g, 5, algo, scheme, crit, workers=1)
        for w in (2, 8):
            r = oracle.run_count(g, 5, algo, scheme, crit, workers=w)
            assert (r.count, r.visits) == (base.count, base.visits)
