"""CPU: host logic above the C ABI -- config validation, the exact finalize
of raw device partials (32-bit limbs, pivot leaf histogram), shard balancing,
and the N>1 path (root-range shards + ONE element-wise u64 all-reduce) over
gloo with world_size 2.  The per-shard partials here come from the C oracle
(test infrastructure), standing in for kc_count on a GPU.
"""

import math
import os
import socket

import numpy as np
import pytest

from conftest import complete_edges, gnp_edges

from paper_2104_13209_b200 import cli, synth
from paper_2104_13209_b200.scheduler import RawCount, RunConfig, finalize, make_tasks, validate
from paper_2104_13209_b200.shard import balanced_ranges, per_rank_sms, spread_per_rank


# ---------------------------------------------------------------- validation
@pytest.mark.parametrize("bad", [
    dict(k=0), dict(k=3, algorithm="x"), dict(k=3, scheme="x"), dict(k=3, criterion="x"),
    dict(k=3, workers=0), dict(k=3, all_k=True), dict(k=3, group_size=3), dict(k=True),
])
def test_validate_rejects_like_reference(bad):
    """scheduler.py:188-200 raise ValueError for every invalid field."""
    with pytest.raises(ValueError):
        validate(RunConfig(**bad))


def test_auto_select_rules():
    """cli.py:50-62."""
    assert cli.auto_select(10, 10, 5, 4) == ("orient", "vertex", "degree")
    assert cli.auto_select(10, 10, 5, 6) == ("orient", "edge", "degree")
    assert cli.auto_select(10, 10, 5, 7) == ("pivot", "edge", "degeneracy")


def test_cli_parse_errors_exit_1(capsys):
    assert cli.main(["-k", "3"]) == 1
    assert cli.main(["-i", "/nonexistent/x.txt", "-k", "3"]) == 1


# ---------------------------------------------------------------- finalize
def _raw_from_count(c, visits=0, hist=None, nsm=4):
    limbs = np.array([(c >> (32 * i)) & 0xFFFFFFFF for i in range(4)], dtype=np.uint64)
    return RawCount(limbs, visits, 1, hist, np.zeros(nsm, dtype=np.uint64), 0.0)


def test_finalize_carries_limbs_beyond_64_bits():
    c = math.comb(75, 37)
    # unnormalized limbs (each a sum of many 32-bit partials) must carry
    lim = np.array([(c & 0xFFFFFFFF) + (5 << 32), ((c >> 32) & 0xFFFFFFFF) - 5,
                    (c >> 64) & 0xFFFFFFFF, c >> 96], dtype=np.uint64)
    raw = RawCount(lim, 0, 0, None, np.zeros(1, dtype=np.uint64), 0.0)
    count, _ = finalize(raw, RunConfig(k=37, algorithm="orient"), 75, 2775)
    assert count == c


def test_finalize_overflow_raises():
    c = (1 << 128) + 5
    lim = np.array([c & 0xFFFFFFFF, (c >> 32) & 0xFFFFFFFF, (c >> 64) & 0xFFFFFFFF,
                    c >> 96], dtype=np.uint64)
    with pytest.raises(OverflowError):
        finalize(RawCount(lim, 0, 0, None, np.zeros(1, dtype=np.uint64), 0.0),
                 RunConfig(k=4), 1, 1)


def test_finalize_pivot_histogram_expansion():
    """count = sum hist[len, np] * C(np, len - t) (engine_pivot.py:173-178);
    all-k: slot len-r += hist * C(np, r) (engine_pivot.py:228-233)."""
    L = 12
    rng = np.random.default_rng(3)
    hist = np.zeros((L, L), dtype=np.uint64)
    for _ in range(20):
        ln = int(rng.integers(0, L))
        npv = int(rng.integers(0, ln + 1))
        hist[ln, npv] += np.uint64(rng.integers(1, 1000))
    for k in range(3, 9):
        t = k - 1
        want = sum(int(hist[ln, npv]) * math.comb(npv, ln - t)
                   for ln in range(L) for npv in range(L) if 0 <= ln - t <= npv)
        raw = RawCount(np.zeros(4, dtype=np.uint64), 0, 0, hist, np.zeros(1, dtype=np.uint64), 0)
        got, _ = finalize(raw, RunConfig(k=k, algorithm="pivot"), 100, 100)
        assert got == want
    raw = RawCount(np.zeros(4, dtype=np.uint64), 0, 0, hist, np.zeros(1, dtype=np.uint64), 0)
    _, counts = finalize(raw, RunConfig(k=5, algorithm="pivot", all_k=True), 100, 200)
    assert counts[1] == 100 and counts[2] == 200
    for kk in range(3, L + 1):
        s = kk - 1
        want = sum(int(hist[ln, npv]) * math.comb(npv, ln - s)
                   for ln in range(L) for npv in range(L) if 0 <= ln - s <= npv)
        assert counts.get(kk, 0) == want


def test_raw_vector_roundtrip():
    hist = np.arange(16, dtype=np.uint64).reshape(4, 4)
    raw = RawCount(np.array([1, 2, 3, 4], dtype=np.uint64), 7, 9, hist,
                   np.array([5, 6], dtype=np.uint64), 1.5)
    back = raw.from_vector(raw.as_vector())
    assert back.limbs.tolist() == [1, 2, 3, 4] and back.visits == 7 and back.tasks_run == 9
    assert np.array_equal(back.hist, hist) and back.visits_per_sm.tolist() == [5, 6]


# ---------------------------------------------------------------- sharding
def test_balanced_ranges_cover_and_balance():
    rng = np.random.default_rng(0)
    costs = rng.pareto(1.5, 10000) * 100
    for world in (1, 2, 3, 4, 8):
        r = balanced_ranges(costs, world)
        assert len(r) == world and r[0][0] == 0 and r[-1][1] == costs.size
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        if world > 1:
            per = [costs[a:b].sum() for a, b in r]
            assert max(per) <= costs.sum() / world + costs.max() + 1e-6
    assert balanced_ranges(np.zeros(0), 4) == [(0, 0)] * 4


def test_make_tasks_matches_reference_definition(oracle):
    """scheduler.py:89-95: vertices with out-degree > 0; every oriented edge."""
    g = oracle.from_edges(gnp_edges(40, 0.2, 1))
    rank, _ = oracle.compute_rank(g, "degree")
    og = oracle.orient(g, rank)

    class _OG:  # the attributes make_tasks reads
        m_dir = og.m_dir

        @staticmethod
        def out_degrees():
            return np.diff(og.row_ptr)

    assert make_tasks(_OG, "vertex").size == oracle.num_tasks(og, "vertex")
    assert make_tasks(_OG, "edge").size == oracle.num_tasks(og, "edge")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_worker(rank, world, port, edges, cfgs, q):
    import torch.distributed as dist

    import oracle
    from paper_2104_13209_b200.shard import allreduce_raw

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = oracle.from_edges(edges)
        out = []
        for k, algo, scheme, crit in cfgs:
            rk, dg = oracle.compute_rank(g, crit)
            og = oracle.orient(g, rk, dg)
            n_tasks = oracle.num_tasks(og, scheme)
            costs = np.ones(n_tasks)
            lo, hi = balanced_ranges(costs, world)[rank]
            c, vis, _ = oracle.run_tasks(og, k, algo, scheme, False, 1, lo, hi)
            raw = _raw_from_count(c, sum(vis))
            # ranks report different SM usage (rank 1 touches a high %smid):
            # the all-reduced vector still has one length on every rank
            per = np.zeros(1024, dtype=np.uint64)
            per[rank] = sum(vis)
            if rank == 1:
                per[700] = 1
            raw.visits_per_sm = per
            raw = spread_per_rank(raw, rank, world)
            tot = allreduce_raw(raw)
            sms = per_rank_sms(tot.visits_per_sm, world, 4)
            assert len(sms) == 4 + 701 and sms[0] + sms[5] == sum(sms) - 1
            count, _ = finalize(tot, RunConfig(k=k, algorithm=algo, scheme=scheme,
                                               criterion=crit), g.n, g.m)
            out.append((count, tot.visits))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shards_sum_to_whole(oracle):
    """two ranks, disjoint root ranges, one u64 all-reduce;
    count and visits equal the single-process run on every rank."""
    import multiprocessing as mp

    edges = synth.rmat(10, 16, seed=1)
    cfgs = [(4, "orient", "vertex", "degree"), (5, "orient", "edge", "degeneracy"),
            (4, "pivot", "edge", "degree")]
    g = oracle.from_edges(edges)
    want = [(r.count, r.visits) for r in
            (oracle.run_count(g, k, a, s, c, workers=2) for k, a, s, c in cfgs)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, edges, cfgs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == want and res[1] == want


def test_complete_graph_closed_form_through_finalize():
    c = math.comb(70, 6)
    count, _ = finalize(_raw_from_count(c), RunConfig(k=6), 70, 2415)
    assert count == c
    assert complete_edges(4).shape == (6, 2)


def test_per_rank_sm_counters_keep_ranks_apart():
    """Advice r1: load statistics per (rank, SM), fixed width for the all-reduce."""
    a = RawCount(np.zeros(4, dtype=np.uint64), 3, 1, None, np.array([1, 2] + [0] * 1022,
                                                                   dtype=np.uint64), 0)
    b = RawCount(np.zeros(4, dtype=np.uint64), 4, 1, None, np.array([5, 0, 0, 7] + [0] * 1020,
                                                                   dtype=np.uint64), 0)
    va = spread_per_rank(a, 0, 2).as_vector()
    vb = spread_per_rank(b, 1, 2).as_vector()
    assert va.size == vb.size
    tot = spread_per_rank(a, 0, 2).from_vector(va + vb)
    assert tot.visits == 7
    assert per_rank_sms(tot.visits_per_sm, 2, 2) == [1, 2, 5, 0, 0, 7]
