"""The decomposition behind the device's exact heap order (csrc/kc_peel.cu),
restated in numpy and checked against the reference's sequential heap
(orientation.py:81-113, via the oracle) on CPU: core numbers -> shell-internal
components -> one heap run per component -> stable sort by (core, prefix-max
key).  If this ever disagrees with the heap, the CUDA path would too."""

import heapq

import numpy as np
import pytest

from conftest import gnp_edges

from paper_2104_13209_b200 import synth


def decomposed_rank(n, row_ptr, col):
    deg = np.diff(row_ptr)
    # core numbers (any peel order gives them)
    core = np.zeros(n, dtype=np.int64)
    d = deg.copy()
    alive = np.ones(n, bool)
    level = 0
    while alive.any():
        level = max(level, int(d[alive].min()))
        stack = list(np.flatnonzero(alive & (d <= level)))
        while stack:
            v = stack.pop()
            if not alive[v]:
                continue
            alive[v] = False
            core[v] = level
            for w in col[row_ptr[v]:row_ptr[v + 1]]:
                if alive[w]:
                    d[w] -= 1
                    if d[w] <= level:
                        stack.append(w)
    # degree inside the own core; shell-internal neighbours
    deg0 = np.array([int((core[col[row_ptr[v]:row_ptr[v + 1]]] >= core[v]).sum())
                     for v in range(n)], dtype=np.int64)
    inner = [[int(w) for w in col[row_ptr[v]:row_ptr[v + 1]] if core[w] == core[v]]
             for v in range(n)]
    comp = -np.ones(n, dtype=np.int64)
    comps = []
    for v in range(n):
        if comp[v] >= 0:
            continue
        comp[v] = len(comps)
        members, stack = [v], [v]
        while stack:
            x = stack.pop()
            for w in inner[x]:
                if comp[w] < 0:
                    comp[w] = len(comps)
                    members.append(w)
                    stack.append(w)
        comps.append(sorted(members))
    items = []
    for members in comps:
        k = core[members[0]]
        dd = {v: int(deg0[v]) for v in members}
        live = set(members)
        emax = (-1, -1)
        for p in range(len(members)):
            v = min(live, key=lambda x: (dd[x], x))
            assert dd[v] <= k
            emax = max(emax, (dd[v], v))
            items.append(((int(k), emax), v))
            live.discard(v)
            for w in inner[v]:
                if w in live:
                    dd[w] -= 1
    items.sort(key=lambda it: it[0])  # stable: (component, pop) order kept on ties
    rank = np.empty(n, dtype=np.int64)
    for i, (_, v) in enumerate(items):
        rank[v] = i
    return rank


def heap_rank(n, row_ptr, col):
    deg = np.diff(row_ptr).astype(np.int64)
    h = [(int(deg[v]), v) for v in range(n)]
    heapq.heapify(h)
    removed = np.zeros(n, bool)
    rank = np.empty(n, dtype=np.int64)
    pos = 0
    while h:
        dv, v = heapq.heappop(h)
        if removed[v] or dv != deg[v]:
            continue
        removed[v] = True
        rank[v] = pos
        pos += 1
        for w in col[row_ptr[v]:row_ptr[v + 1]]:
            if not removed[w]:
                deg[w] -= 1
                heapq.heappush(h, (int(deg[w]), int(w)))
    return rank


def graphs():
    for seed in range(12):
        yield gnp_edges(40 + 7 * seed, [0.05, 0.1, 0.2, 0.4][seed % 4], seed)
    yield synth.rmat(10, 16, seed=1)
    yield synth.planted_cliques(600, n_cliques=4, size_lo=8, size_hi=15, avg_deg=4.0, seed=2)


@pytest.mark.parametrize("gi", range(14))
def test_decomposition_equals_reference_heap(oracle, gi):
    edges = list(graphs())[gi]
    g = oracle.from_edges(edges)
    want, _ = oracle.compute_rank(g, "degeneracy")
    got = decomposed_rank(g.n, g.row_ptr, g.col)
    assert np.array_equal(heap_rank(g.n, g.row_ptr, g.col), want)
    assert np.array_equal(got, want)
