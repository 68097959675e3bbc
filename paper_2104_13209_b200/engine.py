"""Bit-matrix sub-graphs and the single-matrix engines, backed by the GPU.

Mirrors the reference's ``bitgraph``, ``engine_orient`` and ``engine_pivot``
modules (BitGraph, extract_vertex_induced, extract_edge_induced, row_and,
popcount, NodeCounter, count_tcliques_orient, BinomialTable, binomial,
find_pivot, count_tcliques_pivot, count_tcliques_pivot_all_t, value128).

``extract_*`` run the K4 device builder of the counting kernel on one task
(kc_extract); ``count_tcliques_*`` and ``find_pivot`` run the K5/K6/K7 device
traversals on one host-provided matrix (kc_count_bitgraph / kc_find_pivot).
They exist for parity testing and exploration -- run_count never goes
through them.  Bit layout is the reference's: uint64 words, LSB-first.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib

W = 64
_LIMIT_128 = 1 << 128
_MASK_64 = (1 << 64) - 1


def value128(lo, hi) -> int:
    """Python integer from a (lo, hi) 64-bit pair (_bitops.py:129-131)."""
    return int(lo) | (int(hi) << 64)


class BitGraph:
    """Bit adjacency over up to ``capacity`` locals (bitgraph.py:15-56)."""

    def __init__(self, capacity):
        capacity = max(int(capacity), 0)
        self.capacity = capacity
        self.words = np.zeros((capacity, (capacity + W - 1) // W), dtype=np.uint64)
        self.local_to_global = np.empty(capacity, dtype=np.int64)
        self.local_count = 0
        self.words_per_row = 0
        self.directed = True

    def row_set(self, i):
        out = set()
        for w in range(self.words_per_row):
            x = int(self.words[i, w])
            while x:
                low = x & -x
                out.add(w * W + low.bit_length() - 1)
                x ^= low
        return out

    def matrix(self):
        d = self.local_count
        bits = np.unpackbits(self.words[:d, :self.words_per_row].view(np.uint8), axis=1,
                             bitorder="little")
        return bits[:, :d].astype(bool) if d else np.zeros((0, 0), dtype=bool)

    @property
    def nbytes(self):
        return self.words.nbytes + self.local_to_global.nbytes


def _extract(og, scheme, task, directed, out):
    h = og.ensure_on_device()
    cap = max(og.d_max, 1)
    S = out if out is not None else BitGraph(cap)
    wcap = max(S.words.shape[1], 1)
    words = np.zeros((max(S.capacity, 1), wcap), dtype=np.uint64)
    l2g = np.zeros(max(S.capacity, 1), dtype=np.int64)
    d = ctypes.c_int64()
    _lib.check(_lib.load().kc_extract(h, _lib.SCHEME[scheme], int(task), 1 if directed else 0,
                                      _lib._ptr(l2g), _lib._ptr(words), S.capacity, wcap,
                                      ctypes.byref(d)))
    d = int(d.value)
    S.words[:d] = words[:d, :S.words.shape[1]]
    S.local_to_global[:d] = l2g[:d]
    S.local_count = d
    S.words_per_row = (d + W - 1) // W
    S.directed = bool(directed)
    return S


def extract_vertex_induced(og, v, directed=True, out=None):
    """Induced sub-graph on the out-neighbours of v (bitgraph.py:125-137)."""
    rp = og.row_ptr
    if out is not None and int(rp[v + 1] - rp[v]) > out.capacity:
        raise ValueError("scratch BitGraph too small for this vertex")
    return _extract(og, "vertex", v, directed, out)


def extract_edge_induced(og, e, directed=True, out=None):
    """Induced sub-graph on the common out-neighbours of edge e (bitgraph.py:140-152)."""
    if out is not None:
        rp = og.row_ptr
        u, v = int(og.coo_src[e]), int(og.col[e])
        if min(int(rp[u + 1] - rp[u]), int(rp[v + 1] - rp[v])) > out.capacity:
            raise ValueError("scratch BitGraph too small for this edge")
    return _extract(og, "edge", e, directed, out)


def row_and(a, b):
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    if a.shape != b.shape:
        raise ValueError("bit rows differ in width")
    return a & b


def popcount(a):
    return int(np.bitwise_count(np.asarray(a, dtype=np.uint64)).sum())


class NodeCounter:
    """Visited-node tally shared across engine calls (engine_orient.py:22-28)."""

    __slots__ = ("visited",)

    def __init__(self):
        self.visited = 0


def binomial(n, r):
    if n < 0:
        raise ValueError("n must be non-negative")
    if r < 0 or r > n:
        return 0
    return math.comb(n, r)


class BinomialTable:
    """C(n, r) for n <= n_max as (lo, hi) words; >= 2^128 entries flagged
    (engine_pivot.py:41-79).  Built by Pascal's rule with saturation."""

    def __init__(self, n_max):
        n_max = int(n_max)
        if n_max < 0:
            raise ValueError("n_max must be non-negative")
        self.n_max = n_max
        size = n_max + 1
        self.lo = np.zeros((size, size), dtype=np.uint64)
        self.hi = np.zeros((size, size), dtype=np.uint64)
        self.too_big = np.zeros((size, size), dtype=np.uint8)
        row = [1]
        for n in range(size):
            if n:
                row = [1] + [row[i] + row[i + 1] for i in range(n - 1)] + [1]
            for r, c in enumerate(row):
                if c >= _LIMIT_128:
                    self.too_big[n, r] = 1
                else:
                    self.lo[n, r] = c & _MASK_64
                    self.hi[n, r] = c >> 64

    def value(self, n, r):
        if n < 0:
            raise ValueError("n must be non-negative")
        if n > self.n_max:
            raise OverflowError(f"binomial table holds n <= {self.n_max}, got {n}")
        if r < 0 or r > n:
            return 0
        if self.too_big[n, r]:
            raise OverflowError("binomial value exceeds the 128-bit accumulator")
        return value128(self.lo[n, r], self.hi[n, r])


def _rows(S):
    d = S.local_count
    wpr = max((d + W - 1) // W, 1)
    return np.ascontiguousarray(S.words[:d, :wpr], dtype=np.uint64), d


def _device():
    return _lib.current_device()


def count_tcliques_orient(S, t, stats=None):
    """t-cliques of the directed BitGraph S on the GPU (engine_orient.py:91-114)."""
    if t < 0:
        raise ValueError("t must be non-negative")
    if not S.directed:
        raise ValueError("the orientation engine needs a directed sub-graph")
    rows, d = _rows(S)
    out = np.zeros(4, dtype=np.uint64)
    _lib.check(_lib.load().kc_count_bitgraph(_device(), _lib._ptr(rows), d, int(t),
                                             _lib.ALGO["orient"], 0, _lib._ptr(out), None, None))
    if stats is not None:
        stats.visited += int(out[2])
    return value128(out[0], out[1])


def find_pivot(S, cand):
    """Pivot local id and cand minus its row (engine_pivot.py:104-114)."""
    cand = np.ascontiguousarray(cand, dtype=np.uint64)
    wpr = S.words_per_row
    if cand.shape[0] < wpr:
        raise ValueError("candidate row narrower than the sub-graph")
    if not any(int(w) for w in cand[:wpr]):
        raise ValueError("candidate set is empty")
    rows, d = _rows(S)
    pruned = np.zeros_like(cand)
    piv = ctypes.c_int64()
    c = np.ascontiguousarray(cand[:max(wpr, 1)])
    pr = np.zeros_like(c)
    _lib.check(_lib.load().kc_find_pivot(_device(), _lib._ptr(rows), d, _lib._ptr(c),
                                         ctypes.byref(piv), _lib._ptr(pr)))
    pruned[:pr.size] = pr
    return int(piv.value), pruned


def _table_ok(S, table):
    if table is not None and table.n_max < S.local_count:
        raise ValueError("binomial table smaller than the sub-graph")


def count_tcliques_pivot(S, t, stats=None, table=None):
    """t-cliques of the undirected BitGraph S by pivoting (engine_pivot.py:248-274)."""
    if t < 0:
        raise ValueError("t must be non-negative")
    if S.directed:
        raise ValueError("the pivot engine needs an undirected sub-graph")
    _table_ok(S, table)
    rows, d = _rows(S)
    out = np.zeros(4, dtype=np.uint64)
    _lib.check(_lib.load().kc_count_bitgraph(_device(), _lib._ptr(rows), d, int(t),
                                             _lib.ALGO["pivot"], 0, _lib._ptr(out), None, None))
    if stats is not None:
        stats.visited += int(out[2])
    return value128(out[0], out[1])


def count_tcliques_pivot_all_t(S, stats=None, table=None):
    """Counts for every t from one traversal (engine_pivot.py:277-308)."""
    if S.directed:
        raise ValueError("the pivot engine needs an undirected sub-graph")
    _table_ok(S, table)
    rows, d = _rows(S)
    out = np.zeros(4, dtype=np.uint64)
    lo = np.zeros(d + 2, dtype=np.uint64)
    hi = np.zeros(d + 2, dtype=np.uint64)
    _lib.check(_lib.load().kc_count_bitgraph(_device(), _lib._ptr(rows), d, 0,
                                             _lib.ALGO["pivot"], 1, _lib._ptr(out),
                                             _lib._ptr(lo), _lib._ptr(hi)))
    if stats is not None:
        stats.visited += int(out[2])
    return [value128(lo[i], hi[i]) for i in range(d + 1)]
