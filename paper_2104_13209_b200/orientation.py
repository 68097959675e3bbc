"""Total vertex orders and the oriented DAG, computed on the GPU.

Mirrors reference orientation.py: ``CRITERIA``, ``Ranking``,
``OrientedGraph``, ``compute_rank``, ``orient``.

* degree: rank by (undirected degree, id) -- identical to orientation.py:124-128.
* degeneracy: the reference's sequential heap order (orientation.py:81-113),
  rank for rank, computed in parallel (csrc/kc_peel.cu): core numbers by the
  bulk k-core peel (K3), then one heap run per connected component of each
  shell, merged by (core, running-max key).  Visits therefore equal the
  reference's for every engine.
* degeneracy_bulk (extension): the paper's bulk-synchronous peel order
  (PAPER.md:316-321), rank = (round, id) -- a valid degeneracy order
  (same d_max and counts) but different visits.
"""

from __future__ import annotations

import ctypes
import itertools
from dataclasses import dataclass

import numpy as np

from . import _lib

# "degeneracy" is the reference's sequential heap order (orientation.py:81-113)
# reproduced exactly on the GPU (identical ranks, hence identical visits);
# "degeneracy_exact" is its round-1 alias.  "degeneracy_bulk" (extension) is the
# paper's bulk-synchronous peel order: same degeneracy and counts, different
# visits, cheaper to compute.
CRITERIA = ("degree", "degeneracy", "degeneracy_exact", "degeneracy_bulk")
_token = itertools.count(1)


@dataclass
class Ranking:
    rank: np.ndarray
    criterion: str
    degeneracy: int | None = None
    # device-side bookkeeping (not part of the reference dataclass)
    rank_ms: float = 0.0
    rounds: int = 0
    _graph: object = None
    _token: int = 0
    _dag: object = None


class OrientedGraph:
    """DAG form of a Graph (orientation.py:20-45); arrays download lazily."""

    def __init__(self, graph, ranking: Ranking, info: _lib.KcDagInfo, token: int):
        self.graph = graph
        self.n = graph.n
        self.m_dir = int(info.m_dir)
        self.d_max = int(info.d_max)
        self.ranking = ranking
        self.orient_ms = float(info.orient_ms)
        self._token = token
        self._host = None

    def ensure_on_device(self):
        """Make this DAG the one resident on the graph's device handle."""
        g = self.graph
        if g._dag_token != self._token:
            info = _lib.KcDagInfo()
            r = self.ranking
            if isinstance(r, _LazyRanking) and r._rank_cache is None:
                # the permutation was never downloaded and another DAG replaced
                # this one: every criterion is deterministic, so recompute it
                # on the device (reading r.rank here would recurse)
                _lib.check(_lib.load().kc_orient(g.handle, _lib.CRIT[r.criterion], None,
                                                 ctypes.byref(info)))
            else:
                rank = np.ascontiguousarray(r.rank, dtype=np.int32)
                _lib.check(_lib.load().kc_orient(g.handle, _lib.CRIT["given"], _lib._ptr(rank),
                                                 ctypes.byref(info)))
            g._dag_token = self._token
        return g.handle

    def _download(self):
        if self._host is None:
            h = self.ensure_on_device()
            rp = np.zeros(self.n + 1, dtype=np.int64)
            col = np.empty(self.m_dir, dtype=np.int32)
            src = np.empty(self.m_dir, dtype=np.int32)
            _lib.check(_lib.load().kc_dag_download(h, None, _lib._ptr(rp), _lib._ptr(col),
                                                   _lib._ptr(src)))
            self._host = (rp, col, src)
        return self._host

    @property
    def row_ptr(self):
        return self._download()[0]

    @property
    def col(self):
        return self._download()[1]

    @property
    def coo_src(self):
        return self._download()[2]

    @property
    def coo_dst(self):
        return self.col

    def out_degrees(self):
        return np.diff(self.row_ptr)

    def out_neighbors(self, v):
        rp = self.row_ptr
        return self.col[rp[v]:rp[v + 1]]


def _orient_on_device(g, criterion: str, rank=None):
    info = _lib.KcDagInfo()
    arr = None if rank is None else np.ascontiguousarray(rank, dtype=np.int32)
    _lib.check(_lib.load().kc_orient(g.handle, _lib.CRIT[criterion], _lib._ptr(arr),
                                     ctypes.byref(info)))
    tok = next(_token)
    g._dag_token = tok
    return info, tok


def compute_rank(g, criterion: str) -> Ranking:
    """Total order under ``criterion`` (orientation.py:116-136), on the GPU.

    The DAG built alongside stays on the device so ``orient`` is free."""
    if criterion not in CRITERIA:
        raise ValueError(f"unknown orientation criterion: {criterion!r}")
    info, tok = _orient_on_device(g, criterion)
    rank = np.empty(g.n, dtype=np.int32)
    if g.n:
        _lib.check(_lib.load().kc_dag_download(g.handle, _lib._ptr(rank), None, None, None))
    degen = int(info.degeneracy) if criterion.startswith("degeneracy") else None
    r = Ranking(rank, criterion, degen, rank_ms=float(info.rank_ms), rounds=int(info.rounds))
    r._graph, r._token = g, tok
    r._dag = OrientedGraph(g, r, info, tok)
    return r


def orient(g, ranking: Ranking) -> OrientedGraph:
    """Keep each edge rank-ascending (orientation.py:139-153), on the GPU."""
    rank = np.asarray(ranking.rank)
    if len(rank) != g.n:
        raise ValueError("ranking size does not match the graph")
    if ranking._graph is g and ranking._dag is not None:
        return ranking._dag
    info, tok = _orient_on_device(g, "given", rank)
    return OrientedGraph(g, ranking, info, tok)


def rank_and_orient(g, criterion: str) -> OrientedGraph:
    """compute_rank + orient without downloading the rank (hot path)."""
    if criterion not in CRITERIA:
        raise ValueError(f"unknown orientation criterion: {criterion!r}")
    info, tok = _orient_on_device(g, criterion)
    degen = int(info.degeneracy) if criterion.startswith("degeneracy") else None
    r = _LazyRanking(g, criterion, degen, float(info.rank_ms), int(info.rounds))
    r._graph, r._token = g, tok
    og = OrientedGraph(g, r, info, tok)
    r._dag = og
    return og


class _LazyRanking(Ranking):
    """Ranking whose permutation is only downloaded if someone reads it."""

    def __init__(self, g, criterion, degeneracy, rank_ms, rounds):
        super().__init__(None, criterion, degeneracy, rank_ms=rank_ms, rounds=rounds)
        object.__setattr__(self, "_rank_cache", None)

    @property
    def rank(self):
        if self._rank_cache is None:
            g = self._graph
            if self._dag is not None:
                self._dag.ensure_on_device()
            arr = np.empty(g.n, dtype=np.int32)
            if g.n:
                _lib.check(_lib.load().kc_dag_download(g.handle, _lib._ptr(arr), None, None, None))
            self._rank_cache = arr
        return self._rank_cache

    @rank.setter
    def rank(self, value):
        object.__setattr__(self, "_rank_cache", value)
