"""kcliques/_gpu.py -- the binding a maintainer of the reference package adds.

Self-contained (ctypes + numpy only; it does not import this repository's
Python package): it hands a reference ``Graph`` (graph.py:112-131: ``n, m,
row_ptr int64[n+1], col int32[2m], orig_ids``) and its ``Ranking``
(orientation.py:11-17) to libkc.so and returns what ``scheduler._run_tasks``
(scheduler.py:211-248) returns -- the exact count and the visited-node total
-- so ``run_count`` can call it in place of the numba worker pool:

    from kcliques import _gpu
    count, visits = _gpu.run_tasks_gpu(g, cfg, ranking)

C entry points used (include/kclique.h): kc_graph_from_csr (graph.py:112-131),
kc_orient with KC_CRIT_GIVEN (orient(g, ranking), orientation.py:139-153),
kc_count (scheduler.py:141-185 + the reduction of :211-293), kc_last_error.
Status codes map onto the reference's exceptions (scheduler.py:188-200,
:243-244).
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_P, _i64, _i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
KC_CRIT_GIVEN = 2


class _DagInfo(ctypes.Structure):
    _fields_ = [("m_dir", _i64), ("d_max", _i64), ("degeneracy", _i64), ("rounds", _i64),
                ("rank_ms", ctypes.c_double), ("orient_ms", ctypes.c_double)]


class _Args(ctypes.Structure):
    _fields_ = [("k", _i32), ("algorithm", _i32), ("scheme", _i32), ("all_k", _i32),
                ("group_size", _i32), ("block_size", _i32), ("task_lo", _i64), ("task_hi", _i64)]


class _Raw(ctypes.Structure):
    _fields_ = [("limbs", ctypes.c_uint64 * 4), ("visits", ctypes.c_uint64),
                ("tasks_run", ctypes.c_uint64), ("hist_dim", _i64), ("count_ms", ctypes.c_double),
                ("group_size", _i32), ("launches", _i32), ("word_ops", ctypes.c_uint64),
                ("extract_bytes", ctypes.c_uint64)]


_L = None


def _lib(path=None):
    global _L
    if _L is None:
        path = path or os.environ.get("KCLIQUES_LIBKC", "libkc.so")
        L = ctypes.CDLL(path)
        L.kc_graph_from_csr.argtypes = [ctypes.c_int, _i64, _i64, _P, _P, _P, ctypes.POINTER(_P)]
        L.kc_graph_free.argtypes = [_P]
        L.kc_graph_free.restype = None
        L.kc_orient.argtypes = [_P, ctypes.c_int, _P, ctypes.POINTER(_DagInfo)]
        L.kc_count.argtypes = [_P, ctypes.POINTER(_Args), ctypes.POINTER(_Raw), _P, _i64, _P,
                               _i32]
        L.kc_last_error.restype = ctypes.c_char_p
        _L = L
    return _L


def _check(status):
    if status == 0:
        return
    msg = (_lib().kc_last_error() or b"").decode(errors="replace")
    raise {1: ValueError, 3: OverflowError, 5: MemoryError}.get(status, RuntimeError)(msg)


def _ptr(a):
    return a.ctypes.data_as(_P)


def run_tasks_gpu(g, cfg, ranking, device=0):
    """scheduler._run_tasks on the GPU: (count, visits) for RunConfig cfg
    (k >= 3, not all_k) over the reference Graph g oriented by ``ranking``."""
    L = _lib()
    row_ptr = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    ids = np.ascontiguousarray(g.orig_ids, dtype=np.int64)
    rank = np.ascontiguousarray(ranking.rank, dtype=np.int32)
    h = _P()
    _check(L.kc_graph_from_csr(device, g.n, g.m, _ptr(row_ptr), _ptr(col), _ptr(ids),
                               ctypes.byref(h)))
    try:
        info = _DagInfo()
        _check(L.kc_orient(h, KC_CRIT_GIVEN, _ptr(rank), ctypes.byref(info)))
        pivot = cfg.algorithm == "pivot"
        a = _Args(cfg.k, 1 if pivot else 0, 1 if cfg.scheme == "edge" else 0, 0, 0, 0, 0, -1)
        raw = _Raw()
        # pivot: (length, pivots) leaf histogram, expanded exactly below
        dim = int(info.d_max) + 2
        hist = np.zeros(dim * dim if pivot else 1, dtype=np.uint64)
        _check(L.kc_count(h, ctypes.byref(a), ctypes.byref(raw), _ptr(hist) if pivot else None,
                          hist.size if pivot else 0, None, 0))
    finally:
        L.kc_graph_free(h)
    # exact count: 32-bit limb sums, plus (pivot) sum of hist[len, np] * C(np, len - t)
    count = sum(int(raw.limbs[i]) << (32 * i) for i in range(4))
    hd = int(raw.hist_dim)
    if hd:
        t = cfg.k - 1 if cfg.scheme == "vertex" else cfg.k - 2
        hh = hist[:hd * hd].reshape(hd, hd)
        for ln, npv in np.argwhere(hh).tolist():
            if 0 <= ln - t <= npv:
                c = math.comb(npv, ln - t)
                if c >= 1 << 128:
                    raise OverflowError("binomial value exceeds the 128-bit accumulator")
                count += int(hh[ln, npv]) * c
    if count >= 1 << 128:
        raise OverflowError("k-clique count exceeded the 128-bit accumulator")
    return count, int(raw.visits)
