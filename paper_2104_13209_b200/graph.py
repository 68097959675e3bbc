"""Edge-list input and the device-resident CSR+COO graph.

Mirrors the reference's ``graph`` module (graph.py): ``EdgeList``,
``ParseError``, ``load_edge_list``, ``Graph``, ``from_edges``, ``read_graph``,
plus ``normalize_edges`` (the edge-list normal form on the GPU).
``from_edges`` builds the CSR on the GPU (K1, csrc/kc_graph.cu); the host
arrays of ``Graph`` are copied back lazily on first access, so the counting
path never round-trips through host memory.
"""

from __future__ import annotations

import ctypes
import gzip
import io
import warnings

import numpy as np

from . import _lib


class ParseError(ValueError):
    """Malformed edge-list input; ``lineno`` is 1-based (graph.py:10-15)."""

    def __init__(self, lineno, message):
        super().__init__(f"line {lineno}: {message}")
        self.lineno = lineno


class EdgeList:
    """Normalized undirected edges: (m, 2) int64, u < v, sorted, unique."""

    def __init__(self, edges, n_self_loops=0, n_duplicates=0, loop_ids=None):
        self.edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        self.n_self_loops = int(n_self_loops)
        self.n_duplicates = int(n_duplicates)
        self.loop_ids = np.asarray([] if loop_ids is None else loop_ids, dtype=np.int64)

    def __len__(self):
        return int(self.edges.shape[0])

    def __iter__(self):
        return ((int(a), int(b)) for a, b in self.edges)

    def pair_set(self):
        return set(map(tuple, self.edges.tolist()))


def _strict_parse(data: bytes) -> np.ndarray:
    """Line-by-line parse that reports the first bad line."""
    out = []
    for no, raw in enumerate(data.splitlines(), start=1):
        body = raw.partition(b"#")[0].split()
        if not body:
            continue
        if len(body) != 2:
            raise ParseError(no, f"expected two integers, got {len(body)} tokens")
        try:
            a, b = int(body[0]), int(body[1])
        except ValueError:
            raise ParseError(no, "non-integer token") from None
        if a < 0 or b < 0:
            raise ParseError(no, "vertex ids must be non-negative")
        out.append((a, b))
    return np.array(out, dtype=np.int64).reshape(-1, 2)


def parse_edge_pairs(text) -> np.ndarray:
    """Parse ``u v`` lines (``#`` comments) into raw (m, 2) int64 pairs, in file
    order, loops and repeats kept (the parsing half of graph.py:67-91)."""
    data = text.read() if hasattr(text, "read") else text
    if isinstance(data, str):
        data = data.encode()
    arr = None
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            arr = np.loadtxt(io.BytesIO(data), dtype=np.int64, comments="#", ndmin=2)
        if arr.size and (arr.shape[1] != 2 or bool((arr < 0).any())):
            arr = None
    except ValueError:
        arr = None
    if arr is None:
        arr = _strict_parse(data)
    return np.ascontiguousarray(arr.reshape(-1, 2), dtype=np.int64)


def load_edge_list(text) -> EdgeList:
    """Parse ``u v`` lines (``#`` comments) into a normalized EdgeList.

    Self-loops and repeated pairs (either orientation) are dropped and counted.
    Host-side parse helper with the reference's exact semantics; the device
    path for large inputs is ``normalize_edges`` (used by ``read_graph``).
    """
    arr = parse_edge_pairs(text)
    if arr.size == 0:
        return EdgeList(np.empty((0, 2), dtype=np.int64))
    loops = arr[:, 0] == arr[:, 1]
    n_loops = int(loops.sum())
    loop_ids = np.unique(arr[loops, 0]) if n_loops else np.empty(0, dtype=np.int64)
    rest = np.sort(arr[~loops], axis=1)
    if rest.shape[0] == 0:
        return EdgeList(np.empty((0, 2), dtype=np.int64), n_loops, 0, loop_ids)
    uniq = np.unique(rest, axis=0)
    return EdgeList(uniq, n_loops, rest.shape[0] - uniq.shape[0], loop_ids)


def normalize_edges(raw, device: int | None = None, return_ms: bool = False):
    """Edge-list normal form on the GPU (K0, csrc/kc_ingest.cu).

    Same result as the normalization half of ``load_edge_list``
    (graph.py:93-109): self-loops dropped and tallied (ids kept as
    ``loop_ids``), pairs oriented u < v, sorted, repeats dropped and tallied.
    Negative ids raise ``ValueError``.
    """
    raw = np.ascontiguousarray(np.asarray(raw, dtype=np.int64).reshape(-1, 2))
    m_raw = raw.shape[0]
    pairs = np.empty((max(m_raw, 1), 2), dtype=np.int64)
    loop_ids = np.empty(max(m_raw, 1), dtype=np.int64)
    m_out, n_loop, n_self, n_dup = (ctypes.c_int64() for _ in range(4))
    ms = ctypes.c_double()
    dev = _lib.current_device() if device is None else device
    _lib.check(_lib.load().kc_normalize_edges(
        dev, _lib._ptr(raw), m_raw, _lib._ptr(pairs), ctypes.byref(m_out), _lib._ptr(loop_ids),
        ctypes.byref(n_loop), ctypes.byref(n_self), ctypes.byref(n_dup), ctypes.byref(ms)))
    el = EdgeList(pairs[:m_out.value].copy(), n_self.value, n_dup.value,
                  loop_ids[:n_loop.value].copy())
    return (el, float(ms.value)) if return_ms else el


class Graph:
    """Undirected simple graph resident on one GPU: CSR + aligned COO.

    Same public surface as the reference ``Graph`` (graph.py:112-159):
    ``n, m, row_ptr int64[n+1], col int32[2m], coo_src int32[2m], orig_ids,
    coo_dst, id_map, degrees(), max_degree(), neighbors(), has_edge(),
    edge_pairs()``.  Host arrays are downloaded on first use.
    """

    def __init__(self, handle, device: int):
        self._h = handle
        self.device = device
        L = _lib.load()
        n, m, dmax = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        ms = ctypes.c_double()
        _lib.check(L.kc_graph_info(handle, ctypes.byref(n), ctypes.byref(m), ctypes.byref(dmax),
                                   ctypes.byref(ms)))
        self.n = int(n.value)
        self.m = int(m.value)
        self._d_max_und = int(dmax.value)
        self.build_ms = float(ms.value)
        self._host = None
        self._id_map = None
        self._dag_token = None  # identity of the DAG currently on the device

    # -- lifetime -----------------------------------------------------------
    @property
    def handle(self):
        if self._h is None:
            raise ValueError("graph has been freed")
        return self._h

    def free(self):
        if self._h is not None:
            _lib.load().kc_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    # -- host mirrors -------------------------------------------------------
    def _download(self):
        if self._host is None:
            rp = np.zeros(self.n + 1, dtype=np.int64)
            col = np.empty(2 * self.m, dtype=np.int32)
            src = np.empty(2 * self.m, dtype=np.int32)
            ids = np.empty(self.n, dtype=np.int64)
            _lib.check(_lib.load().kc_graph_download(self.handle, _lib._ptr(rp), _lib._ptr(col),
                                                     _lib._ptr(src), _lib._ptr(ids)))
            self._host = (rp, col, src, ids)
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
    def orig_ids(self):
        return self._download()[3]

    @property
    def coo_dst(self):
        return self.col

    @property
    def id_map(self):
        if self._id_map is None:
            self._id_map = {int(o): i for i, o in enumerate(self.orig_ids.tolist())}
        return self._id_map

    def degrees(self):
        return np.diff(self.row_ptr)

    def max_degree(self):
        return self._d_max_und

    def neighbors(self, v):
        rp = self.row_ptr
        return self.col[rp[v]:rp[v + 1]]

    def has_edge(self, u, v):
        seg = self.neighbors(u)
        i = int(np.searchsorted(seg, v))
        return i < seg.size and int(seg[i]) == int(v)

    def edge_pairs(self):
        keep = self.coo_src < self.col
        return np.stack([self.coo_src[keep], self.col[keep]], axis=1).astype(np.int64)


def from_edges(edges, device: int | None = None) -> Graph:
    """Build the CSR+COO graph on the GPU (graph.py:162-200 semantics).

    Ids are compacted to 0..n-1 in ascending original-id order; both arc
    directions are stored and each row is sorted ascending.
    """
    if isinstance(edges, EdgeList):
        pairs, extra = edges.edges, edges.loop_ids
    else:
        src = edges if isinstance(edges, np.ndarray) else list(edges)
        pairs = np.asarray(src, dtype=np.int64).reshape(-1, 2)
        extra = np.empty(0, dtype=np.int64)
    pairs = np.ascontiguousarray(pairs, dtype=np.int64)
    extra = np.ascontiguousarray(extra, dtype=np.int64)
    dev = _lib.current_device() if device is None else device
    h = ctypes.c_void_p()
    _lib.check(_lib.load().kc_graph_from_edges(dev, _lib._ptr(pairs), pairs.shape[0],
                                               _lib._ptr(extra), extra.size, ctypes.byref(h)))
    return Graph(h, dev)


def from_raw_edges(raw, device: int | None = None) -> Graph:
    """``from_edges(load_edge_list(...))`` for already-parsed raw pairs, all on
    the GPU: K0 normal form kept on the device, then K1.  The graph carries
    ``n_self_loops``, ``n_duplicates`` and ``normalize_ms``."""
    raw = np.ascontiguousarray(np.asarray(raw, dtype=np.int64).reshape(-1, 2))
    dev = _lib.current_device() if device is None else device
    h = ctypes.c_void_p()
    n_self, n_dup, ms = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    _lib.check(_lib.load().kc_graph_from_raw_edges(dev, _lib._ptr(raw), raw.shape[0],
                                                   ctypes.byref(n_self), ctypes.byref(n_dup),
                                                   ctypes.byref(ms), ctypes.byref(h)))
    g = Graph(h, dev)
    g.n_self_loops, g.n_duplicates, g.normalize_ms = n_self.value, n_dup.value, ms.value
    return g


def read_graph(path, device: int | None = None) -> Graph:
    """SNAP-style edge list (plain or gzip) -> device Graph (graph.py:203-209)."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:2] == b"\x1f\x8b":
        raw = gzip.decompress(raw)
    return from_raw_edges(parse_edge_pairs(raw), device=device)
