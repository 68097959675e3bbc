"""Run configuration, the GPU counting entry point and its report.

Mirrors reference scheduler.py: ``RunConfig``, ``LoadStats``, ``load_stats``,
``CountReport``, ``make_tasks``, ``run_count``.  The reference's worker pool
(scheduler.py:141-293: per-thread scratch, atomic task cursor, Python-int
reduction) is replaced by one ``kc_count`` call: persistent CTAs on the GPU
pull tasks from a device atomic queue and return reducible partial sums
(32-bit count limbs, a (path length, pivot count) leaf histogram for the
pivot engine, per-SM visit counts).  ``finalize`` turns those sums into the
exact integer count on the host; a multi-GPU run all-reduces the same
buffers first (see shard.py).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .orientation import CRITERIA, rank_and_orient

ALGORITHMS = ("orient", "pivot")
SM_SLOTS = 1024  # width of the per-SM visit counters (kc_count's kSmidSlots)
SCHEMES = ("vertex", "edge")
_LIMIT_128 = 1 << 128


@dataclass
class RunConfig:
    k: int
    algorithm: str = "orient"
    scheme: str = "vertex"
    criterion: str = "degree"
    workers: int = 1          # accepted for API parity; parallelism is the GPU's
    all_k: bool = False
    group_size: int = 0       # orient sub-warp group size: 0 auto, 1..32


@dataclass
class LoadStats:
    """Visited-node summary per worker; here a worker is one SM."""

    per_worker: list
    min: int
    max: int
    mean: float
    normalized_max: float
    total: int


def load_stats(counters) -> LoadStats:
    c = [int(x) for x in counters]
    total = sum(c)
    mean = total / len(c) if c else 0.0
    return LoadStats(per_worker=c, min=min(c, default=0), max=max(c, default=0), mean=mean,
                     normalized_max=(max(c) / mean) if mean > 0 else 1.0, total=total)


@dataclass
class CountReport:
    n: int
    m: int
    d_max_undirected: int
    d_max: int
    config: RunConfig
    count: int
    orient_ms: float
    count_ms: float
    load: LoadStats
    scratch_bytes: int
    counts: dict | None = None
    degeneracy: int | None = None
    load_ms: float = 0.0
    device_ms: dict | None = None  # CUDA-event times of each device phase
    counters: dict | None = None   # this rank's kernel counters (roofline inputs)

    @property
    def total_ms(self):
        return self.orient_ms + self.count_ms


def make_tasks(og, scheme):
    """Vertex tasks (out-degree > 0) or every oriented edge (scheduler.py:89-95)."""
    if scheme == "vertex":
        return np.flatnonzero(og.out_degrees() > 0).astype(np.int64)
    if scheme == "edge":
        return np.arange(og.m_dir, dtype=np.int64)
    raise ValueError(f"unknown scheme: {scheme!r}")


def validate(cfg: RunConfig) -> None:
    """scheduler.py:188-200, plus the GPU group-size knob."""
    if not isinstance(cfg.k, int) or isinstance(cfg.k, bool) or cfg.k < 1:
        raise ValueError("k must be an integer >= 1")
    if cfg.algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm: {cfg.algorithm!r}")
    if cfg.scheme not in SCHEMES:
        raise ValueError(f"unknown scheme: {cfg.scheme!r}")
    if cfg.criterion not in CRITERIA:
        raise ValueError(f"unknown orientation criterion: {cfg.criterion!r}")
    if cfg.workers < 1:
        raise ValueError("workers must be >= 1")
    if cfg.all_k and cfg.algorithm != "pivot":
        raise ValueError("all-k reporting requires the pivot algorithm")
    if cfg.group_size not in (0, 1, 2, 4, 8, 16, 32):
        raise ValueError("group_size must be 0 (auto) or a power of two <= 32")


# --------------------------------------------------------------------------
# raw device partials -> exact counts
# --------------------------------------------------------------------------
@dataclass
class RawCount:
    """Element-wise summable partials of one or more kc_count calls."""

    limbs: np.ndarray        # uint64[4]
    visits: int
    tasks_run: int
    hist: np.ndarray | None  # uint64[L, L] (pivot) or None
    visits_per_sm: np.ndarray
    count_ms: float
    word_ops: int = 0        # roofline counters of the counting kernel
    extract_bytes: int = 0
    group_size: int = 0      # sub-warp group size the orientation warp tier ran with
    launches: int = 0        # counting-kernel launches

    def as_vector(self) -> np.ndarray:
        """Flatten for an element-wise u64 all-reduce."""
        parts = [self.limbs, np.array([self.visits, self.tasks_run], dtype=np.uint64),
                 self.visits_per_sm]
        if self.hist is not None:
            parts.append(self.hist.ravel())
        return np.concatenate(parts).astype(np.uint64)

    def from_vector(self, vec: np.ndarray) -> "RawCount":
        vec = np.asarray(vec, dtype=np.uint64)
        nsm = self.visits_per_sm.size
        hist = None
        if self.hist is not None:
            hist = vec[6 + nsm:].reshape(self.hist.shape).copy()
        return RawCount(vec[:4].copy(), int(vec[4]), int(vec[5]), hist, vec[6:6 + nsm].copy(),
                        self.count_ms, self.word_ops, self.extract_bytes, self.group_size,
                        self.launches)


def device_count_raw(og, cfg: RunConfig, task_lo: int = 0, task_hi: int = -1) -> RawCount:
    """One kc_count call over [task_lo, task_hi) of make_tasks order."""
    L = _lib.load()
    h = og.ensure_on_device()
    k = max(cfg.k, 3) if cfg.all_k else cfg.k  # all-k ignores k on the device
    a = _lib.KcCountArgs(k, _lib.ALGO[cfg.algorithm], _lib.SCHEME[cfg.scheme],
                         1 if cfg.all_k else 0, int(cfg.group_size), 0, int(task_lo),
                         int(task_hi))
    raw = _lib.KcCountRaw()
    pivot = cfg.algorithm == "pivot"
    # pivot: the (length, pivots) leaf histogram, expanded on the host
    dim = og.d_max + 2
    hist = np.zeros(dim * dim if pivot else 1, dtype=np.uint64)
    # fixed width (every rank's vector has the same length for the all-reduce);
    # trimmed to the SMs actually used only when reported (used_sms)
    per_sm = np.zeros(SM_SLOTS, dtype=np.uint64)
    _lib.check(L.kc_count(h, ctypes.byref(a), ctypes.byref(raw),
                          _lib._ptr(hist) if pivot else None, hist.size if pivot else 0,
                          _lib._ptr(per_sm), per_sm.size))
    hd = int(raw.hist_dim)
    return RawCount(np.array(raw.limbs[:], dtype=np.uint64), int(raw.visits), int(raw.tasks_run),
                    hist[:hd * hd].reshape(hd, hd) if hd else None, per_sm,
                    float(raw.count_ms), int(raw.word_ops), int(raw.extract_bytes),
                    int(raw.group_size), int(raw.launches))


def used_sms(per_sm, nsm: int) -> list:
    """Per-SM visit counters trimmed to the device's SMs (%smid can exceed the
    SM count, so a counter above nsm that is non-zero extends the list)."""
    per_sm = np.asarray(per_sm)
    used = max(nsm, int(np.flatnonzero(per_sm).max()) + 1 if per_sm.any() else 0)
    return [int(x) for x in per_sm[:used]]


def _binom_checked(n: int, r: int) -> int:
    c = math.comb(n, r)
    if c >= _LIMIT_128:
        raise OverflowError("binomial value exceeds the 128-bit accumulator")
    return c


def finalize(raw: RawCount, cfg: RunConfig, n: int, m: int):
    """Exact count (and all-k table) from summed partials.

    count = limbs[0] + limbs[1]*2^32 + limbs[2]*2^64 + limbs[3]*2^96
          + sum_{len,np} hist[len, np] * C(np, len - t)           (pivot, per k)
    all-k: slot s += hist[len, np] * C(np, r) at s = len - r.
    Raises OverflowError when a touched binomial or the total reaches 2^128
    (the reference's 128-bit accumulator contract, scheduler.py:243-244).
    """
    lim = [int(x) for x in raw.limbs]
    direct = lim[0] + (lim[1] << 32) + (lim[2] << 64) + (lim[3] << 96)
    t = cfg.k - 1 if cfg.scheme == "vertex" else cfg.k - 2
    counts = None
    if raw.hist is None:
        count = direct
    else:
        nz = np.argwhere(raw.hist)
        if cfg.all_k:
            slots = {}
            for ln, npv in nz.tolist():
                c = int(raw.hist[ln, npv])
                for r in range(npv + 1):
                    slots[ln - r] = slots.get(ln - r, 0) + c * _binom_checked(npv, r)
            offset = 1 if cfg.scheme == "vertex" else 2
            counts = {1: n, 2: m}
            for s, val in sorted(slots.items()):
                if val >= _LIMIT_128:
                    raise OverflowError("k-clique count exceeded the 128-bit accumulator")
                kk = s + offset
                if kk >= 3 and val:
                    counts[kk] = val
            count = counts.get(cfg.k, 0)
        else:
            count = direct
            for ln, npv in nz.tolist():
                r = ln - t
                if 0 <= r <= npv:
                    count += int(raw.hist[ln, npv]) * _binom_checked(npv, r)
    if count >= _LIMIT_128:
        raise OverflowError("k-clique count exceeded the 128-bit accumulator")
    return count, counts


def scratch_bytes(og, cfg: RunConfig) -> int:
    """Per-task device scratch (bit matrix + locals + stacks) of one CTA."""
    cap = max(og.d_max, 1)
    W = (cap + 31) // 32
    rows = cap * (W | 1) * 4 + cap * 4
    t = cfg.k - 1 if cfg.scheme == "vertex" else cfg.k - 2
    if cfg.algorithm == "pivot":
        stack = 8 * (cap + 2) * (3 * W + 3) * 4
    else:
        stack = 256 * max(t - 2, 0) * 2 * 4
    return rows + stack


def run_count(g, cfg: RunConfig) -> CountReport:
    """Count k-cliques of ``g`` on its GPU (scheduler.py:296-338 contract)."""
    validate(cfg)
    t0 = time.perf_counter()
    og = rank_and_orient(g, cfg.criterion)
    orient_ms = (time.perf_counter() - t0) * 1000.0
    ranking = og.ranking
    t1 = time.perf_counter()
    counts = None
    dev = {"rank": ranking.rank_ms, "orient": og.orient_ms, "count": 0.0}
    nsm = _lib.num_sms(g.device)
    counters = None
    if cfg.k <= 2 and not cfg.all_k:
        count = g.n if cfg.k == 1 else g.m
        visits = [0] * nsm
        sbytes = 0
    else:
        raw = device_count_raw(og, cfg)
        count, counts = finalize(raw, cfg, g.n, g.m)
        visits = used_sms(raw.visits_per_sm, nsm)
        dev["count"] = raw.count_ms
        sbytes = scratch_bytes(og, cfg)
        counters = {"word_ops": raw.word_ops, "extract_bytes": raw.extract_bytes,
                    "kernel_ms": raw.count_ms, "tasks_run": raw.tasks_run,
                    "group_size": raw.group_size, "launches": raw.launches}
    count_ms = (time.perf_counter() - t1) * 1000.0
    return CountReport(n=g.n, m=g.m, d_max_undirected=g.max_degree(), d_max=og.d_max, config=cfg,
                       count=count, counts=counts, orient_ms=orient_ms, count_ms=count_ms,
                       load=load_stats(visits), scratch_bytes=sbytes,
                       degeneracy=ranking.degeneracy, device_ms=dev, counters=counters)
