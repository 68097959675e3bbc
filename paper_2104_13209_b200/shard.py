"""Multi-GPU root-range sharding.

One process per GPU.  Every rank builds and orients the graph on its own
device (replicated preprocessing), takes a contiguous range of make_tasks
order balanced by a prefix sum over a per-task cost estimate, runs kc_count
on it, and the ranks meet in ONE element-wise u64 all-reduce of the raw
partials (count limbs, visits, pivot leaf histogram) -- exact, because every
field is a plain sum.  The host then carries the limbs / expands the
histogram into the exact count (scheduler.finalize).

The collective is ``torch.distributed.all_reduce`` (NCCL on GPUs, gloo in the
CPU tests); tasks are independent, so this is the only exchange.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .scheduler import CountReport, RawCount, RunConfig, device_count_raw, finalize, load_stats
from .scheduler import scratch_bytes, used_sms, validate


def balanced_ranges(costs: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Split [0, len(costs)) into ``world`` contiguous ranges of ~equal cost."""
    costs = np.asarray(costs, dtype=np.float64)
    n = costs.size
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(world - 1, 0)
    cum = np.cumsum(costs)
    total = cum[-1] if cum[-1] > 0 else float(n)
    if cum[-1] <= 0:
        cum = np.arange(1, n + 1, dtype=np.float64)
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")) + 1)
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(world)]


def _args(cfg: RunConfig):
    k = max(cfg.k, 3) if cfg.all_k else cfg.k
    return _lib.KcCountArgs(k, _lib.ALGO[cfg.algorithm], _lib.SCHEME[cfg.scheme],
                            1 if cfg.all_k else 0, int(cfg.group_size), 0, 0, -1)


def task_costs(og, cfg: RunConfig) -> np.ndarray:
    """Per-task cost estimate in make_tasks order (kc_task_costs, on the device)."""
    L = _lib.load()
    h = og.ensure_on_device()
    n = ctypes.c_int64()
    _lib.check(L.kc_num_tasks(h, _lib.SCHEME[cfg.scheme], ctypes.byref(n)))
    costs = np.zeros(max(n.value, 1), dtype=np.int64)
    a = _args(cfg)
    _lib.check(L.kc_task_costs(h, ctypes.byref(a), _lib._ptr(costs), n.value))
    return costs[:n.value]


def shard_ranges(og, cfg: RunConfig, world: int) -> list[tuple[int, int]]:
    """balanced_ranges over kc_task_costs, computed on the device: only the
    world + 1 cuts cross to the host (kc_shard_ranges)."""
    L = _lib.load()
    h = og.ensure_on_device()
    cuts = np.zeros(world + 1, dtype=np.int64)
    a = _args(cfg)
    _lib.check(L.kc_shard_ranges(h, ctypes.byref(a), int(world), _lib._ptr(cuts)))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(world)]


def spread_per_rank(raw: RawCount, rank: int, world: int) -> RawCount:
    """Place this rank's per-SM visit counters in its own slice of a
    world x SM_SLOTS vector, so the element-wise all-reduce keeps load
    statistics per (rank, SM) instead of summing SMs of different GPUs."""
    per = np.asarray(raw.visits_per_sm, dtype=np.uint64)
    wide = np.zeros(world * per.size, dtype=np.uint64)
    wide[rank * per.size:(rank + 1) * per.size] = per
    return RawCount(raw.limbs, raw.visits, raw.tasks_run, raw.hist, wide, raw.count_ms,
                    raw.word_ops, raw.extract_bytes, raw.group_size, raw.launches)


def per_rank_sms(wide, world: int, nsm: int) -> list:
    """Concatenated per-SM counters of every rank (each trimmed to its SMs)."""
    wide = np.asarray(wide)
    width = wide.size // max(world, 1)
    out = []
    for r in range(world):
        out += used_sms(wide[r * width:(r + 1) * width], nsm)
    return out


def allreduce_raw(raw: RawCount, group=None) -> RawCount:
    """Element-wise u64 sum of the raw partials across ranks (one collective)."""
    import torch
    import torch.distributed as dist

    vec = raw.as_vector()
    # u64 sums travel as int64 bit patterns; two's-complement addition is the
    # same modulo 2^64 and every field stays far below 2^63
    t = torch.from_numpy(vec.view(np.int64).copy())
    backend = dist.get_backend(group)
    if backend == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    out = t.cpu().numpy().view(np.uint64)
    return raw.from_vector(out)


def run_count_sharded(g, cfg: RunConfig, rank: int, world: int, group=None,
                      og=None, ranges=None) -> CountReport:
    """run_count over this rank's shard + all-reduce; identical result on every rank."""
    import time

    from .orientation import rank_and_orient

    validate(cfg)
    t0 = time.perf_counter()
    if og is None:
        og = rank_and_orient(g, cfg.criterion)
    orient_ms = (time.perf_counter() - t0) * 1000.0
    t1 = time.perf_counter()
    if ranges is None:
        ranges = shard_ranges(og, cfg, world)
    lo, hi = ranges[rank]
    raw = device_count_raw(og, cfg, lo, hi)
    counters = {"word_ops": raw.word_ops, "extract_bytes": raw.extract_bytes,
                "kernel_ms": raw.count_ms, "tasks_run": raw.tasks_run}
    nsm = _lib.num_sms(g.device)
    raw = spread_per_rank(raw, rank, world)
    if world > 1:
        raw = allreduce_raw(raw, group)
    count, counts = finalize(raw, cfg, g.n, g.m)
    count_ms = (time.perf_counter() - t1) * 1000.0
    return CountReport(n=g.n, m=g.m, d_max_undirected=g.max_degree(), d_max=og.d_max, config=cfg,
                       count=count, counts=counts, orient_ms=orient_ms, count_ms=count_ms,
                       load=load_stats(per_rank_sms(raw.visits_per_sm, world, nsm)),
                       scratch_bytes=scratch_bytes(og, cfg), degeneracy=og.ranking.degeneracy,
                       device_ms={"count": raw.count_ms}, counters=counters)
