"""Benchmark of the k-clique counting hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload rmat18] [--k 7] [--algo orient] [--scheme vertex]
                    [--criterion degeneracy]

A *step* is one pass of the reference's counting path over one synthetic
graph: ``run_count(g, cfg)`` = device degree/k-core ranking + orientation +
induced-bitmap extraction + traversal + exact reduction (the reference's
``orient_ms + count_ms``, PAPER.md:568 -- graph load excluded).  ``value`` is
k-cliques/s with the undirected CSR already resident in HBM; ``e2e`` is the
same metric through the public API from pinned host edge pairs
(``from_edges`` + ``run_count``, H2D of the pairs and D2H of the result inside
the timed region).  N>1: one process per GPU (torchrun), root-range shards,
one NCCL u64 all-reduce of the raw partials (shard.py), max-over-ranks time.

``--impl reference`` times the CPU restatement of the reference (oracle/,
C + pthreads, every host core) on a bounded task sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

# BASELINE.json configs[1]: RMAT scale-18 ef16, degeneracy orientation, 1 GPU
DEFAULTS = dict(workload="rmat18", k=7, algo="auto", scheme="auto", criterion="degeneracy")
METRIC = "k-cliques/sec"
FLUSH_BYTES = 512 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default=DEFAULTS["workload"])
    ap.add_argument("--k", type=int, default=DEFAULTS["k"])
    ap.add_argument("--algo", default=DEFAULTS["algo"])
    ap.add_argument("--scheme", default=DEFAULTS["scheme"])
    ap.add_argument("--criterion", default=DEFAULTS["criterion"])
    ap.add_argument("--group", type=int, default=0)
    ap.add_argument("--cpu-sample-s", type=float, default=12.0,
                    help="target CPU seconds of the oracle baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the side measurements of the other BASELINE.json configs")
    ap.add_argument("--per-k", default="4,7,10",
                    help="also time these k (1 warm-up + 2 timed steps each; runs over a "
                         "minute: the first run is the timed step) into per_k")
    a = ap.parse_args()
    from paper_2104_13209_b200.cli import b200_auto

    auto_algo, auto_scheme = b200_auto(a.k)
    if a.algo == "auto":
        a.algo = auto_algo
    if a.scheme == "auto":
        a.scheme = auto_scheme
    return a


def workload_edges(name):
    from paper_2104_13209_b200 import synth

    cache = os.environ.get("KC_GRAPH_CACHE")
    if cache:
        p = os.path.join(cache, f"{name}.npy")
        if os.path.exists(p):
            return np.load(p)
    e = synth.workload(name)
    if cache:
        os.makedirs(cache, exist_ok=True)
        np.save(os.path.join(cache, f"{name}.npy"), e)
    return e


def config_dict(a, world):
    return {"workload": a.workload, "k": a.k, "algorithm": a.algo, "scheme": a.scheme,
            "criterion": a.criterion, "group_size": a.group,
            "parallelism": f"root-range shards x{world}" if world > 1 else "1 GPU",
            "l2": "flushed between timed steps (512 MiB write)",
            "step": "run_count: rank + orient + extract + traverse + exact reduce"}


# ----------------------------------------------------------------------------
# dist helpers
# ----------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def count_kernel_launches(step):
    """Kernels launched by one step, counted by CUPTI through torch.profiler."""
    try:
        import torch
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        names = {}
        for ev in prof.events():
            if ev.device_type.name == "CUDA" and not ev.name.startswith("Memcpy") \
                    and not ev.name.startswith("Memset"):
                nm = ev.name.replace("(anonymous namespace)::", "").replace("void ", "")
                nm = nm.split("(")[0].split("<")[0][-60:]
                names[nm] = names.get(nm, 0) + 1
        return sum(names.values()), names
    except Exception as exc:  # profiler unavailable: report unknown
        return None, {"error": str(exc)[:200]}


def run_ours(a):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    # one process per GPU; KC_DIST_BACKEND=gloo + fewer GPUs than ranks lets the
    # N>1 path run on a 1-GPU box (ranks share devices) for testing
    backend = os.environ.get("KC_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    os.environ["KC_DEVICE"] = str(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2104_13209_b200 as kc
    from paper_2104_13209_b200 import _lib
    from paper_2104_13209_b200.shard import run_count_sharded

    _lib.load()
    edges = workload_edges(a.workload)
    g = kc.from_edges(edges, device=local)
    cfg = kc.RunConfig(k=a.k, algorithm=a.algo, scheme=a.scheme, criterion=a.criterion,
                       group_size=a.group)

    def step(graph=g):
        if world > 1:
            return run_count_sharded(graph, cfg, rank, world)
        return kc.run_count(graph, cfg)

    stream = torch.cuda.ExternalStream(_lib.graph_stream(g.handle), device=local)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device=f"cuda:{local}")
    rep = None
    for _ in range(max(a.warmup, 0)):
        rep = step()
    # every rank runs the profiled step: it contains the all-reduce at N>1
    n_launch, launch_names = count_kernel_launches(step)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        """device times: the job's time is the slowest rank's"""
        dev = f"cuda:{local}" if backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def time_steps(fn, n):
        """n steps timed with events on the library stream, L2 flushed between."""
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(n)]
        r = None
        barrier()
        for i in range(n):
            flush.fill_(i)
            torch.cuda.synchronize()
            evs[i][0].record(stream)
            r = fn()
            evs[i][1].record(stream)
            torch.cuda.synchronize()
        barrier()
        tot = float(sum(s0.elapsed_time(s1) for s0, s1 in evs))
        if world > 1:
            tot = max_over_ranks(tot)
        return r, tot

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    phase = {"orient_ms": [], "count_ms": [], "device_count_ms": []}
    with Clocks(local) as clk:
        barrier()
        for i in range(a.steps):
            flush.fill_(i)                       # L2 flush (outside the timed events)
            torch.cuda.synchronize()
            starts[i].record(stream)
            rep = step()
            ends[i].record(stream)
            torch.cuda.synchronize()
            phase["orient_ms"].append(rep.orient_ms)
            phase["count_ms"].append(rep.count_ms)
            phase["device_count_ms"].append((rep.device_ms or {}).get("count", 0.0))
        barrier()
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(sum(ms))
    if world > 1:
        total_ms = max_over_ranks(total_ms)
    count = rep.count
    value = count * a.steps / (total_ms / 1e3)

    # e2e: public API from pinned host pairs (H2D in the timed region)
    e2e = None
    if not a.no_e2e:
        pinned = torch.from_numpy(np.ascontiguousarray(edges)).pin_memory()
        host_edges = pinned.numpy()
        d2h = 8 * 8 + 8 * 1024 + (8 * (rep.d_max + 2) ** 2 if a.algo == "pivot" else 0)

        def e2e_step():
            gg = kc.from_edges(host_edges, device=local)
            r = step(gg)
            gg.free()
            return r

        if total_ms / a.steps < 60e3:  # (a step of minutes needs no warm-up)
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            r = e2e_step()
            assert r.count == count
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - t0) * 1e3
        if world > 1:
            e_ms = max_over_ranks(e_ms)
        e2e = {"value": count * a.steps / (e_ms / 1e3), "unit": "k-cliques/s",
               "ms_per_step": e_ms / a.steps, "h2d_bytes_per_step": int(edges.nbytes),
               "d2h_bytes_per_step": int(d2h), "timer": "host wall clock, synced"}

    # the other k of the metric (BASELINE.json: k=4/7/10), auto algorithm per k
    per_k = {}
    from paper_2104_13209_b200.cli import b200_auto

    for kk in [int(x) for x in a.per_k.split(",") if x.strip()]:
        if kk == a.k:
            per_k[str(kk)] = {"algorithm": a.algo, "scheme": a.scheme, "count": str(count),
                              "ms_per_step": total_ms / a.steps, "cliques_per_s": value}
            continue
        al, sc = b200_auto(kk)
        c2 = kc.RunConfig(k=kk, algorithm=al, scheme=sc, criterion=a.criterion)

        def st(c2=c2):
            if world > 1:
                return run_count_sharded(g, c2, rank, world)
            return kc.run_count(g, c2)

        # the first run is timed like a step; it is the warm-up unless it took
        # over a minute (k=10 pivot at RMAT-18: minutes per run -- the library
        # has no JIT and its buffers come from the stream-ordered pool, so a
        # first run is representative), then 2 (or 1 if > 20 s) timed steps
        r1, t1 = time_steps(st, 1)
        if t1 > 60e3:
            r2, t2, n_t, warm = r1, t1, 1, 0
        else:
            warm = 1
            n_t = 2 if t1 < 20e3 else 1
            r2, t2 = time_steps(st, n_t)
        per_k[str(kk)] = {"algorithm": al, "scheme": sc, "count": str(r2.count),
                          "ms_per_step": t2 / n_t, "cliques_per_s": r2.count * n_t / (t2 / 1e3),
                          "visits": r2.load.total, "steps": n_t, "warmup": warm}

    # the other BASELINE.json configs (1 GPU only; 1 warm-up + 2 timed steps)
    side = {}
    if world == 1 and not a.no_configs:
        side = other_configs(kc, time_steps, local)

    roof = roofline(kc, g, cfg, rep, a, local) if rank == 0 else None
    gold = golden(a.workload, dict(k=a.k, algorithm=a.algo, scheme=a.scheme,
                                   criterion=a.criterion))
    full_check = None
    if gold is not None:
        full_check = {"count_matches": str(count) == gold["count"],
                      "visits_match": (None if gold["visits"] is None
                                       else rep.load.total == gold["visits"]),
                      "oracle_count": gold["count"], "source": gold["source"]}
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(edges, a, count, target_s=a.cpu_sample_s)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "k-cliques/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_ms / a.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "dtype_note": "u32 bitmap words (AND/POPC), u64 count limbs",
            "data": "synthetic (seeded generator)",
            "config": config_dict(a, world), "count": str(count),
            "full_count_check": full_check,
            "phases_ms": {k: float(np.median(v)) for k, v in phase.items()},
            "d_max": rep.d_max, "degeneracy": rep.degeneracy, "visits": rep.load.total,
            "normalized_max": rep.load.normalized_max, "step_ms": ms,
            "clocks": clk.summary(), "e2e": e2e, "gpu_launches": (n_launch * a.steps
                                                                  if n_launch else None),
            "gpu_launches_per_step": n_launch, "kernels": launch_names,
            "roofline": roof, "cpu_baseline": cpu, "per_k": per_k, "configs": side,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def golden(workload, kw):
    """The reference-generated (tests/golden/medium.json) or full-graph oracle
    (tests/golden/scale.json) record of this exact run, if one is committed:
    {"count", "visits", "source"} (all-k: {"counts", "visits", "source"})."""
    gdir = os.path.join(HERE, "tests", "golden")
    crit = kw.get("criterion", "degree")
    try:
        with open(os.path.join(gdir, "medium.json")) as f:
            for rec in json.load(f):
                if rec["name"] != workload:
                    continue
                if kw.get("all_k"):
                    for r in rec.get("all_k", []):
                        if (r["scheme"], r["criterion"]) == (kw["scheme"], crit):
                            return {"counts": r["counts"], "visits": r["visits"],
                                    "source": "tests/golden/medium.json (reference run)"}
                for r in rec["runs"]:
                    if (r["k"], r["algorithm"], r["scheme"], r["criterion"]) == (
                            kw["k"], kw["algorithm"], kw["scheme"], crit):
                        return {"count": r["count"], "visits": r["visits"],
                                "source": "tests/golden/medium.json (reference run)"}
        with open(os.path.join(gdir, "scale.json")) as f:
            for r in json.load(f):
                if (r["workload"], r["k"], r["algorithm"], r["scheme"], r["criterion"],
                        r["all_k"]) == (workload, kw["k"], kw["algorithm"], kw["scheme"], crit,
                                        bool(kw.get("all_k"))):
                    return {"count": r["count"], "visits": r["visits"],
                            "source": "tests/golden/scale.json (full-graph oracle, "
                                      f"{r['workers']} threads, {r['oracle_count_s']} s)"}
        # counts do not depend on algorithm, scheme or order: any record of
        # this workload and k pins the count (visits then unchecked)
        with open(os.path.join(gdir, "scale.json")) as f:
            for r in json.load(f):
                if (r["workload"], r["k"]) == (workload, kw["k"]) and not kw.get("all_k"):
                    return {"count": r["count"], "visits": None,
                            "source": "tests/golden/scale.json (full-graph oracle, count only)"}
    except OSError:
        pass
    return None


def other_configs(kc, time_steps, local):
    """Side measurements of BASELINE.json configs 0, 2 and 3 (config 1 is the
    headline; config 4 is the multi-GPU run of this script with --gpus N),
    each checked against a committed reference / full-oracle record where one
    exists (`golden_match`) or against the oracle run here (ER)."""
    import oracle

    out = {}
    plan = [
        ("er2000_k4_degree_vertex", "er2000", dict(k=4, algorithm="orient", scheme="vertex",
                                                     criterion="degree"), True),
        ("planted_allk_pivot_edge", "planted", dict(k=10, algorithm="pivot", scheme="edge",
                                                      criterion="degeneracy", all_k=True), False),
        ("planted_allk_pivot_vertex", "planted", dict(k=10, algorithm="pivot", scheme="vertex",
                                                        criterion="degeneracy", all_k=True), False),
        ("rmat18_k4_bulk_order", "rmat18", dict(k=4, algorithm="orient", scheme="vertex",
                                                 criterion="degeneracy_bulk"), False),
    ]
    # BASELINE configs[2]: RMAT-20 edge- vs vertex-centric x sub-warp group size
    for scheme in ("vertex", "edge"):
        for gs in (32, 8, 1):
            plan.append((f"rmat20_k5_orient_{scheme}_g{gs}", "rmat20",
                         dict(k=5, algorithm="orient", scheme=scheme, criterion="degeneracy",
                              group_size=gs), False))
    # k = 10 (the metric's third k) where a run takes seconds: RMAT-14
    for scheme in ("edge", "vertex"):
        plan.append((f"rmat14_k10_pivot_{scheme}", "rmat14",
                     dict(k=10, algorithm="pivot", scheme=scheme, criterion="degeneracy"), False))
    graphs = {}
    for name, wl, kw, check in plan:
        try:
            if wl not in graphs:
                for _, old in graphs.values():
                    old.free()
                graphs.clear()
                e = workload_edges(wl)
                graphs[wl] = (e, kc.from_edges(e, device=local))
            e, gg = graphs[wl]
            c = kc.RunConfig(**kw)
            st = lambda gg=gg, c=c: kc.run_count(gg, c)  # noqa: E731
            n_t = 1 if check == "once" else 2
            if check != "once":
                st()  # warm-up (the library has no JIT; pools and caches)
            r, t = time_steps(st, n_t)
            rec = {"config": kw, "count": str(r.count), "ms_per_step": t / n_t,
                   "steps": n_t, "warmup": 0 if check == "once" else 1,
                   "cliques_per_s": r.count * n_t / (t / 1e3) if t else None,
                   "visits": r.load.total, "normalized_max": r.load.normalized_max,
                   "n": gg.n, "m": gg.m, "d_max": r.d_max,
                   "group_size_run": (r.counters or {}).get("group_size")}
            if r.counts:
                rec["max_k"] = max(r.counts)
                rec["counts_k10_k30"] = {str(k): str(r.counts.get(k, 0)) for k in (10, 20, 30)}
            gold = golden(wl, kw)
            if gold is not None:
                if "counts" in gold:
                    ok = {str(k): str(v) for k, v in (r.counts or {}).items()} == gold["counts"]
                else:
                    ok = str(r.count) == gold["count"]
                rec["golden_match"] = bool(ok and (gold["visits"] is None
                                                   or r.load.total == gold["visits"]))
                rec["golden_source"] = gold["source"]
            if check is True:  # bit-exact against the CPU oracle on the same input
                o = oracle.run_count(oracle.from_edges(e), kw["k"], kw["algorithm"], kw["scheme"],
                                     kw["criterion"], workers=os.cpu_count() or 1)
                rec["oracle_match"] = (o.count == r.count and o.visits == r.load.total)
            out[name] = rec
        except Exception as exc:  # a side measurement never breaks the headline line
            out[name] = {"error": str(exc)[:200]}
    for _, gg in graphs.values():
        gg.free()
    try:
        out["ingest_rmat20_raw"] = ingest_side(kc, local)
    except Exception as exc:
        out["ingest_rmat20_raw"] = {"error": str(exc)[:200]}
    return out


def ingest_side(kc, local):
    """K0: the edge-list normal form of graph.py:93-109
    on the raw RMAT-20 draws (16.8M pairs with loops and repeats), GPU vs the C
    restatement (single-thread qsort), results compared element-wise."""
    import oracle
    from paper_2104_13209_b200 import synth

    raw = synth.rmat_raw(20, 16, seed=1)
    kc.normalize_edges(raw[:1024], device=local)  # warm-up (pool, module load)
    dev_ms, wall_ms = [], []
    for _ in range(3):
        t0 = time.perf_counter()
        el, ms = kc.normalize_edges(raw, device=local, return_ms=True)
        wall_ms.append((time.perf_counter() - t0) * 1e3)
        dev_ms.append(ms)
    t0 = time.perf_counter()
    o_pairs, o_loops, o_self, o_dup = oracle.normalize_edges(raw)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    match = (np.array_equal(el.edges, o_pairs) and np.array_equal(el.loop_ids, o_loops)
             and (el.n_self_loops, el.n_duplicates) == (o_self, o_dup))
    fused = []
    for _ in range(3):
        t0 = time.perf_counter()
        g = kc.from_raw_edges(raw, device=local)
        fused.append(((time.perf_counter() - t0) * 1e3, g.normalize_ms, g.build_ms))
        fused_nm = (g.n, g.m)
        g.free()
    m_raw = raw.shape[0]
    dev = float(np.median(dev_ms))
    return {"m_raw": m_raw, "m_out": len(el), "n_self_loops": el.n_self_loops,
            "n_duplicates": el.n_duplicates,
            "gpu_ms": dev, "gpu_wall_ms": float(np.median(wall_ms)),
            "gpu_note": "device events around H2D (pageable) + sort/unique + D2H",
            "raw_pairs_per_s": m_raw / (dev / 1e3), "cpu_oracle_ms": cpu_ms,
            "cpu_note": "oracle/kc_oracle.c oc_normalize_edges, 1 thread", "oracle_match": match,
            "raw_to_csr": {"n": fused_nm[0], "m": fused_nm[1],
                           "wall_ms": float(np.median([f[0] for f in fused])),
                           "normalize_ms": float(np.median([f[1] for f in fused])),
                           "csr_build_ms": float(np.median([f[2] for f in fused])),
                           "note": "from_raw_edges: K0 kept on the device, then K1 (one H2D)"}}


def roofline(kc, g, cfg, rep, a, local):
    """Roofline of the dominant kernel (k_count) from an instrumented re-run.

    ALU bound: algorithmic word-ops = sum over expanded tree nodes of the
    u32 words of the row AND+POPC'd; the peak is the
    measured sustained AND+POPC word rate of this GPU (kc_microbench).
    """
    try:
        from paper_2104_13209_b200 import profile as kprof
    except ImportError:
        return None
    try:
        return kprof.roofline(g, cfg, rep)
    except Exception as exc:
        return {"error": str(exc)[:300]}


# ----------------------------------------------------------------------------
# CPU baseline / reference arm: the C restatement of the reference
# ----------------------------------------------------------------------------
def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuBaseline:
    """The C restatement of the reference (oracle/, pthreads, every host core)
    timed on a stratified sample of the workload's tasks, projected to the
    whole graph.

    prepare(): full-graph CSR, ranking (the reference's heap order for
    degeneracy) and orientation on the CPU -- the ranking + orientation time
    is measured and charged in full.  Tasks (make_tasks order,
    scheduler.py:89-95) are sorted by a cost proxy (out-degree for vertex
    tasks, min(d+(u), d+(v)) for edge tasks) and every `step`-th one is taken
    (a systematic sample across all strata, heavy tasks included); `step` is
    calibrated once so a sample costs ~target_s of wall time.
    measure(): the pool runs the sample (heaviest task first) and reports
    every thread's CPU time; the whole-graph estimate is the ratio estimator
        wall = orient_s + (sample thread-CPU s) * (full count / sample count) / cores
    i.e. the sample's cliques per core-second, with the full run's work queue
    keeping every core busy (thread-CPU time is immune to the sample's tail
    imbalance; the full run has 10^5+ tasks).  value = exact count / wall.
    The stratum-scaled projection is reported next to it, and the committed
    whole-graph oracle run of the same workload (tests/golden/scale.json:
    count, wall, cores, CPU model) as `full_run`."""

    def __init__(self, edges, a, target_s=12.0, workers=None):
        import oracle

        self.a = a
        self.workers = workers or os.cpu_count() or 1
        g = oracle.from_edges(edges)
        t0 = time.perf_counter()
        crit = "degeneracy" if a.criterion.startswith("degeneracy") else a.criterion
        rank, degen = oracle.compute_rank(g, crit)
        self.og = oracle.orient(g, rank, degen)
        self.orient_s = time.perf_counter() - t0
        tasks = oracle.make_tasks(self.og, a.scheme)
        dout = np.diff(self.og.row_ptr)
        if a.scheme == "vertex":
            proxy = dout[tasks]
        else:
            proxy = np.minimum(dout[self.og.coo_src[tasks]], dout[self.og.col[tasks]])
        self.order = tasks[np.argsort(-proxy, kind="stable")]
        n = max(self.order.size, 1)
        # calibration: from a sparse sample (16 tasks) to denser ones until a
        # sample costs ~1 s of wall time (RMAT-22 k=7: one heavy task alone
        # is seconds of CPU; a fixed 1/256 sample would be hours)
        step0 = max(1, n // 16)
        while True:
            t0 = time.perf_counter()
            _, _, b0, _ = self._run(step0)
            if step0 == 1 or time.perf_counter() - t0 > 1.0 or step0 <= n // 256:
                break
            step0 = max(1, step0 // 4)
        # thread-CPU seconds of the whole graph ~ b0 * step0; a sample of
        # `target_s` wall on every core takes step = that / (target_s * cores)
        self.step = min(n, max(1, int(b0 * step0 / max(target_s * self.workers, 1e-9))))

    def _run(self, step):
        import oracle

        sample = self.order[step // 2::step]
        c, vis, busy = oracle.run_task_list(self.og, self.a.k, self.a.algo, self.a.scheme,
                                            sample, self.workers)
        return c, vis, float(sum(busy)), int(sample.size)

    def measure(self, full_count=None):
        step = self.step
        t1 = time.perf_counter()
        c1, v1, b1, n1 = self._run(step)
        sample_wall = time.perf_counter() - t1
        count = full_count if full_count is not None else c1 * step
        # ratio estimator: the sample's cliques per thread-CPU second hold for
        # the whole graph (cost tracks cliques much more tightly than the
        # cost proxy does); the full run's pool keeps every core busy
        busy_full = b1 * (count / c1) if c1 else b1 * step
        wall = self.orient_s + busy_full / self.workers
        rec = {"value": count / wall if wall > 0 else None, "unit": "k-cliques/s",
               "cores": self.workers, "kind": "port", "cpu_model": _cpu_model(),
               "sample": (f"oracle/kc_oracle.c worker pool on every {step}-th task of "
                          f"{self.order.size} sorted by cost proxy ({n1} tasks, "
                          f"{100.0 / step:.2f}%; {sample_wall:.1f}s wall, {b1:.1f} thread-CPU s)"
                          f" + full-graph ranking/orientation {self.orient_s:.2f}s"),
               "estimated_full_wall_s": wall, "orient_s_full": self.orient_s,
               "estimated_full_wall_s_stratum_scaling": self.orient_s + b1 * step / self.workers,
               "sample_count_scaled": str(c1 * step), "sample_visits_scaled": v1 * step,
               "step": step}
        rec.update(full_run_record(self.a))
        return rec


def cpu_baseline(edges, a, full_count=None, target_s=12.0, workers=None):
    return CpuBaseline(edges, a, target_s, workers).measure(full_count)


def full_run_record(a):
    """The committed whole-graph oracle run of this exact workload, if any."""
    try:
        with open(os.path.join(HERE, "tests", "golden", "scale.json")) as f:
            recs = json.load(f)
    except OSError:
        return {}
    for r in recs:
        if (r["workload"], r["k"], r["algorithm"], r["scheme"], r["criterion"]) == (
                a.workload, a.k, a.algo, a.scheme,
                "degeneracy" if a.criterion.startswith("degeneracy") else a.criterion) \
                and not r["all_k"]:
            wall = r["oracle_orient_s"] + r["oracle_count_s"]
            return {"full_run": {"count": r["count"], "visits": r["visits"], "wall_s": wall,
                                 "value": int(r["count"]) / wall, "cores": r["workers"],
                                 "cpu_model": r["cpu_model"], "source": r["recipe"],
                                 "when": r["when"]}}
    return {}


def run_reference(a):
    """The reference arm: the CPU restatement on this host (rank 0 only), on the
    same workload / metric; each step is one measured sample (CpuBaseline)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    edges = workload_edges(a.workload)
    # a compiled CPU port needs no warm-up beyond the first (page-faulting) pass:
    # one warm-up step whatever --warmup says keeps the arm within minutes
    per = max(2.0, min(a.cpu_sample_s, 150.0 / max(a.steps + 1, 1)))
    cb = CpuBaseline(edges, a, target_s=per)
    full = cb.measure()  # warm-up
    full_count = int(full["full_run"]["count"]) if "full_run" in full else None
    vals, ms = [], []
    last = None
    for _ in range(a.steps):
        t0 = time.perf_counter()
        last = cb.measure(full_count)
        ms.append((time.perf_counter() - t0) * 1e3)
        vals.append(last["value"])
    value = float(np.median(vals))
    cpu = dict(last)
    cpu["value"] = value
    cpu["values_per_step"] = vals
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "k-cliques/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": float(np.mean(ms)), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded generator)", "config": config_dict(a, world),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "k-cliques/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
