"""Seeded synthetic graphs for the BASELINE.json configs.

All generators return a normalized ``(m, 2)`` int64 edge array: ``u < v`` per
row, rows sorted and unique, no self-loops -- the same normal form
``load_edge_list`` produces (reference graph.py:93-109), so the arrays feed
``from_edges`` directly.
"""

from __future__ import annotations

import hashlib

import numpy as np


def normalize(pairs) -> np.ndarray:
    """Drop self-loops, orient u < v, dedupe, sort (reference graph.py:93-109)."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    u, v = pairs[:, 0], pairs[:, 1]
    keep = u != v
    lo = np.minimum(u, v)[keep]
    hi = np.maximum(u, v)[keep]
    if lo.size == 0:
        return np.empty((0, 2), dtype=np.int64)
    key = (lo.astype(np.uint64) << np.uint64(32)) | hi.astype(np.uint64)
    key.sort()  # sort + adjacent dedup == np.unique, without its hash-table cost
    if key.size > 1:
        key = key[np.concatenate(([True], key[1:] != key[:-1]))]
    out = np.empty((key.size, 2), dtype=np.int64)
    out[:, 0] = (key >> np.uint64(32)).astype(np.int64)
    out[:, 1] = (key & np.uint64(0xFFFFFFFF)).astype(np.int64)
    return out


def erdos_renyi(n: int, p: float, seed: int = 0) -> np.ndarray:
    """G(n, p) over all pairs (triu order), ``default_rng(seed)``."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    mask = rng.random(iu.size) < p
    return np.stack([iu[mask], ju[mask]], axis=1).astype(np.int64)


def rmat(scale: int, edgefactor: int = 16, a=0.57, b=0.19, c=0.19, seed: int = 1,
         permute: bool = True) -> np.ndarray:
    """Graph500-style R-MAT / Kronecker edges, 2^scale ids, ef * 2^scale draws.

    Quadrant probabilities (a, b, c, d = 1-a-b-c); vertex labels are randomly
    permuted (as Graph500 does) so id order carries no degree information.
    Self-loops and duplicates are removed by ``normalize``.
    """
    return normalize(rmat_raw(scale, edgefactor, a, b, c, seed, permute))


def rmat_raw(scale: int, edgefactor: int = 16, a=0.57, b=0.19, c=0.19, seed: int = 1,
             permute: bool = True) -> np.ndarray:
    """The raw (m, 2) R-MAT draws of ``rmat`` in draw order, with their
    self-loops and repeated pairs (an un-normalized edge list)."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = edgefactor * n
    src = np.zeros(m, dtype=np.int64)
    dst = np.zeros(m, dtype=np.int64)
    ab = a + b
    c_norm = c / (1.0 - ab)
    a_norm = a / ab
    chunk = 1 << 22
    for lo in range(0, m, chunk):
        hi = min(m, lo + chunk)
        s = np.zeros(hi - lo, dtype=np.int64)
        d = np.zeros(hi - lo, dtype=np.int64)
        for level in range(scale):
            ii = rng.random(hi - lo) > ab
            jj = rng.random(hi - lo) > np.where(ii, c_norm, a_norm)
            s |= ii.astype(np.int64) << level
            d |= jj.astype(np.int64) << level
        src[lo:hi] = s
        dst[lo:hi] = d
    if permute:
        perm = rng.permutation(n).astype(np.int64)
        src = perm[src]
        dst = perm[dst]
    return np.stack([src, dst], axis=1)


def planted_cliques(n: int = 50_000, n_cliques: int = 100, size_lo: int = 30,
                    size_hi: int = 60, avg_deg: float = 10.0, seed: int = 3) -> np.ndarray:
    """Sparse G(n, avg_deg/n) background plus cliques of U[size_lo, size_hi] sizes
    planted on random vertex subsets."""
    rng = np.random.default_rng(seed)
    n_pairs = n * (n - 1) // 2
    m_bg = int(rng.binomial(n_pairs, avg_deg / n))
    bg = rng.integers(0, n, size=(m_bg, 2), dtype=np.int64)
    parts = [bg]
    for _ in range(n_cliques):
        size = int(rng.integers(size_lo, size_hi + 1))
        members = rng.choice(n, size=size, replace=False).astype(np.int64)
        iu, ju = np.triu_indices(size, 1)
        parts.append(np.stack([members[iu], members[ju]], axis=1))
    return normalize(np.concatenate(parts, axis=0))


def edges_digest(edges: np.ndarray) -> str:
    """sha256 of the normalized edge array (fixture pinning)."""
    return hashlib.sha256(np.ascontiguousarray(edges, dtype=np.int64).tobytes()).hexdigest()[:16]


# named workloads (BASELINE.json configs)
def workload(name: str) -> np.ndarray:
    if name == "er2000":
        return erdos_renyi(2000, 0.01, seed=0)
    if name.startswith("rmat"):
        return rmat(int(name[4:]), 16, seed=1)
    if name == "planted":
        return planted_cliques()
    raise ValueError(f"unknown workload {name!r}")
