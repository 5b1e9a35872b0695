"""Seeded synthetic inputs for BASELINE.json's configs (host side).

* gen_random_graph / gen_random_queries / gen_insert_workload restate the
  reference generators (workload.py:41-48, 116-172) on the stdlib Mersenne
  Twister so config 1 reproduces the reference's own graph and queries
  exactly (checked against tests/golden/cfg1.npz).
* rmat_edges is the R-MAT generator configs 2-5 need (the reference ships
  none): numpy PCG64, quadrant probabilities
  (a, b, c, d), self-loops dropped; duplicates are removed by the graph build.
  Vertex ids are NOT permuted, so low ids are the hubs.
* positive_queries stands in for "(u, random vertex on a BFS path from u)":
  u uniform over vertices with out-degree > 0, v the endpoint of a seeded
  random walk of 1..8 steps (pairs with v == u dropped) -- SURVEY.md §8(d).
"""
from __future__ import annotations

import random

import numpy as np

from .errors import ConfigError, WorkloadExhaustedError


def gen_random_graph(n: int, avg_degree: float, seed: int, *, acyclic: bool = False
                     ) -> tuple[np.ndarray, np.ndarray]:
    """Edge arrays of the reference's uniform random digraph (workload.py:147-172)."""
    if n < 1:
        raise ConfigError("n must be >= 1")
    rng = random.Random(seed)
    m = min(int(round(avg_degree * n)), n * (n - 1) // (2 if acyclic else 1))
    order = list(range(n))
    rng.shuffle(order)
    rank = {v: i for i, v in enumerate(order)}
    seen: set[tuple[int, int]] = set()
    src: list[int] = []
    dst: list[int] = []
    attempts, cap = 0, 100 * m + 1000
    while len(src) < m and attempts < cap:
        attempts += 1
        u = rng.randrange(n)
        v = rng.randrange(n)
        if u == v:
            continue
        if acyclic and rank[u] > rank[v]:
            u, v = v, u
        if (u, v) in seen:
            continue
        seen.add((u, v))
        src.append(u)
        dst.append(v)
    return np.array(src, np.uint32), np.array(dst, np.uint32)


def gen_random_queries(n_vertices: int, count: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Uniform (u, v) pairs of the reference generator (workload.py:41-48)."""
    if count < 0:
        raise ConfigError(f"count must be >= 0, got {count}")
    if count > 0 and n_vertices < 1:
        raise ConfigError("cannot sample queries from an empty graph")
    rng = random.Random(seed)
    flat = [rng.randrange(n_vertices) for _ in range(2 * count)]
    a = np.array(flat, np.uint32).reshape(-1, 2) if count else np.zeros((0, 2), np.uint32)
    return np.ascontiguousarray(a[:, 0]), np.ascontiguousarray(a[:, 1])


def uniform_queries(n: int, count: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Fast seeded uniform pairs (numpy PCG64) for the large configs."""
    rng = np.random.default_rng(seed)
    return (rng.integers(0, n, count, dtype=np.uint32), rng.integers(0, n, count, dtype=np.uint32))


def rmat_edges(scale: int, edge_factor: int, seed: int, a: float = 0.57, b: float = 0.19,
               c: float = 0.19, chunk: int = 1 << 22) -> tuple[np.ndarray, np.ndarray]:
    """R-MAT edges (2^scale vertices, edge_factor * 2^scale draws), self-loops dropped."""
    m = edge_factor << scale
    rng = np.random.default_rng(seed)
    ab, abc = a + b, a + b + c
    srcs, dsts = [], []
    for lo in range(0, m, chunk):
        cnt = min(chunk, m - lo)
        s = np.zeros(cnt, np.uint32)
        d = np.zeros(cnt, np.uint32)
        for bit in range(scale):
            r = rng.random(cnt, dtype=np.float32)
            sb = r >= ab                          # quadrants c, d
            db = ((r >= a) & (r < ab)) | (r >= abc)  # quadrants b, d
            s |= sb.astype(np.uint32) << np.uint32(bit)
            d |= db.astype(np.uint32) << np.uint32(bit)
        keep = s != d
        srcs.append(s[keep])
        dsts.append(d[keep])
    return np.concatenate(srcs), np.concatenate(dsts)


def host_csr(n: int, src: np.ndarray, dst: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Deduplicated CSR on the host (numpy) for generators only."""
    key = np.unique(src.astype(np.uint64) << np.uint64(32) | dst.astype(np.uint64))
    s = (key >> np.uint64(32)).astype(np.int64)
    col = (key & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    ptr = np.zeros(n + 1, np.int64)
    ptr[1:] = np.cumsum(np.bincount(s, minlength=n))
    return ptr, col


def positive_queries(n: int, src: np.ndarray, dst: np.ndarray, count: int, seed: int,
                     max_steps: int = 8) -> tuple[np.ndarray, np.ndarray]:
    """(u, endpoint of a 1..max_steps random walk from u) pairs, v != u."""
    ptr, col = host_csr(n, src, dst)
    deg = np.diff(ptr)
    starts = np.flatnonzero(deg > 0)
    rng = np.random.default_rng(seed)
    us, vs = [], []
    need = count
    while need > 0:
        k = int(need * 1.3) + 16
        u = starts[rng.integers(0, len(starts), k)]
        steps = rng.integers(1, max_steps + 1, k)
        x = u.copy()
        for t in range(max_steps):
            active = (steps > t) & (deg[x] > 0)
            pick = ptr[x] + (rng.random(k) * np.maximum(deg[x], 1)).astype(np.int64)
            x = np.where(active, col[np.minimum(pick, len(col) - 1)], x)
        ok = x != u
        us.append(u[ok])
        vs.append(x[ok])
        need -= int(ok.sum())
    return (np.concatenate(us)[:count].astype(np.uint32), np.concatenate(vs)[:count].astype(np.uint32))


def gen_insert_workload(src: np.ndarray, dst: np.ndarray, n: int, count: int, seed: int,
                        exclude: tuple[np.ndarray, np.ndarray] | None = None
                        ) -> tuple[np.ndarray, np.ndarray]:
    """Absent, distinct, non-loop edges (the rule of workload.py:116-141), vectorised.

    `exclude` adds extra edges (e.g. earlier batches) that must not be drawn.
    """
    if count < 0:
        raise ConfigError(f"count must be >= 0, got {count}")
    present = src.astype(np.uint64) << np.uint64(32) | dst.astype(np.uint64)
    if exclude is not None:
        present = np.concatenate([present, exclude[0].astype(np.uint64) << np.uint64(32)
                                  | exclude[1].astype(np.uint64)])
    present = np.unique(present)
    rng = np.random.default_rng(seed)
    chosen = np.zeros(0, np.uint64)
    order = np.zeros(0, np.int64)
    tries = 0
    while len(chosen) < count:
        tries += 1
        if tries > 100:
            raise WorkloadExhaustedError(f"could only draw {len(chosen)}/{count} new edges")
        k = 2 * (count - len(chosen)) + 64
        u = rng.integers(0, n, k, dtype=np.uint64)
        v = rng.integers(0, n, k, dtype=np.uint64)
        key = u << np.uint64(32) | v
        key = key[u != v]
        pos = np.searchsorted(present, key)
        pos = np.minimum(pos, max(len(present) - 1, 0))
        absent = present[pos] != key if len(present) else np.ones(len(key), bool)
        key = key[absent]
        allk = np.concatenate([chosen, key])
        _, first = np.unique(allk, return_index=True)
        first.sort()
        chosen = allk[first]
    chosen = chosen[:count]
    return ((chosen >> np.uint64(32)).astype(np.uint32), (chosen & np.uint64(0xFFFFFFFF)).astype(np.uint32))


def rmat_edges_device(scale: int, edge_factor: int, seed: int, device: int = 0, a: float = 0.57,
                      b: float = 0.19, c: float = 0.19):
    """R-MAT edges generated on the GPU (dbl_rmat_generate), self-loops dropped.

    Returns (src, dst) int32 CUDA tensors holding uint32 ids.  Used for the
    large configs (2^22..2^26) where host generation would dominate.
    """
    import torch

    from . import _native as N
    m = edge_factor << scale
    dev = torch.device("cuda", device)
    src = torch.empty(m, dtype=torch.int32, device=dev)
    dst = torch.empty(m, dtype=torch.int32, device=dev)
    N.call("dbl_rmat_generate", scale, m, seed, a, b, c, N.ptr(src), N.ptr(dst), device)
    keep = src != dst
    return src[keep].contiguous(), dst[keep].contiguous()
