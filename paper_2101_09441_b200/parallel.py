"""Multi-GPU paths: query batches split over replicas, and the label build.

SURVEY.md §8(e).  The reference's only parallelism is the fork pool of
query_batch (queries.py:224-247): contiguous, order-preserving slices of
ceil(q / workers) queries, one per worker.  Here the workers are GPUs.

* Queries.  Every GPU holds a replica of the graph (CSR + CSC) and of the
  label table; a batch is cut into the reference's slices and each GPU
  answers one -- no collective on the data path.
  - one process, several devices: query_batch_sharded(replicas, queries)
    runs dbl_query_multi (one host thread per device, slices concurrent);
  - one process per GPU (torchrun): query_batch_split(g, idx, u, v, rank,
    world) answers this rank's slice; gather=True all-gathers the codes.
* Build.  Two modes, chosen by build_index_distributed(mode=...):
  - "replicated" (default): every rank runs the whole build on its replica.
    No collective.  Measured to be faster at every N: the
    build writes the label table at HBM rate (the cfg5 table, 8.6 GB, in
    ~1.3 ms of a 7.1 ms build), while shipping 7/8 of it over NVLink
    (~0.75-0.9 TB/s per GPU) costs more than computing it.
  - "words": the north_star's landmark/bit-word sharding.  Each 64-bit word
    of a record ({dl_in | bl_in | dl_out | bl_out}, csrc/internal.cuh) is an
    independent least fixpoint, so ranks build disjoint word sets of the
    same table (the frozen metadata is deterministic and replicated), pack
    their words into a word-major slab, all-gather the slabs (NCCL on GPUs,
    staged through host memory under gloo) and scatter the peers' words back
    into their own table (K5 interleave).

The word exchange is written against a small engine interface so that its
host logic is tested on CPU with gloo (tests/test_parallel.py) and the
device path with several ranks sharing one GPU (tests/test_multirank.py).
"""
from __future__ import annotations

import ctypes
import time
from typing import Callable, Protocol, Sequence

import numpy as np


# ------------------------------------------------------------------ queries

def slice_bounds(count: int, parts: int) -> list[tuple[int, int]]:
    """The reference pool's slices (queries.py:231-232): chunk = ceil(count /
    parts), bounds (i, min(i + chunk, count)) for i in range(0, count, chunk),
    padded with empty slices up to `parts` entries."""
    if parts < 1:
        from .errors import ConfigError
        raise ConfigError(f"parts must be >= 1, got {parts}")
    chunk = max(1, -(-count // parts))
    b = [(i, min(i + chunk, count)) for i in range(0, count, chunk)]
    while len(b) < parts:
        b.append((count, count))
    return b


def replicate(n: int, src, dst, devices: Sequence[int], config=None):
    """Graph + index replicas on `devices` (each builds its own: no collective).

    Returns a list of (DynamicGraph, DblIndex), one per device.
    """
    from .graph import DynamicGraph
    from .labels import build_index
    if hasattr(src, "is_cuda"):   # device tensors live on one GPU: replicate from host copies
        src, dst = src.cpu().numpy(), dst.cpu().numpy()
    out = []
    for d in devices:
        g = DynamicGraph.from_edges(n, src, dst, device=d)
        out.append((g, build_index(g, config)))
    return out


def query_batch_sharded(replicas, queries, flags=None):
    """query_batch over several replicas (one per device) in one process.

    `replicas` is a list of (graph, index) pairs with identical contents
    (see replicate()).  The batch is split into the reference's contiguous
    slices, answered concurrently by dbl_query_multi, and returned in input
    order as (Outcomes, BatchStats), exactly like query_batch.  `queries`
    may be a (u, v) pair of CUDA tensors on one GPU: the other GPUs then read
    their slices and write their answers over NVLink (peer access).
    """
    from . import _native as N
    from .queries import DEFAULT_FLAGS, BatchStats, Outcomes, _check_consistent, _pairs_to_arrays
    from .graph import as_device_graph
    flags = DEFAULT_FLAGS if flags is None else flags
    if not replicas:
        from .errors import ConfigError
        raise ConfigError("query_batch_sharded needs at least one replica")
    gs, ids = [], []
    for g, idx in replicas:
        g = as_device_graph(g)
        _check_consistent(g, idx)
        gs.append(g.handle)
        ids.append(idx.handle)
    garr = (ctypes.c_void_p * len(gs))(*[h.value for h in gs])
    iarr = (ctypes.c_void_p * len(ids))(*[h.value for h in ids])
    if isinstance(queries, tuple) and len(queries) == 2 and all(getattr(q, "is_cuda", False) for q in queries):
        # a batch resident on one GPU: slices read and codes written over NVLink
        import torch
        u, v = queries
        N.check_device_ids(u, v, u.device.index)
        torch.cuda.current_stream(u.device).synchronize()
        codes = torch.empty(u.numel(), dtype=torch.uint8, device=u.device)
        vis = torch.empty(u.numel(), dtype=torch.int32, device=u.device)
        t0 = time.perf_counter()
        N.call("dbl_query_multi", iarr, garr, len(gs), N.ptr(u), N.ptr(v), u.numel(), flags.bits(),
               N.ptr(codes), N.ptr(vis), N.MEM_DEVICE)
        elapsed_ms = (time.perf_counter() - t0) * 1e3
        out = Outcomes(codes.cpu().numpy(), vis.cpu().numpy().view(np.uint32))
        return out, BatchStats.collect(out, elapsed_ms)
    u, v = _pairs_to_arrays(queries)
    codes = np.zeros(len(u), np.uint8)
    vis = np.zeros(len(u), np.uint32)
    t0 = time.perf_counter()
    N.call("dbl_query_multi", iarr, garr, len(gs), N.ptr(u), N.ptr(v), len(u), flags.bits(),
           N.ptr(codes), N.ptr(vis), N.MEM_HOST)
    elapsed_ms = (time.perf_counter() - t0) * 1e3
    out = Outcomes(codes, vis)
    return out, BatchStats.collect(out, elapsed_ms)


def query_batch_split(g, idx, u, v, rank: int, world: int, flags=None, gather: bool = True,
                      group=None):
    """One process per GPU: answer this rank's slice of the batch (u, v).

    u, v are the WHOLE batch (host arrays or tensors, identical on every
    rank); rank r answers slice slice_bounds(len(u), world)[r].  With
    gather=True the codes of all slices are all-gathered (torch.distributed,
    any backend) and every rank returns the whole batch's codes in input
    order; otherwise it returns only its slice's codes.
    """
    from .queries import DEFAULT_FLAGS, query_codes
    flags = DEFAULT_FLAGS if flags is None else flags
    count = len(u)
    lo, hi = slice_bounds(count, world)[rank]
    codes, _ = query_codes(g, idx, u[lo:hi], v[lo:hi], flags, with_visited=False)
    if not gather or world == 1:
        return codes
    import torch
    import torch.distributed as dist
    t = codes if hasattr(codes, "is_cuda") else torch.from_numpy(np.asarray(codes))
    if dist.get_backend(group) == "nccl":
        t = t.to(f"cuda:{g.device}")
    else:
        t = t.cpu()
    b = slice_bounds(count, world)
    chunk = max(b[0][1] - b[0][0], 1)
    padded = torch.zeros(chunk, dtype=torch.uint8, device=t.device)
    padded[:t.numel()] = t
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    full = torch.cat([p[:h - l] for p, (l, h) in zip(parts, b)])
    return full.cpu().numpy() if not hasattr(codes, "is_cuda") else full


# -------------------------------------------------------------------- build

def plan_words(rw: int, world: int) -> list[list[int]]:
    """Round-robin record words over ranks (word w -> rank w % world)."""
    return [[w for w in range(rw) if w % world == r] for r in range(world)]


class WordEngine(Protocol):
    n: int
    rw: int

    def build_words(self, words: Sequence[int]) -> None: ...
    def pack(self, words: Sequence[int], out) -> None: ...
    def unpack(self, words: Sequence[int], slab) -> None: ...
    def empty_slab(self, nwords: int): ...


def sharded_exchange(engine: WordEngine, rank: int, world: int,
                     allgather: Callable[[object, object], None]) -> list[list[int]]:
    """Build this rank's words, allgather all slabs, scatter peers' words.

    allgather(out, inp) must fill `out` (world * slab) with every rank's `inp`
    in rank order (dist.all_gather_into_tensor semantics).
    """
    plan = plan_words(engine.rw, world)
    own = plan[rank]
    if own:
        engine.build_words(own)
    maxw = max(len(p) for p in plan)
    slab = engine.empty_slab(maxw)
    if own:
        engine.pack(own, slab)
    gathered = engine.empty_slab(maxw * world)
    allgather(gathered, slab)
    per = maxw * engine.n
    for r in range(world):
        if r == rank or not plan[r]:
            continue
        engine.unpack(plan[r], gathered[r * per:(r + 1) * per])
    return plan


class DeviceWordEngine:
    """WordEngine over the C ABI; slabs are int64 CUDA tensors (u64 bits)."""

    def __init__(self, g, idx):
        from . import _native as N
        self.N = N
        self.g, self.idx = g, idx
        self.n = idx.vertex_count
        self.rw = 2 * (idx.wdl + idx.wbl)
        self.device = g.device

    def build_words(self, words):
        w = np.ascontiguousarray(words, dtype=np.uint32)
        self.N.call("dbl_index_build_words", self.g.handle, self.idx.handle, self.N.ptr(w), len(w))

    def empty_slab(self, nwords: int):
        import torch
        return torch.zeros(max(nwords, 1) * self.n, dtype=torch.int64, device=f"cuda:{self.device}")

    def _stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def pack(self, words, out):
        w = np.ascontiguousarray(words, dtype=np.uint32)
        self.N.call("dbl_index_pack_words", self.idx.handle, self.N.ptr(w), len(w), self.N.ptr(out),
                    self._stream())

    def unpack(self, words, slab):
        w = np.ascontiguousarray(words, dtype=np.uint32)
        self.N.call("dbl_index_unpack_words", self.idx.handle, self.N.ptr(w), len(w), self.N.ptr(slab),
                    self._stream())
        self.idx._invalidate()


def create_index(g, config=None, *, landmarks=None, leaf_sets=None):
    """Select/pin metadata and seed labels without propagating (dbl_index_create)."""
    from . import _native as N
    from .graph import as_device_graph
    from .labels import DblIndex, IndexConfig, LandmarkSet, LeafSets, LandmarkStrategy
    g = as_device_graph(g)
    cfg = config if config is not None else IndexConfig()
    cfg.validate(g.vertex_count)
    lm = fl = bk = None
    if landmarks is not None:
        LandmarkSet.of(landmarks)
        lm = N.u32_array(list(landmarks))
    if leaf_sets is not None:
        if not isinstance(leaf_sets, LeafSets):
            leaf_sets = LeafSets(leaf_sets.leaves_in, leaf_sets.leaves_out, leaf_sets.bucket)
        fl, bk = leaf_sets.for_vertex_count(g.vertex_count)
    h = ctypes.c_void_p()
    N.call("dbl_index_create", g.handle, ctypes.byref(cfg.to_c()), N.ptr(lm), N.ptr(fl), N.ptr(bk),
           None, None, 0, ctypes.byref(h))
    return DblIndex(h, g, IndexConfig(cfg.k, cfg.k_prime, LandmarkStrategy(cfg.landmark_strategy),
                                      cfg.leaf_threshold, cfg.hash_seed))


def _allgather_for(group):
    """all_gather_into_tensor on the group's backend: device tensors under
    NCCL, staged through host memory otherwise (gloo has no device allgather)."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        def allgather(out, inp):
            dist.all_gather_into_tensor(out, inp, group=group)
        return allgather
    world = dist.get_world_size(group)

    def allgather(out, inp):
        h = inp.cpu()
        parts = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(parts, h, group=group)
        out.copy_(torch.cat(parts).to(out.device))
    return allgather


def sharded_build(g, config, rank: int, world: int, group=None):
    """build_index with record words sharded across `world` ranks + allgather."""
    import torch
    idx = create_index(g, config)
    eng = DeviceWordEngine(g, idx)
    # the engine's stream runs the word builds; the allgather runs on torch's
    # stream of the same device, which must see the finished slab
    sharded_exchange(eng, rank, world, _allgather_for(group))
    torch.cuda.current_stream(g.device).synchronize()
    return idx


BUILD_MODES = ("replicated", "words")


def build_index_distributed(g, config, rank: int, world: int, mode: str = "replicated", group=None):
    """Label build on `world` ranks (one GPU each); every rank ends with the
    whole index.  mode "replicated" (default, no collective) or "words"
    (word-sharded + allgather); see the module docstring for the choice."""
    from .labels import build_index
    if mode not in BUILD_MODES:
        from .errors import ConfigError
        raise ConfigError(f"build mode must be one of {BUILD_MODES}, got {mode!r}")
    if mode == "replicated" or world == 1:
        return build_index(g, config)
    return sharded_build(g, config, rank, world, group)
