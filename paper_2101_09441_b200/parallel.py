"""Multi-GPU label build: record words sharded across ranks + NCCL allgather.

SURVEY.md §8(e): each 64-bit word of a label record ({dl_in | bl_in | dl_out
| bl_out}, csrc/internal.cuh) is an independent least fixpoint, so ranks
build disjoint word sets of the same record table (every rank holds the
replicated graph and the frozen metadata, which are deterministic), pack
their words into a word-major slab, allgather the slabs, and scatter the
peers' words back into their own AoS table (K5 interleave).  Queries and
insertions need no collective: query batches are split per rank and every
rank applies the same insertion batch to its replica.

The orchestration is written against a small engine interface so that the
host logic is tested on CPU with gloo (tests/test_parallel.py) and runs on
GPUs with the C ABI + NCCL.
"""
from __future__ import annotations

import ctypes
from typing import Callable, Protocol, Sequence

import numpy as np


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


def sharded_build(g, config, rank: int, world: int, group=None):
    """build_index across `world` GPUs (one rank per GPU, NCCL process group)."""
    import torch.distributed as dist
    idx = create_index(g, config)
    eng = DeviceWordEngine(g, idx)

    def allgather(out, inp):
        dist.all_gather_into_tensor(out, inp, group=group)

    sharded_exchange(eng, rank, world, allgather)
    return idx
