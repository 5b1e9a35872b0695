"""Batched reach(u, v) queries (drop-in for the reference's queries.py).

Reference: queries.py:1-267.  query_batch runs the label-check kernel K6
(rules 0-4 on every pair, one thread per query) and the batched pruned-BFS
kernel K7 for the rest (csrc/query.cu); answers and provenance codes equal
the reference's for every pair.  `visited` is 0 exactly for label-answered
queries, as in the reference; for BFS answers it counts the frontier
expansions of that query in the bit-parallel BFS, which is not the
reference's FIFO dequeue count (SURVEY.md §4 excludes those counts from the
parity contract).
"""
from __future__ import annotations

import ctypes
import os
import threading
import itertools
import time
from dataclasses import dataclass
from enum import Enum
from typing import Iterable, Sequence

import numpy as np

from . import _native as N
from .errors import ConfigError, IndexGraphMismatchError, VertexRangeError
from .graph import as_device_graph
from .labels import DblIndex

WORKERS_ENV_VAR = "DBLREACH_WORKERS"


class AnsweredBy(str, Enum):
    """Provenance codes in the reference's _ANSWER_ORDER (queries.py:40-47, 188-189)."""

    REFLEXIVE = "REFLEXIVE"
    DL_POSITIVE = "DL_POSITIVE"
    BL_NEGATIVE = "BL_NEGATIVE"
    THM1_NEGATIVE = "THM1_NEGATIVE"
    THM2_NEGATIVE = "THM2_NEGATIVE"
    BFS_POSITIVE = "BFS_POSITIVE"
    BFS_NEGATIVE = "BFS_NEGATIVE"


ANSWER_ORDER = tuple(AnsweredBy)
REACHABLE_CODES = (0, 1, 5)
_REACHABLE_LUT = np.zeros(256, bool)
_REACHABLE_LUT[list(REACHABLE_CODES)] = True


@dataclass(frozen=True)
class QueryOutcome:
    """Answer plus provenance; visited is 0 iff label-answered (queries.py:50-56)."""

    reachable: bool
    answered_by: AnsweredBy
    visited: int = 0


@dataclass(frozen=True)
class QueryFlags:
    """Rule toggles (queries.py:59-75)."""

    use_dl: bool = True
    use_bl: bool = True
    use_thm1: bool = True
    use_thm2: bool = True
    prune_dl: bool = True
    prune_bl: bool = True

    def bits(self) -> int:
        return (int(self.use_dl) | int(self.use_bl) << 1 | int(self.use_thm1) << 2
                | int(self.use_thm2) << 3 | int(self.prune_dl) << 4 | int(self.prune_bl) << 5)


DEFAULT_FLAGS = QueryFlags()
DL_ONLY = QueryFlags(use_bl=False)
BL_ONLY = QueryFlags(use_dl=False)


class Outcomes(Sequence):
    """Sequence of QueryOutcome backed by the device's code/visited arrays.

    Behaves like the reference's list[QueryOutcome] (indexing, iteration,
    equality with a list) without materialising 10^6 dataclasses.
    """

    def __init__(self, codes: np.ndarray, visited: np.ndarray):
        self.codes = codes
        self.visited = visited

    @property
    def reachable(self) -> np.ndarray:
        return _REACHABLE_LUT[self.codes]

    def __len__(self) -> int:
        return len(self.codes)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return Outcomes(self.codes[i], self.visited[i])
        c = int(self.codes[i])
        return QueryOutcome(c in REACHABLE_CODES, ANSWER_ORDER[c], int(self.visited[i]))

    def __eq__(self, other) -> bool:
        if isinstance(other, Outcomes):
            return (np.array_equal(self.codes, other.codes)
                    and np.array_equal(self.visited, other.visited))
        if isinstance(other, (list, tuple)):
            return len(other) == len(self) and all(a == b for a, b in zip(self, other))
        return NotImplemented

    def __repr__(self) -> str:
        return f"Outcomes(n={len(self)})"


@dataclass(frozen=True)
class BatchStats:
    """Aggregates over one query batch; times are milliseconds (queries.py:145-166)."""

    query_count: int
    label_answered: int
    rho: float
    visited_total: int
    reachable_count: int
    elapsed_ms: float

    @classmethod
    def collect(cls, outcomes, elapsed_ms: float) -> "BatchStats":
        if isinstance(outcomes, Outcomes):
            q = len(outcomes)
            c = outcomes.codes
            # visited == 0 exactly for the label-answered codes 0..4, and the
            # reachable codes are 0, 1, 5 (queries.py:50-56): counted on the
            # u8 codes instead of materialising boolean arrays; the u32 visited
            # counts sum in numpy's native u64 accumulator (an explicit
            # dtype= casts every element: 1.7x slower)
            la = int(np.count_nonzero(c < 5))
            reach = int(np.count_nonzero(c <= 1)) + int(np.count_nonzero(c == 5))
            vt = int(outcomes.visited.sum()) if la < q else 0
            return cls(q, la, la / q if q else 0.0, vt, reach, elapsed_ms)
        label_answered = sum(1 for o in outcomes if o.visited == 0)
        return cls(len(outcomes), label_answered,
                   label_answered / len(outcomes) if outcomes else 0.0,
                   sum(o.visited for o in outcomes), sum(1 for o in outcomes if o.reachable),
                   elapsed_ms)


def default_workers() -> int:
    """Worker count from DBLREACH_WORKERS, else the processor count (queries.py:199-207).

    Accepted for API compatibility: the GPU engine ignores it.
    """
    value = os.environ.get(WORKERS_ENV_VAR)
    if value:
        try:
            return max(1, int(value))
        except ValueError:
            raise ConfigError(f"{WORKERS_ENV_VAR} must be an integer, got {value!r}") from None
    return os.cpu_count() or 1


def _check_consistent(g, idx: DblIndex) -> None:
    if g.vertex_count != idx.vertex_count:
        raise IndexGraphMismatchError(
            f"graph has {g.vertex_count} vertices but index has {idx.vertex_count}")


def _is_column(x) -> bool:
    return isinstance(x, np.ndarray) or (hasattr(x, "is_cuda") and hasattr(x, "numel"))


def _pair_list_to_array(ql) -> np.ndarray:
    # a list of 2-tuples of Python ints flattens ~2.4x faster through fromiter than
    # through np.array's nested-sequence discovery (100k pairs: 6.9 vs 16.7 ms);
    # anything else (ragged, non-integer, nested arrays) takes np.array and its errors
    if not ql:
        return np.zeros((0, 2), np.int64)
    if type(ql[0]) is tuple:
        try:
            if set(map(len, ql)) != {2}:
                raise ValueError
            return np.fromiter(itertools.chain.from_iterable(ql), dtype=np.int64,
                               count=2 * len(ql)).reshape(-1, 2)
        except (TypeError, ValueError, OverflowError):
            pass
    return np.array(ql, dtype=np.int64).reshape(-1, 2)


def _pairs_to_arrays(queries) -> tuple[np.ndarray, np.ndarray]:
    # the column form (u_array, v_array) only for a 2-tuple of 1-D arrays /
    # tensors of equal length; any other iterable is a sequence of (u, v)
    # pairs as in the reference (so ((0, 5), (3, 7)) is the pairs (0,5), (3,7))
    if isinstance(queries, tuple) and len(queries) == 2 and _is_column(queries[0]) \
            and _is_column(queries[1]) and np.ndim(queries[0]) == 1 and np.ndim(queries[1]) == 1 \
            and len(queries[0]) == len(queries[1]):
        u, v = queries
        if hasattr(u, "is_cuda"):
            u, v = u.cpu().numpy(), v.cpu().numpy()
        return N.u32_array(u), N.u32_array(v)
    if isinstance(queries, np.ndarray):
        a = queries.reshape(-1, 2)
    else:
        ql = list(queries)
        a = _pair_list_to_array(ql)
    if a.size and (a.min() < 0 or a.max() >= 2**32):
        raise VertexRangeError("query vertex outside the uint32 range")
    return np.ascontiguousarray(a[:, 0], dtype=np.uint32), np.ascontiguousarray(a[:, 1], dtype=np.uint32)


def query_codes(g, idx: DblIndex, u, v, flags: QueryFlags = DEFAULT_FLAGS,
                with_visited: bool = True):
    """Array API: AnsweredBy codes (u8) and visited counts (u32) for pairs u[i], v[i].

    u/v may be host arrays (numpy) or CUDA tensors on the index's device; the
    results live where the inputs live.
    """
    g = as_device_graph(g)
    _check_consistent(g, idx)
    if (hasattr(u, "is_cuda") and u.is_cuda) or (hasattr(v, "is_cuda") and v.is_cuda):
        import torch
        N.check_device_ids(u, v, g.device)
        codes = torch.empty(u.numel(), dtype=torch.uint8, device=u.device)
        vis = torch.empty(u.numel(), dtype=torch.int32, device=u.device) if with_visited else None
        N.device_inputs_ready(u, v)
        N.call("dbl_query", idx.handle, g.handle, N.ptr(u), N.ptr(v), u.numel(), flags.bits(),
               N.ptr(codes), N.ptr(vis), N.MEM_DEVICE)
        return codes, vis
    a, b = N.u32_array(u), N.u32_array(v)
    if a.ndim != 1 or b.ndim != 1 or len(a) != len(b):
        raise ValueError(f"u and v must be 1-D and of equal length ({a.shape} vs {b.shape})")
    codes = np.zeros(len(a), np.uint8)
    vis = np.zeros(len(a), np.uint32) if with_visited else None
    N.call("dbl_query", idx.handle, g.handle, N.ptr(a), N.ptr(b), len(a), flags.bits(), N.ptr(codes),
           N.ptr(vis), N.MEM_HOST)
    return codes, vis


_ONE = threading.local()
_DEFAULT_BITS = DEFAULT_FLAGS.bits()
# outcomes are immutable: one shared instance per label-answered code
_LABEL_OUTCOMES = tuple(QueryOutcome(c in REACHABLE_CODES, ANSWER_ORDER[c], 0) for c in range(len(ANSWER_ORDER)))


def query(g, idx: DblIndex, u: int, v: int, flags: QueryFlags = DEFAULT_FLAGS) -> QueryOutcome:
    """Answer q(u, v) (queries.py:94-142) through the per-call service
    (dbl_query_one: no kernel launch per call)."""
    g = as_device_graph(g)
    _check_consistent(g, idx)
    g._check_vertex(u)
    g._check_vertex(v)
    out = getattr(_ONE, "out", None)
    if out is None:   # per-thread result words (code, visited)
        out = _ONE.out = (ctypes.c_uint32 * 2)()
    fb = _DEFAULT_BITS if flags is DEFAULT_FLAGS else flags.bits()
    st = _query_one()(idx.handle, g.handle, u, v, fb, out)
    if st:
        N.check(st)
    c, vis = out[0], out[1]
    if vis == 0:   # label-answered (BFS answers expand at least the source)
        return _LABEL_OUTCOMES[c]
    return QueryOutcome(c in REACHABLE_CODES, ANSWER_ORDER[c], vis)


_QUERY_ONE = None


def _query_one():
    global _QUERY_ONE
    if _QUERY_ONE is None:
        _QUERY_ONE = N.lib().dbl_query_one
    return _QUERY_ONE


def query_batch(g, idx: DblIndex, queries: Iterable[tuple[int, int]], workers: int = 1,
                flags: QueryFlags = DEFAULT_FLAGS) -> tuple[Outcomes, BatchStats]:
    """Evaluate many queries in input order (queries.py:210-249).

    `queries` is any iterable of (u, v) pairs, an (q, 2) array, or a (u, v)
    tuple of arrays.  `workers` is validated as in the reference and
    otherwise ignored: the batch is one GPU launch sequence.
    """
    if workers < 1:
        raise ConfigError(f"workers must be >= 1, got {workers}")
    g = as_device_graph(g)
    _check_consistent(g, idx)
    u, v = _pairs_to_arrays(queries)
    started = time.perf_counter()
    codes, vis = query_codes(g, idx, u, v, flags)
    elapsed_ms = (time.perf_counter() - started) * 1000.0
    out = Outcomes(codes, vis)
    return out, BatchStats.collect(out, elapsed_ms)


def explain(outcome: QueryOutcome) -> str:
    """One-line provenance string (queries.py:252-267)."""
    by = outcome.answered_by
    if by is AnsweredBy.REFLEXIVE:
        return "answered positive: self-query, reachability is reflexive"
    if by is AnsweredBy.DL_POSITIVE:
        return "answered positive by DL label intersection"
    if by is AnsweredBy.BL_NEGATIVE:
        return "answered negative by BL label containment failure"
    if by is AnsweredBy.THM1_NEGATIVE:
        return "answered negative by reverse DL intersection early termination"
    if by is AnsweredBy.THM2_NEGATIVE:
        return "answered negative by landmark coverage early termination"
    if by is AnsweredBy.BFS_POSITIVE:
        return f"answered positive by pruned BFS, visited {outcome.visited} vertices"
    return f"answered negative by exhausted pruned BFS, visited {outcome.visited} vertices"
