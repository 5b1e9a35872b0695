"""Index construction API (drop-in for the reference's labels.py).

Reference: labels.py:1-327.  Every computation runs on the GPU through the
C ABI: landmark ranking (K1), leaf selection + splitmix64 leaf hashing (K2)
and the bit-parallel label fixpoint (K3/K4, csrc/fixpoint.cu).  The
classes here only carry metadata and hand labels back to Python on demand.

Labels are the reference's exact reachability sets (labels.py:10-15), so a
build on the same graph with the same landmark/leaf metadata is bit-identical
to the reference's build_index.
"""
from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass, field
from enum import Enum
from typing import Mapping, Sequence

import numpy as np

from . import _native as N
from .errors import ConfigError, VertexRangeError
from .graph import DynamicGraph, as_device_graph


class LandmarkStrategy(str, Enum):
    """Degree heuristics for ranking landmark candidates (labels.py:31-46)."""

    MAX = "max"
    MIN = "min"
    SUM = "sum"
    PRODUCT = "product"

    def score(self, in_deg: int, out_deg: int) -> int:
        if self is LandmarkStrategy.MAX:
            return max(in_deg, out_deg)
        if self is LandmarkStrategy.MIN:
            return min(in_deg, out_deg)
        if self is LandmarkStrategy.SUM:
            return in_deg + out_deg
        return in_deg * out_deg


STRATEGY_CODE = {LandmarkStrategy.MAX: 0, LandmarkStrategy.MIN: 1, LandmarkStrategy.SUM: 2,
                 LandmarkStrategy.PRODUCT: 3}
CODE_STRATEGY = {v: k for k, v in STRATEGY_CODE.items()}


@dataclass(frozen=True)
class LandmarkSet:
    """Ordered landmarks; position i owns DL bit i (labels.py:54-74)."""

    landmarks: tuple[int, ...]
    position: Mapping[int, int] = field(repr=False)

    @classmethod
    def of(cls, landmarks: Sequence[int]) -> "LandmarkSet":
        seq = tuple(int(v) for v in landmarks)
        if len(set(seq)) != len(seq):
            raise ConfigError("landmark vertices must be distinct")
        return cls(seq, {v: i for i, v in enumerate(seq)})

    def __len__(self) -> int:
        return len(self.landmarks)

    def bit(self, v: int) -> int:
        i = self.position.get(v)
        return 0 if i is None else 1 << i


class LeafSets:
    """Source/sink leaves plus bucket assignment (labels.py:77-89).

    Stored as two per-vertex arrays (flags bit0 = leaves_in, bit1 =
    leaves_out; bucket); the frozenset/dict views of the reference are
    materialised lazily.
    """

    def __init__(self, leaves_in=None, leaves_out=None, bucket: Mapping[int, int] | None = None,
                 *, flags: np.ndarray | None = None, bucket_array: np.ndarray | None = None):
        if flags is not None:
            self.flags = np.ascontiguousarray(flags, dtype=np.uint8)
            self.bucket_array = np.ascontiguousarray(bucket_array, dtype=np.uint32)
        else:
            li = frozenset(int(v) for v in (leaves_in or ()))
            lo = frozenset(int(v) for v in (leaves_out or ()))
            bk = dict(bucket or {})
            n = 1 + max([*li, *lo, *bk.keys(), -1])
            self.flags = np.zeros(n, np.uint8)
            self.bucket_array = np.zeros(n, np.uint32)
            for v in li:
                self.flags[v] |= 1
            for v in lo:
                self.flags[v] |= 2
            for v, b in bk.items():
                self.bucket_array[v] = b
        self._cache = {}

    def for_vertex_count(self, n: int) -> tuple[np.ndarray, np.ndarray]:
        f = np.zeros(n, np.uint8)
        b = np.zeros(n, np.uint32)
        m = min(n, len(self.flags))
        f[:m] = self.flags[:m]
        b[:m] = self.bucket_array[:m]
        return f, b

    @property
    def leaves_in(self) -> frozenset:
        if "in" not in self._cache:
            self._cache["in"] = frozenset(np.flatnonzero(self.flags & 1).tolist())
        return self._cache["in"]

    @property
    def leaves_out(self) -> frozenset:
        if "out" not in self._cache:
            self._cache["out"] = frozenset(np.flatnonzero(self.flags & 2).tolist())
        return self._cache["out"]

    @property
    def bucket(self) -> Mapping[int, int]:
        if "bucket" not in self._cache:
            idx = np.flatnonzero(self.flags)
            self._cache["bucket"] = dict(zip(idx.tolist(), self.bucket_array[idx].tolist()))
        return self._cache["bucket"]

    def in_bit(self, v: int) -> int:
        return 1 << int(self.bucket_array[v]) if v < len(self.flags) and self.flags[v] & 1 else 0

    def out_bit(self, v: int) -> int:
        return 1 << int(self.bucket_array[v]) if v < len(self.flags) and self.flags[v] & 2 else 0

    def __eq__(self, other) -> bool:
        if not isinstance(other, LeafSets):
            return NotImplemented
        return (self.leaves_in == other.leaves_in and self.leaves_out == other.leaves_out
                and dict(self.bucket) == dict(other.bucket))

    def __repr__(self) -> str:
        return f"LeafSets(in={int((self.flags & 1).sum())}, out={int((self.flags & 2 > 0).sum())})"


@dataclass
class IndexConfig:
    """Build-time parameters (labels.py:92-116)."""

    k: int = 64
    k_prime: int = 64
    landmark_strategy: LandmarkStrategy = LandmarkStrategy.PRODUCT
    leaf_threshold: int = 0
    hash_seed: int = 0

    def validate(self, vertex_count: int) -> None:
        if self.k < 0:
            raise ConfigError(f"k must be >= 0, got {self.k}")
        if self.k > vertex_count:
            raise ConfigError(f"k={self.k} exceeds vertex count {vertex_count}")
        if self.k_prime < 1:
            raise ConfigError(f"k_prime must be >= 1, got {self.k_prime}")
        if self.leaf_threshold < 0:
            raise ConfigError(f"leaf_threshold must be >= 0, got {self.leaf_threshold}")
        if self.hash_seed < 0:
            raise ConfigError(f"hash_seed must be >= 0, got {self.hash_seed}")

    def to_c(self) -> N.Config:
        return N.Config(self.k, self.k_prime, STRATEGY_CODE[LandmarkStrategy(self.landmark_strategy)],
                        self.leaf_threshold, self.hash_seed & 0xFFFFFFFFFFFFFFFF)


def _words_to_ints(a: np.ndarray) -> list[int]:
    """(n, w) u64 words (LSW first) -> Python ints (the reference's masks)."""
    if a.shape[1] == 0:
        return [0] * a.shape[0]
    if a.shape[1] == 1:
        return a[:, 0].tolist()
    out = []
    for row in a.tolist():
        x = 0
        for j, w in enumerate(row):
            x |= w << (64 * j)
        out.append(x)
    return out


class DblIndex:
    """Device-resident DL/BL labels plus frozen metadata (labels.py:184-244).

    Labels live on the GPU as one AoS record per vertex
    {dl_in | bl_in | dl_out | bl_out}; the reference-shaped attributes
    (``dl_in`` etc., lists of Python ints) are exported on access.
    """

    def __init__(self, handle, graph: DynamicGraph, config: IndexConfig):
        self._h = handle
        self.config = config
        self.device = graph.device
        self._n = graph.vertex_count
        self._graph_ref = weakref.ref(graph)
        self._meta = None
        self._labels = None
        self.version = 0
        weakref.finalize(self, N.lib().dbl_index_free, handle)

    @property
    def handle(self):
        return self._h

    @property
    def vertex_count(self) -> int:
        return self._n

    @property
    def wdl(self) -> int:
        return (self.config.k + 63) // 64

    @property
    def wbl(self) -> int:
        return (self.config.k_prime + 63) // 64

    def _invalidate(self) -> None:
        self._labels = None
        self.version += 1

    def _metadata(self):
        if self._meta is None:
            lm = np.zeros(max(self.config.k, 1), np.uint32)
            fl = np.zeros(self._n, np.uint8)
            bk = np.zeros(self._n, np.uint32)
            N.call("dbl_index_metadata", self._h, N.ptr(lm), N.ptr(fl), N.ptr(bk))
            self._meta = (LandmarkSet.of(lm[:self.config.k].tolist()),
                          LeafSets(flags=fl, bucket_array=bk))
        return self._meta

    @property
    def landmark_set(self) -> LandmarkSet:
        return self._metadata()[0]

    @property
    def leaf_sets(self) -> LeafSets:
        return self._metadata()[1]

    def export_words(self) -> dict[str, np.ndarray]:
        """Labels as (n, words) u64 arrays, LSW first, per family."""
        if self._labels is None:
            n, wdl, wbl = self._n, self.wdl, self.wbl
            out = {"dl_in": np.zeros((n, wdl), np.uint64), "dl_out": np.zeros((n, wdl), np.uint64),
                   "bl_in": np.zeros((n, wbl), np.uint64), "bl_out": np.zeros((n, wbl), np.uint64)}
            N.call("dbl_index_export", self._h, N.ptr(out["dl_in"]), N.ptr(out["dl_out"]),
                   N.ptr(out["bl_in"]), N.ptr(out["bl_out"]))
            self._labels = out
        return self._labels

    def import_words(self, words: Mapping[str, np.ndarray]) -> None:
        arrs = [np.ascontiguousarray(words[f], dtype=np.uint64) for f in ("dl_in", "dl_out", "bl_in", "bl_out")]
        N.call("dbl_index_import", self._h, *[N.ptr(a) for a in arrs])
        self._invalidate()

    def _family(self, fam: str) -> "_LabelList":
        return _LabelList(self, fam, _words_to_ints(self.export_words()[fam]))

    def _write_family(self, fam: str, values: Sequence[int]) -> None:
        """Write one family's labels (ints, LSW first) back to the device."""
        w = self.wdl if fam.startswith("dl") else self.wbl
        arr = np.zeros((self._n, w), np.uint64)
        mask = (1 << 64) - 1
        for x, val in enumerate(values):
            for k in range(w):
                arr[x, k] = (int(val) >> (64 * k)) & mask
        ptrs = [N.ptr(arr) if f == fam else None for f in ("dl_in", "dl_out", "bl_in", "bl_out")]
        N.call("dbl_index_import", self._h, *ptrs)
        self._invalidate()

    @property
    def dl_in(self) -> "_LabelList":
        return self._family("dl_in")

    @property
    def dl_out(self) -> "_LabelList":
        return self._family("dl_out")

    @property
    def bl_in(self) -> "_LabelList":
        return self._family("bl_in")

    @property
    def bl_out(self) -> "_LabelList":
        return self._family("bl_out")

    def _check_vertex(self, v: int) -> None:
        if not 0 <= v < self._n:
            raise VertexRangeError(f"vertex {v} outside [0, {self._n})")

    def grow_to(self, vertex_count: int) -> None:
        """Extend label storage; new vertices start with empty labels (labels.py:209-216)."""
        if vertex_count < self._n:
            raise ConfigError("index cannot shrink")
        N.call("dbl_index_grow", self._h, vertex_count)
        self._n = vertex_count
        self._meta = None
        self._invalidate()

    def labels_equal(self, other: "DblIndex") -> bool:
        """Bit-identical label comparison on the device (labels.py:238-244)."""
        eq = ctypes.c_int()
        N.call("dbl_index_equal", self._h, other._h, ctypes.byref(eq))
        return bool(eq.value)

    def digest(self, g=None, *, with_state: bool = False):
        """The query digest (u32 per vertex, dbl_index_digest), recomputed if stale;
        with_state=True also returns whether it was current before the call."""
        g = g if g is not None else self._graph_ref()
        if g is None:
            raise ValueError("the index's graph is gone: pass it explicitly")
        out = np.zeros(max(self._n, 1), np.uint32)
        cur = ctypes.c_int()
        N.call("dbl_index_digest", self._h, g.handle, N.ptr(out), ctypes.byref(cur))
        return (out[:self._n], bool(cur.value)) if with_state else out[:self._n]

    def records(self) -> tuple[int, int]:
        """(device pointer, words per record) of the AoS label table."""
        p = ctypes.c_void_p()
        w = ctypes.c_uint32()
        N.call("dbl_index_records", self._h, ctypes.byref(p), ctypes.byref(w))
        return int(p.value or 0), int(w.value)

    def __repr__(self) -> str:
        return f"DblIndex(n={self._n}, k={self.config.k}, k_prime={self.config.k_prime})"


class _LabelList(list):
    """One label family as ints, one per vertex (labels.py:194-207).  Item
    assignment writes the family back to the device, so code that edits a
    label in place (`idx.dl_in[x] &= ~1`, as the reference's tests do to
    forge or drop a bit) changes the index the engine uses."""

    def __init__(self, idx: "DblIndex", fam: str, values: list[int]):
        super().__init__(values)
        self._idx, self._fam = idx, fam

    def __setitem__(self, i, value):
        super().__setitem__(i, value)
        self._idx._write_family(self._fam, self)


def leaf_hash(v: int, k_prime: int, seed: int = 0, *, device: int = 0) -> int:
    """Bucket of a leaf vertex: splitmix64 mix mod k' (labels.py:119-137), on the GPU."""
    return int(leaf_hash_batch([v], k_prime, seed, device=device)[0])


def leaf_hash_batch(ids, k_prime: int, seed: int = 0, *, device: int = 0) -> np.ndarray:
    if k_prime < 1:
        raise ConfigError(f"k_prime must be >= 1, got {k_prime}")
    a = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64))
    out = np.zeros(len(a), np.uint32)
    N.call("dbl_leaf_hash", N.ptr(a), len(a), k_prime, seed & 0xFFFFFFFFFFFFFFFF, N.ptr(out), device)
    return out


def select_landmarks(g, k: int, strategy: LandmarkStrategy = LandmarkStrategy.PRODUCT) -> LandmarkSet:
    """Top-k vertices by strategy score, ties to the smaller id (labels.py:140-147)."""
    g = as_device_graph(g)
    if k < 0 or k > g.vertex_count:
        raise ConfigError(f"k={k} outside [0, {g.vertex_count}]")
    out = np.zeros(max(k, 1), np.uint32)
    N.call("dbl_select_landmarks", g.handle, k, STRATEGY_CODE[LandmarkStrategy(strategy)], N.ptr(out))
    return LandmarkSet.of(out[:k].tolist())


def _override_arrays(bucket_override):
    if not bucket_override:
        return None, None, 0
    ids = np.array(list(bucket_override.keys()), dtype=np.int64)
    bks = np.array(list(bucket_override.values()), dtype=np.int64)
    keep = (ids >= 0) & (ids < 2**32)
    ids, bks = ids[keep], bks[keep]
    if len(bks) and (bks.min() < 0 or bks.max() >= 2**32):
        bks = np.clip(bks, 0, 2**32 - 2)  # out of range either way: the device rejects it
    return (np.ascontiguousarray(ids.astype(np.uint32)), np.ascontiguousarray(bks.astype(np.uint32)),
            len(ids))


def select_leaves(g, threshold: int = 0, *, k_prime: int = 64, hash_seed: int = 0,
                  bucket_override: Mapping[int, int] | None = None) -> LeafSets:
    """Zero in/out-degree leaves (+ M(v) <= r) with buckets (labels.py:150-181)."""
    g = as_device_graph(g)
    if threshold < 0:
        raise ConfigError(f"threshold must be >= 0, got {threshold}")
    if k_prime < 1:
        raise ConfigError(f"k_prime must be >= 1, got {k_prime}")
    # the reference rejects an out-of-range override only for leaves
    # (labels.py:167-171); the device kernel applies the same rule
    ids, bks, cnt = _override_arrays(bucket_override)
    n = g.vertex_count
    flags = np.zeros(n, np.uint8)
    bucket = np.zeros(n, np.uint32)
    N.call("dbl_select_leaves", g.handle, threshold, k_prime, hash_seed & 0xFFFFFFFFFFFFFFFF,
           N.ptr(ids), N.ptr(bks), cnt, N.ptr(flags), N.ptr(bucket))
    return LeafSets(flags=flags, bucket_array=bucket)


def build_index(g, config: IndexConfig | None = None, *, landmarks: Sequence[int] | None = None,
                leaf_sets: LeafSets | None = None, bucket_override: Mapping[int, int] | None = None
                ) -> DblIndex:
    """Construct the four label families from scratch (labels.py:263-306)."""
    g = as_device_graph(g)
    cfg = config if config is not None else IndexConfig()
    cfg.validate(g.vertex_count)
    lm = None
    if landmarks is not None:
        if len(landmarks) != cfg.k:
            raise ConfigError(f"{len(landmarks)} landmarks given but k={cfg.k}")
        for v in landmarks:
            g._check_vertex(int(v))
        LandmarkSet.of(landmarks)
        lm = N.u32_array(list(landmarks)) if cfg.k else None
    fl = bk = None
    if leaf_sets is not None:
        if not isinstance(leaf_sets, LeafSets):
            leaf_sets = LeafSets(leaf_sets.leaves_in, leaf_sets.leaves_out, leaf_sets.bucket)
        fl, bk = leaf_sets.for_vertex_count(g.vertex_count)
    ids, bks, cnt = _override_arrays(bucket_override)
    h = ctypes.c_void_p()
    N.call("dbl_index_build", g.handle, ctypes.byref(cfg.to_c()), N.ptr(lm), N.ptr(fl), N.ptr(bk),
           N.ptr(ids), N.ptr(bks), cnt, ctypes.byref(h))
    return DblIndex(h, g, IndexConfig(cfg.k, cfg.k_prime, LandmarkStrategy(cfg.landmark_strategy),
                                      cfg.leaf_threshold, cfg.hash_seed))


def rebuild_index(g, idx: DblIndex) -> DblIndex:
    """Fresh build reusing idx's frozen landmark/leaf metadata (labels.py:309-312)."""
    g = as_device_graph(g)
    ls, leaves = idx._metadata()
    return build_index(g, idx.config, landmarks=ls.landmarks, leaf_sets=leaves)


def rebuild_in_place(g, idx: DblIndex) -> DblIndex:
    """rebuild_index into idx's own device storage (no new allocation)."""
    g = as_device_graph(g)
    N.call("dbl_index_rebuild", g.handle, idx.handle)
    idx._invalidate()
    return idx


def _label_tests(idx: DblIndex, x, y):
    a, b = N.u32_array(x), N.u32_array(y)
    dl = np.zeros(len(a), np.uint8)
    bl = np.zeros(len(a), np.uint8)
    N.call("dbl_label_tests", idx.handle, N.ptr(a), N.ptr(b), len(a), N.ptr(dl), N.ptr(bl))
    return dl.astype(bool), bl.astype(bool)


def dl_intersec(idx: DblIndex, x: int, y: int) -> bool:
    """True iff some landmark is reached by x and reaches y (labels.py:315-319)."""
    idx._check_vertex(x)
    idx._check_vertex(y)
    return bool(_label_tests(idx, [x], [y])[0][0])


def bl_contain(idx: DblIndex, x: int, y: int) -> bool:
    """Leaf-label containment; False proves x cannot reach y (labels.py:322-327)."""
    idx._check_vertex(x)
    idx._check_vertex(y)
    return bool(_label_tests(idx, [x], [y])[1][0])
