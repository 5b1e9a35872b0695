"""Device-resident directed graph with the reference DynamicGraph's surface.

Reference: graph.py:31-145 (DynamicGraph).  The adjacency lives in HBM as a
CSR (out-edges) plus a CSC (in-edges), built and deduplicated on the GPU by
dbl_graph_create (K0, csrc/graph.cu); later insertions go to a sorted delta
CSR/CSC that every traversal reads alongside the base.

Edges added before the graph is first used on the device are buffered on
the host (with the reference's duplicate check, graph.py:60-61) and
uploaded in one batch; afterwards every add_edge goes straight to the device.
"""
from __future__ import annotations

import ctypes
import weakref
from typing import Iterator

import numpy as np

from . import _native as N
from .errors import VertexRangeError


class DynamicGraph:
    """Directed graph on one GPU; ids are dense ints 0..n-1 (graph.py:31-46)."""

    def __init__(self, vertex_count: int = 0, *, device: int = 0):
        if vertex_count < 0:
            raise VertexRangeError("vertex_count must be >= 0")
        self._n = int(vertex_count)
        self.device = int(device)
        self._h = None
        self._pending: dict[tuple[int, int], None] = {}
        self._m_dev = 0
        self.version = 0
        self.original_ids: list[int] | None = None
        self._dense_of: dict[int, int] | None = None

    # -- construction -----------------------------------------------------
    @classmethod
    def from_edges(cls, n: int, src, dst, *, device: int = 0) -> "DynamicGraph":
        """Bulk constructor: upload an edge list and build CSR/CSC on device.

        src/dst may be host arrays or CUDA tensors (uint32 ids, any 32-bit dtype).
        """
        g = cls(n, device=device)
        if (hasattr(src, "is_cuda") and src.is_cuda) or (hasattr(dst, "is_cuda") and dst.is_cuda):
            N.check_device_ids(src, dst, src.device.index if hasattr(src, "device") else device)
            h = ctypes.c_void_p()
            N.device_inputs_ready(src, dst)
            N.call("dbl_graph_create", n, N.ptr(src), N.ptr(dst), src.numel(), N.MEM_DEVICE, src.device.index,
                   ctypes.byref(h))
            g._h = h
            g.device = src.device.index
            g._refresh_count()
            weakref.finalize(g, N.lib().dbl_graph_free, h)
            return g
        s = N.u32_array(src)
        d = N.u32_array(dst)
        if len(s) != len(d):
            raise ValueError("src and dst differ in length")
        g._create(s, d)
        return g

    def _create(self, s: np.ndarray, d: np.ndarray) -> None:
        h = ctypes.c_void_p()
        N.call("dbl_graph_create", self._n, N.ptr(s), N.ptr(d), len(s), N.MEM_HOST, self.device,
               ctypes.byref(h))
        self._h = h
        self._refresh_count()
        weakref.finalize(self, N.lib().dbl_graph_free, h)

    @property
    def handle(self) -> ctypes.c_void_p:
        """The device graph (materialises buffered edges on first use)."""
        if self._h is None:
            if self._pending:
                e = np.array(list(self._pending), dtype=np.uint32).reshape(-1, 2)
                s, d = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
            else:
                s = d = np.zeros(0, np.uint32)
            self._pending = {}
            self._create(s, d)
        return self._h

    def _refresh_count(self) -> None:
        n = ctypes.c_uint32()
        m = ctypes.c_uint64()
        N.call("dbl_graph_info", self._h, ctypes.byref(n), ctypes.byref(m))
        self._m_dev = int(m.value)

    # -- reference surface ------------------------------------------------
    @property
    def vertex_count(self) -> int:
        return self._n

    @property
    def edge_count(self) -> int:
        return self._m_dev if self._h is not None else len(self._pending)

    def _check_vertex(self, v: int) -> None:
        if not 0 <= v < self._n:
            raise VertexRangeError(f"vertex {v} outside [0, {self._n})")

    def add_vertex(self) -> int:
        if self._h is not None:
            N.call("dbl_graph_add_vertices", self._h, 1)
        self._n += 1
        self.version += 1
        return self._n - 1

    def add_vertices(self, count: int) -> range:
        if count and self._h is not None:
            N.call("dbl_graph_add_vertices", self._h, count)
        first = self._n
        self._n += count
        self.version += 1
        return range(first, self._n)

    def add_edge(self, u: int, v: int) -> bool:
        """Insert edge (u, v); False if it was already present (graph.py:56-66)."""
        self._check_vertex(u)
        self._check_vertex(v)
        if self._h is None:
            if (u, v) in self._pending:
                return False
            self._pending[(u, v)] = None
            self.version += 1
            return True
        return self.add_edges([u], [v]) == 1

    def add_edges(self, src, dst) -> int:
        """Batch add_edge; returns how many distinct new edges were added."""
        s = N.u32_array(src)
        d = N.u32_array(dst)
        if len(s) != len(d):
            raise ValueError("src and dst differ in length")
        if not len(s):
            return 0
        if s.max() >= self._n or d.max() >= self._n:
            bad = int(s.max() if s.max() >= self._n else d.max())
            raise VertexRangeError(f"vertex {bad} outside [0, {self._n})")
        if self._h is None:
            before = len(self._pending)
            for a, b in zip(s.tolist(), d.tolist()):
                self._pending[(a, b)] = None
            self.version += 1
            return len(self._pending) - before
        out = ctypes.c_uint64()
        N.call("dbl_graph_add_edges", self.handle, N.ptr(s), N.ptr(d), len(s), ctypes.byref(out))
        self._refresh_count()
        self.version += 1
        return int(out.value)

    def has_edge(self, u: int, v: int) -> bool:
        if self._h is None:
            return (u, v) in self._pending
        return bool(self.has_edges([u], [v])[0])

    def has_edges(self, u, v) -> np.ndarray:
        a, b = N.u32_array(u), N.u32_array(v)
        out = np.zeros(len(a), np.uint8)
        N.call("dbl_graph_has_edges", self.handle, N.ptr(a), N.ptr(b), len(a), N.ptr(out))
        return out.astype(bool)

    def degrees(self) -> tuple[np.ndarray, np.ndarray]:
        """(in_degree[n], out_degree[n]) computed on the device."""
        ind = np.zeros(self._n, np.uint32)
        outd = np.zeros(self._n, np.uint32)
        N.call("dbl_graph_degrees", self.handle, N.ptr(ind), N.ptr(outd))
        return ind, outd

    def out_degree(self, u: int) -> int:
        self._check_vertex(u)
        return int(self.degrees()[1][u])

    def in_degree(self, v: int) -> int:
        self._check_vertex(v)
        return int(self.degrees()[0][v])

    def edge_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        """All edges as (src, dst) arrays sorted by (src, dst)."""
        h = self.handle
        m = self.edge_count
        s = np.zeros(m, np.uint32)
        d = np.zeros(m, np.uint32)
        if m:
            N.call("dbl_graph_edges", h, N.ptr(s), N.ptr(d))
        return s, d

    def adjacency(self, reverse: bool = False) -> tuple[np.ndarray, np.ndarray]:
        """(ptr u32[n+1], col u32[m]) of the out-edges (or in-edges if reverse)."""
        h = self.handle
        ptr = np.zeros(self._n + 1, np.uint32)
        col = np.zeros(max(self.edge_count, 1), np.uint32)
        N.call("dbl_graph_adjacency", h, int(reverse), N.ptr(ptr), N.ptr(col))
        return ptr, col[:self.edge_count]

    def edges(self) -> Iterator[tuple[int, int]]:
        s, d = self.edge_arrays()
        return iter(zip(s.tolist(), d.tolist()))

    def successors(self, u: int) -> list[int]:
        self._check_vertex(u)
        s, d = self.edge_arrays()
        return d[s == u].tolist()

    def predecessors(self, v: int) -> list[int]:
        self._check_vertex(v)
        s, d = self.edge_arrays()
        return s[d == v].tolist()

    def vertices(self) -> range:
        return range(self._n)

    def _lists(self, reverse: bool) -> list[list[int]]:
        key = (self._n, self.edge_count, self.version, reverse)
        cache = getattr(self, "_list_cache", None)
        if cache is not None and cache[0] == key:
            return cache[1]
        if self._h is None:
            lists: list[list[int]] = [[] for _ in range(self._n)]
            for u, v in self._pending:
                (lists[v] if reverse else lists[u]).append(u if reverse else v)
        else:
            ptr, col = self.adjacency(reverse)
            cl = col.tolist()
            p = ptr.tolist()
            lists = [cl[p[i]:p[i + 1]] for i in range(self._n)]
        self._list_cache = (key, lists)
        return lists

    @property
    def forward(self) -> list[list[int]]:
        """Out-adjacency lists (graph.py:36), a read-only host copy sorted by id
        (the reference keeps insertion order; reachability is the same)."""
        return self._lists(False)

    @property
    def reverse(self) -> list[list[int]]:
        """In-adjacency lists (graph.py:37), read-only host copy."""
        return self._lists(True)

    def to_original(self, dense: int) -> int:
        self._check_vertex(dense)
        return self.original_ids[dense] if self.original_ids else dense

    def to_dense(self, original: int) -> int:
        """Dense id of an original id (graph.py:126-133)."""
        if self._dense_of is None:
            self._check_vertex(original)
            return original
        try:
            return self._dense_of[original]
        except KeyError:
            raise VertexRangeError(f"unknown original vertex id {original}") from None

    def register_original(self, original: int) -> int:
        """Map an original id to a dense id, creating a vertex if unseen (graph.py:135-145)."""
        if self._dense_of is None:
            self._dense_of = {self.to_original(v): v for v in self.vertices()}
            self.original_ids = [self.to_original(v) for v in self.vertices()]
        dense = self._dense_of.get(original)
        if dense is None:
            dense = self.add_vertex()
            self._dense_of[original] = dense
            self.original_ids.append(original)
        return dense

    def __repr__(self) -> str:
        return f"DynamicGraph(n={self._n}, m={self.edge_count}, device={self.device})"


def load_edge_list(source, gzipped: bool | None = None, *, device: int = 0) -> DynamicGraph:
    """Parse "src dst" lines into a device graph with densely remapped ids
    (graph.py:174-210): '#' lines are comments, duplicates collapse, dense
    ids follow first appearance (src before dst on a line), original ids are
    kept on the side table.  The edges go to the device in one upload.
    """
    import gzip
    import io
    from .errors import EdgeListFormatError
    if isinstance(source, str):
        if gzipped or (gzipped is None and source.endswith(".gz")):
            stream = io.TextIOWrapper(gzip.open(source, "rb"), encoding="utf-8")
        else:
            stream = open(source, "r", encoding="utf-8")
    elif isinstance(source, bytes):
        raw = gzip.decompress(source) if (gzipped or (gzipped is None and source[:2] == b"\x1f\x8b")) else source
        stream = io.StringIO(raw.decode("utf-8"))
    elif hasattr(source, "read") and isinstance(source.read(0), bytes):
        # binary stream (graph.py:162-169): gzip by flag or magic bytes
        if gzipped is None and hasattr(source, "peek"):
            gzipped = source.peek(2)[:2] == b"\x1f\x8b"
        stream = io.TextIOWrapper(gzip.GzipFile(fileobj=source) if gzipped else source, encoding="utf-8")
    else:
        stream = source
    flat: list[int] = []
    with stream:
        for line_no, line in enumerate(stream, start=1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            if len(parts) != 2:
                raise EdgeListFormatError(line_no, f"expected 'src dst', got {line!r}")
            try:
                raw_u, raw_v = int(parts[0]), int(parts[1])
            except ValueError:
                raise EdgeListFormatError(line_no, f"non-integer vertex id in {line!r}") from None
            if raw_u < 0 or raw_v < 0:
                raise EdgeListFormatError(line_no, f"negative vertex id in {line!r}")
            flat.append(raw_u)
            flat.append(raw_v)
    a = np.array(flat, dtype=np.int64)
    uniq, first, inv = np.unique(a, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")          # originals in first-appearance order
    rank = np.empty(len(uniq), np.int64)
    rank[order] = np.arange(len(uniq))
    dense = rank[inv].astype(np.uint32)
    g = DynamicGraph.from_edges(len(uniq), dense[0::2], dense[1::2], device=device)
    g.original_ids = uniq[order].tolist()
    g._dense_of = {o: i for i, o in enumerate(g.original_ids)}
    return g


_converted: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def as_device_graph(g, device: int = 0) -> DynamicGraph:
    """Accept this package's graph or any reference-style graph object.

    A reference dblreach.DynamicGraph (forward adjacency lists, graph.py:36)
    is uploaded once and cached per (object, device) until its vertex or edge
    count -- or its `version` attribute, if it has one -- changes.  The
    reference graph carries no mutation counter, so a remove_edge followed by
    an add_edge on the reference object itself keeps both counts and the
    cached copy would be stale: call forget_device_graph(g) after mutating a
    reference graph directly (edges inserted through this package's
    insert_edge / insert_edges go to the cached device copy and stay
    consistent with the index).
    """
    if isinstance(g, DynamicGraph):
        return g
    if hasattr(g, "forward") and hasattr(g, "vertex_count"):
        key = (g.vertex_count, getattr(g, "edge_count", None), getattr(g, "version", None), device)
        try:
            cached = _converted.get(g)
        except TypeError:
            cached = None
        if cached is not None and cached[0] == key:
            return cached[1]
        src = np.fromiter((u for u, succ in enumerate(g.forward) for _ in succ), np.uint32)
        dst = np.fromiter((v for succ in g.forward for v in succ), np.uint32)
        dg = DynamicGraph.from_edges(g.vertex_count, src, dst, device=device)
        try:
            _converted[g] = (key, dg)
        except TypeError:
            pass
        return dg
    raise TypeError(f"expected a DynamicGraph, got {type(g)!r}")


def sync_reference_graph(orig, dg: DynamicGraph, pairs=(), new_vertices: int = 0) -> None:
    """Mirror an engine-side mutation into the reference DynamicGraph the caller
    passed (insert_edge adds its edge to g, updates.py:124; insert_vertex adds
    the vertex, :255-271), and re-key the cached device copy so it is kept."""
    if isinstance(orig, DynamicGraph) or not hasattr(orig, "add_edge"):
        return
    for _ in range(new_vertices):
        orig.add_vertex()
    for u, v in pairs:
        orig.add_edge(int(u), int(v))
    key = (orig.vertex_count, getattr(orig, "edge_count", None), getattr(orig, "version", None), dg.device)
    try:
        _converted[orig] = (key, dg)
    except TypeError:
        pass


def forget_device_graph(g) -> None:
    """Drop the cached device copy of a reference graph (re-uploaded on next use)."""
    try:
        _converted.pop(g, None)
    except TypeError:
        pass
