"""Incremental edge insertion (drop-in for the insertion half of updates.py).

Reference: updates.py:31-50 (UpdateStats), 89-137 (_propagate_union,
insert_edge), 255-271 (insert_vertex).  Deletion (updates.py:140-252) is
experimental and cyclic-unsafe in the reference and is out of scope
(SURVEY.md §2 row 3b).

insert_edge keeps the reference's exact UpdateStats: the pre-check runs on
pre-insertion labels, and because labels are exact reachability closures the
set of vertices whose label grows is order-independent, so labels_changed
and visited (= 1 + changed non-seed vertices per direction) match the
reference bit-for-bit.

insert_edges applies a whole batch with one device fixpoint (K8): new edges
seed the in-half at their heads and the out-half at their tails, and the
shared frontier kernel propagates only from vertices whose labels grew.  The
final labels equal the sequential insert_edge loop and rebuild_index
(least fixpoint); see BatchUpdateStats for how its counters differ.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable

import numpy as np

from . import _native as N
from .graph import as_device_graph, sync_reference_graph
from .labels import DblIndex
from .queries import _check_consistent


@dataclass
class UpdateStats:
    """Work accounting for one maintenance operation (updates.py:31-50)."""

    visited: int = 0
    labels_changed: int = 0
    early_terminated: bool = False
    tainted: bool = False

    def absorb(self, other: "UpdateStats") -> None:
        self.visited += other.visited
        self.labels_changed += other.labels_changed
        self.tainted = self.tainted or other.tainted


@dataclass
class BatchUpdateStats:
    """Counters of one batched insertion.

    certified: edges whose *pre-batch* DL labels already proved u -> v (the
    reference's per-edge pre-check evaluates on labels that include earlier
    edges of the sequence, so its count can be larger).
    labels_changed: distinct (vertex, direction) pairs whose label grew over
    the whole batch (the sequential loop counts a vertex once per edge).
    """

    requested: int = 0
    inserted: int = 0
    certified: int = 0
    labels_changed: int = 0
    levels: int = 0
    delta_merged: bool = False
    fix_items: int = 0     # delta fixpoint: frontier items expanded (work counter)
    fix_edges: int = 0     # delta fixpoint: edges relaxed (work counter)


def insert_edge(g, idx: DblIndex, u: int, v: int) -> UpdateStats:
    """Insert (u, v) and repair all four label families (updates.py:112-137)."""
    orig, g = g, as_device_graph(g)
    _check_consistent(g, idx)
    g._check_vertex(u)
    g._check_vertex(v)
    st = N.UpdateStatsC()
    N.check(N.lib().dbl_insert_edge(idx.handle, g.handle, u, v, ctypes.byref(st)))
    g._m_dev += int(st.inserted)   # add_edge's return (the C side counts it the same way)
    g.version += 1
    idx._invalidate()
    sync_reference_graph(orig, g, ((u, v),))
    return UpdateStats(int(st.visited), int(st.labels_changed), bool(st.early_terminated))


def insert_edges(g, idx: DblIndex, u, v) -> BatchUpdateStats:
    """Insert a batch of edges with one device fixpoint (K8).

    u/v are host arrays or CUDA tensors (device pointers) of equal length.
    """
    orig, g = g, as_device_graph(g)
    _check_consistent(g, idx)
    st = N.BatchStatsC()
    if (hasattr(u, "is_cuda") and u.is_cuda) or (hasattr(v, "is_cuda") and v.is_cuda):
        N.check_device_ids(u, v, g.device)
        N.device_inputs_ready(u, v)
        N.call("dbl_insert_edges", idx.handle, g.handle, N.ptr(u), N.ptr(v), u.numel(), N.MEM_DEVICE,
               ctypes.byref(st))
    else:
        a, b = N.u32_array(u), N.u32_array(v)
        if len(a) != len(b):
            raise ValueError("u and v differ in length")
        N.call("dbl_insert_edges", idx.handle, g.handle, N.ptr(a), N.ptr(b), len(a), N.MEM_HOST,
               ctypes.byref(st))
    g._refresh_count()
    g.version += 1
    idx._invalidate()
    if orig is not g:
        hu = u.cpu().numpy() if hasattr(u, "cpu") else np.asarray(u)
        hv = v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)
        sync_reference_graph(orig, g, zip(hu.tolist(), hv.tolist()))
    return BatchUpdateStats(int(st.requested), int(st.inserted), int(st.certified),
                            int(st.labels_changed), int(st.levels), bool(st.delta_merged),
                            int(st.fix_items), int(st.fix_edges))


def insert_vertex(g, idx: DblIndex, out_edges: Iterable[int] = (),
                  in_edges: Iterable[int] = ()) -> UpdateStats:
    """Add a vertex with empty labels and wire its edges (updates.py:255-271)."""
    orig, g = g, as_device_graph(g)
    _check_consistent(g, idx)
    vid = g.add_vertex()
    idx.grow_to(g.vertex_count)
    stats = UpdateStats()
    outs, ins = list(out_edges), list(in_edges)
    for w in outs:
        stats.absorb(insert_edge(g, idx, vid, w))
    for w in ins:
        stats.absorb(insert_edge(g, idx, w, vid))
    sync_reference_graph(orig, g, [(vid, w) for w in outs] + [(w, vid) for w in ins], new_vertices=1)
    return stats
