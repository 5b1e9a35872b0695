"""Single-edge insert_edge fast path (csrc/insert_one.cu) against the oracle.

The fast path answers a call with one kernel and one host sync: pre-check,
add_edge into the graph's pending-edge log, and both propagations as a
discovery BFS + one write pass.  Every case here checks the reference's exact
UpdateStats per edge (updates.py:112-137) and the labels afterwards, and the
pending log's visibility to every other graph operation (queries, batch
inserts, has_edge, degrees, exports) and its fold into the delta adjacency.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu

FAMS = ("dl_in", "dl_out", "bl_in", "bl_out")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def labels_match(idx, oidx):
    w = idx.export_words()
    return all(np.array_equal(w[f], getattr(oidx, f)) for f in FAMS)


def run_sequence(n, src, dst, iu, iv, k=64, kp=64, query_every=0, seed=0):
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=k, k_prime=kp))
    og = O.OracleGraph(n, src, dst)
    oidx = og.build(k, kp, threads=2)
    assert labels_match(idx, oidx)
    rng = np.random.default_rng(seed)
    for j, (u, v) in enumerate(zip(iu.tolist(), iv.tolist())):
        st = E.insert_edge(g, idx, u, v)
        ost = og.insert_edge(oidx, u, v)
        assert (st.visited, st.labels_changed, st.early_terminated) == ost, (j, u, v)
        if query_every and (j + 1) % query_every == 0:
            # queries see the logged edges (the log is folded in first)
            qu = rng.integers(0, n, 3000, dtype=np.uint32)
            qv = rng.integers(0, n, 3000, dtype=np.uint32)
            out, _ = E.query_batch(g, idx, (qu, qv))
            oc, _ = og.query_batch(oidx, qu, qv, threads=2)
            np.testing.assert_array_equal(out.codes, oc)
    assert g.edge_count == og.edge_count
    assert labels_match(idx, oidx)
    assert idx.labels_equal(E.rebuild_index(g, idx))
    return g, idx, og, oidx


@pytest.mark.parametrize("k,kp", [(64, 64), (256, 64), (0, 200)])
def test_rmat_sequence_with_queries(k, kp):
    n = 1 << 12
    src, dst = W.rmat_edges(12, 4, seed=31)
    iu, iv = W.gen_insert_workload(src, dst, n, 400, seed=32)
    run_sequence(n, src, dst, iu, iv, k=k, kp=kp, query_every=50)


def test_pending_log_overflow_and_repeats():
    """More single inserts than the log holds (1024): folds mid-sequence;
    repeated edges (present, logged or folded) insert nothing."""
    n = 1 << 11
    src, dst = W.rmat_edges(11, 2, seed=33)
    iu, iv = W.gen_insert_workload(src, dst, n, 1300, seed=34)
    iu = np.concatenate([iu, iu[:40], src[:20]])
    iv = np.concatenate([iv, iv[:40], dst[:20]])
    g, idx, og, oidx = run_sequence(n, src, dst, iu, iv, k=100, kp=13)
    assert g.has_edges(iu, iv).all()


def test_large_cone_falls_back_to_batch_fixpoint():
    """A cone larger than the CTA's tables (a 20k-vertex chain) takes the
    batch fixpoint; stats and labels still equal the reference's."""
    n = 20_002
    chain = np.arange(20_000, dtype=np.uint32)
    src, dst = chain[:-1], chain[1:]
    # u = 20000 (isolated: both leaf sets) -> head 0: the whole chain lacks u's bits
    iu = np.array([20_000, 19_999, 20_001, 5], np.uint32)
    iv = np.array([0, 20_001, 3, 20_000], np.uint32)
    run_sequence(n, src, dst, iu, iv, k=4, kp=64)


def test_pending_edges_visible_to_graph_ops():
    n = 64
    src = np.arange(0, 30, dtype=np.uint32)
    dst = src + 1
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=4, k_prime=8))
    m0 = g.edge_count
    st = E.insert_edge(g, idx, 40, 41)
    assert g.edge_count == m0 + 1
    assert g.has_edge(40, 41) and not g.has_edge(41, 40)
    indeg, outdeg = g.degrees()
    assert outdeg[40] == 1 and indeg[41] == 1
    # a query whose only path uses logged edges
    E.insert_edge(g, idx, 41, 50)
    o = E.query(g, idx, 40, 50)
    assert o.reachable
    # a batch insert after logged single inserts, then more single inserts
    E.insert_edges(g, idx, np.array([50, 51], np.uint32), np.array([51, 52], np.uint32))
    E.insert_edge(g, idx, 52, 0)
    assert E.query(g, idx, 40, 30).reachable
    assert g.edge_count == m0 + 5
    ptr, col = g.adjacency(False)
    assert ptr[-1] == g.edge_count
    og = O.OracleGraph(n, src, dst)
    oidx = og.build(4, 8, landmarks=idx.landmark_set.landmarks, leaf_flags=idx.leaf_sets.flags,
                    bucket=idx.leaf_sets.bucket_array)
    for u, v in ((40, 41), (41, 50), (50, 51), (51, 52), (52, 0)):
        og.insert_edge(oidx, u, v)
    assert labels_match(idx, oidx)
    assert st.early_terminated is False


# ------------------------------------------------------- batched insertion --

def _batch_vs_oracle(n, src, dst, iu, iv, k=64, kp=64):
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=k, k_prime=kp))
    og = O.OracleGraph(n, src, dst)
    oidx = og.build(k, kp, threads=2)
    st = E.insert_edges(g, idx, iu, iv)
    for u, v in zip(iu.tolist(), iv.tolist()):
        og.insert_edge(oidx, u, v)
    assert g.edge_count == og.edge_count
    assert labels_match(idx, oidx)
    assert idx.labels_equal(E.rebuild_index(g, idx))
    return g, idx, st


def test_batch_prep_duplicates_and_skew():
    """Batched insertion on batches with heavy duplication (6000 copies of one
    edge), on a batch of edges all leaving one hub, tiny batches and batches
    of already-present edges."""
    n = 1 << 12
    src, dst = W.rmat_edges(12, 4, seed=51)
    rng = np.random.default_rng(52)
    # 6000 copies of one edge + 2000 random ones
    iu = np.concatenate([np.full(6000, 7, np.uint32), rng.integers(0, n, 2000, dtype=np.uint32)])
    iv = np.concatenate([np.full(6000, 4000, np.uint32), rng.integers(0, n, 2000, dtype=np.uint32)])
    _, _, st = _batch_vs_oracle(n, src, dst, iu, iv)
    assert st.requested == 8000
    # 3000 edges from one hub
    hv = rng.permutation(n)[:3000].astype(np.uint32)
    _batch_vs_oracle(n, src, dst, np.full(3000, 1, np.uint32), hv)
    # tiny batches, and a batch that repeats already-present edges
    _batch_vs_oracle(n, src, dst, np.array([5], np.uint32), np.array([9], np.uint32))
    _batch_vs_oracle(n, src, dst, src[:500].copy(), dst[:500].copy())


def test_batch_prep_range_error_is_a_noop():
    n = 1 << 10
    src, dst = W.rmat_edges(10, 4, seed=53)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g)
    before = idx.export_words()
    m0 = g.edge_count
    iu = np.array([1, 2, 3, n], np.uint32)
    iv = np.array([4, 5, 6, 7], np.uint32)
    with pytest.raises(E.VertexRangeError):
        E.insert_edges(g, idx, iu, iv)
    assert g.edge_count == m0
    after = idx.export_words()
    assert all(np.array_equal(before[f], after[f]) for f in FAMS)
