"""GPU tests for the §8(f) rows: snapshot I/O (byte-exact vs the reference's
own save_index output), the on-GPU verifier, and the estimator facade."""
from __future__ import annotations

import io

import numpy as np
import pytest

import paper_2101_09441_b200 as E
from conftest import golden
from oracle import oracle as O
from test_snapshot import CASES

pytestmark = pytest.mark.gpu

EXAMPLE_EDGES = [(0, 3), (1, 4), (1, 5), (2, 6), (3, 7), (4, 5), (5, 7), (5, 8), (6, 10), (7, 9), (8, 4), (8, 10)]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def gpu_index(d, name):
    spec = CASES[name]
    g = E.DynamicGraph.from_edges(int(d[f"{name}_n"]), d[f"{name}_src"], d[f"{name}_dst"])
    cfg = spec["cfg"]
    if "landmarks" in spec:
        leaves = E.select_leaves(g, 0, k_prime=cfg.k_prime, bucket_override=spec["ovr"])
        return g, E.build_index(g, cfg, landmarks=spec["landmarks"], leaf_sets=leaves)
    return g, E.build_index(g, cfg)


@pytest.mark.parametrize("name", list(CASES))
def test_save_matches_reference_bytes(name, tmp_path):
    d = golden("snapshots")
    g, idx = gpu_index(d, name)
    buf = io.BytesIO()
    E.save_index(idx, buf)
    assert buf.getvalue() == d[f"{name}_bytes"].tobytes()
    path = str(tmp_path / "idx.bin")
    E.save_index(idx, path)
    assert E.sniff_snapshot(path)


@pytest.mark.parametrize("name", list(CASES))
def test_load_reference_snapshot(name):
    d = golden("snapshots")
    g, idx = gpu_index(d, name)
    loaded = E.load_index(io.BytesIO(d[f"{name}_bytes"].tobytes()), g)
    assert loaded.labels_equal(idx)
    assert loaded.landmark_set == idx.landmark_set
    assert loaded.leaf_sets == idx.leaf_sets
    n = g.vertex_count
    qu = np.repeat(np.arange(n, dtype=np.uint32), n)
    qv = np.tile(np.arange(n, dtype=np.uint32), n)
    a, _ = E.query_batch(g, idx, (qu, qv))
    b, _ = E.query_batch(g, loaded, (qu, qv))
    np.testing.assert_array_equal(a.codes, b.codes)
    with pytest.raises(E.IndexGraphMismatchError):
        E.load_index(io.BytesIO(d[f"{name}_bytes"].tobytes()), E.DynamicGraph.from_edges(n + 1, [], []))


def test_verify_fresh_and_after_inserts():
    from paper_2101_09441_b200 import workload as W
    src, dst = W.gen_random_graph(50, 2, seed=17)
    g = E.DynamicGraph.from_edges(50, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=8, k_prime=8))
    assert E.verify_labels(g, idx).ok
    iu, iv = W.gen_insert_workload(src, dst, 50, 60, seed=18)
    for u, v in zip(iu.tolist(), iv.tolist()):
        E.insert_edge(g, idx, u, v)
    assert E.verify_labels(g, idx).ok
    assert E.verify_labels(g, idx, exhaustive=True).ok


def test_verify_corrupted_bit_one_violation():
    # tests/test_updates.py:337-344: drop v5's bit at the sink v10
    g = E.DynamicGraph.from_edges(11, [e[0] for e in EXAMPLE_EDGES], [e[1] for e in EXAMPLE_EDGES])
    leaves = E.select_leaves(g, 0, k_prime=2, bucket_override={0: 0, 9: 0, 1: 1, 2: 1, 10: 1})
    idx = E.build_index(g, E.IndexConfig(k=2, k_prime=2), landmarks=[4, 7], leaf_sets=leaves)
    w = {k: v.copy() for k, v in idx.export_words().items()}
    w["dl_in"][9, 0] &= ~np.uint64(1)
    idx.import_words(w)
    rep = E.verify_labels(g, idx, exhaustive=False)
    assert not rep.ok and len(rep.violations) == 1
    v = rep.violations[0]
    assert (v.vertex, v.family) == (9, "dl_in") and v.expected & ~v.actual == 1
    assert "missing bits [0]" in str(v)


def test_verify_exhaustive_catches_cycle_sustained_bits():
    # 0 -> 1 and a 2-cycle {2, 3} that still carries landmark 0's bit
    g = E.DynamicGraph.from_edges(4, [0, 2, 3], [1, 3, 2])
    idx = E.build_index(g, E.IndexConfig(k=1, k_prime=1), landmarks=[0])
    w = {k: v.copy() for k, v in idx.export_words().items()}
    w["dl_in"][2, 0] |= np.uint64(1)
    w["dl_in"][3, 0] |= np.uint64(1)
    idx.import_words(w)
    assert E.verify_labels(g, idx, exhaustive=False).ok        # the fixpoint check is blind to it
    rep = E.verify_labels(g, idx, exhaustive=True)
    assert not rep.ok and any(v.family == "dl_in" and v.vertex in (2, 3) for v in rep.violations)


def test_verify_large_random_fixpoint():
    from paper_2101_09441_b200 import workload as W
    s, d = W.rmat_edges(16, 8, 3)
    g = E.DynamicGraph.from_edges(1 << 16, s, d)
    idx = E.build_index(g, E.IndexConfig(k=128, k_prime=64))
    assert E.verify_labels(g, idx).ok
    iu, iv = W.gen_insert_workload(s, d, 1 << 16, 5000, seed=4)
    E.insert_edges(g, idx, iu, iv)
    assert E.verify_labels(g, idx, exhaustive=True).ok


# ------------------------------------------------------------- estimator --

def test_estimator_fit_predict():
    est = E.DblReachability(k=2, k_prime=2).fit(EXAMPLE_EDGES)
    assert est.predict([(0, 9), (3, 5), (2, 10)]) == [True, False, True]   # test_estimator.py:9-11
    assert est.predict_outcomes([(1, 9)])[0].answered_by.value == "DL_POSITIVE"
    assert set(est.index_.landmark_set.landmarks) == {5, 4}


def test_estimator_params_and_errors():
    assert E.DblReachability().fit([(0, 1), (1, 2)]).index_.config.k == 3
    with pytest.raises(E.NotFittedError):
        E.DblReachability().predict([(0, 1)])
    est = E.DblReachability(k=2, k_prime=2).fit([(0, 1)])
    with pytest.raises(E.VertexRangeError):
        est.predict([(0, 5)])
    with pytest.raises(ValueError):
        est.predict([(0, 1, 2)])
    est2 = E.DblReachability(k=8, seed=3)
    est2.set_params(k=16, workers=2)
    assert est2.k == 16 and est2.workers == 2 and "k=16" in repr(est2)
    with pytest.raises(ValueError):
        est2.set_params(nope=1)


def test_estimator_mutations_stay_truthful():
    from paper_2101_09441_b200 import workload as W
    s, d = W.gen_random_graph(30, 1.5, seed=23, acyclic=True)
    est = E.DblReachability(k=8, k_prime=8).fit(list(zip(s.tolist(), d.tolist())))
    est.insert_vertex(out_edges=[0, 5])
    est.insert_edge(2, 3)
    n = est.n_vertices_
    pairs = [(u, v) for u in range(n) for v in range(n)]
    src, dst = est.graph_.edge_arrays()
    og = O.OracleGraph(n, src, dst)
    truth = og.reach_batch([p[0] for p in pairs], [p[1] for p in pairs])
    assert est.predict(pairs) == truth.tolist()


@pytest.mark.parametrize("k", [128, 256])
def test_wide_records_roundtrip_and_verify(k):
    """Padded record strides (k = 128: 48 -> 64 B, k = 256: 80 -> 128 B):
    snapshot save/load (import into a fresh index), export/import, the
    exhaustive verifier (a fresh rebuild compared record by record, pad words
    included via labels_equal), and answers vs the oracle on the same labels."""
    from paper_2101_09441_b200 import workload as W
    s, d = W.rmat_edges(14, 8, 9)
    n = 1 << 14
    g = E.DynamicGraph.from_edges(n, s, d)
    idx = E.build_index(g, E.IndexConfig(k=k, k_prime=64))
    buf = io.BytesIO()
    E.save_index(idx, buf)
    loaded = E.load_index(io.BytesIO(buf.getvalue()), g)
    assert loaded.labels_equal(idx)
    assert E.verify_labels(g, idx, exhaustive=True).ok
    assert E.verify_labels(g, loaded, exhaustive=True).ok
    w = idx.export_words()
    other = E.rebuild_index(g, idx)
    other.import_words(w)
    assert other.labels_equal(idx)
    og = O.OracleGraph(n, s, d)
    oidx = og.build(k, 64, threads=8)
    for f in ("dl_in", "dl_out", "bl_in", "bl_out"):
        np.testing.assert_array_equal(w[f], getattr(oidx, f), err_msg=f)
    qu, qv = W.uniform_queries(n, 200_000, 11)
    out, _ = E.query_batch(g, loaded, (qu, qv))
    oc, ov = og.query_batch(oidx, qu, qv, threads=8)
    np.testing.assert_array_equal(out.codes, oc)
    np.testing.assert_array_equal(out.visited == 0, ov == 0)
