"""GPU parity: the CUDA engine (through the C ABI) against the golden vectors
and the CPU oracle.  Bit-exact for labels, metadata and answer codes.

Golden fixtures come from the reference itself (oracle/gen_golden.py); larger
cases compare with the oracle restatement (oracle/dbl_oracle.c), which
tests/test_oracle.py pins to the same fixtures.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu

FAMS = ("dl_in", "dl_out", "bl_in", "bl_out")
FLAGSETS = {
    "default": E.QueryFlags(),
    "dl_only": E.QueryFlags(use_bl=False),
    "bl_only": E.QueryFlags(use_dl=False),
    "no_early": E.QueryFlags(use_thm1=False, use_thm2=False),
    "no_prune": E.QueryFlags(prune_dl=False, prune_bl=False),
    "bare": E.QueryFlags(use_thm1=False, use_thm2=False, prune_dl=False, prune_bl=False),
}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def graph_of(d, p=""):
    return E.DynamicGraph.from_edges(int(d[p + "n"]), d[p + "src"], d[p + "dst"])


def assert_labels(idx, d, p=""):
    w = idx.export_words()
    for f in FAMS:
        np.testing.assert_array_equal(w[f], d[p + f], err_msg=f)


def assert_labels_equal_oracle(idx, oidx):
    w = idx.export_words()
    for f in FAMS:
        np.testing.assert_array_equal(w[f], getattr(oidx, f), err_msg=f)


def assert_meta(idx, d, p=""):
    assert idx.landmark_set.landmarks == tuple(d[p + "landmarks"].tolist())
    np.testing.assert_array_equal(idx.leaf_sets.flags, d[p + "leaf_flags"])
    m = d[p + "leaf_flags"] != 0
    np.testing.assert_array_equal(idx.leaf_sets.bucket_array[m], d[p + "bucket"][m])


def toy_index(d):
    g = graph_of(d)
    ovr = {0: 0, 9: 0, 1: 1, 2: 1, 10: 1}   # EXAMPLE_BUCKETS, pkg/tests/conftest.py:23
    leaves = E.select_leaves(g, 0, k_prime=2, bucket_override=ovr)
    idx = E.build_index(g, E.IndexConfig(k=2, k_prime=2), landmarks=[4, 7], leaf_sets=leaves)
    return g, idx


# ------------------------------------------------------------------ toy --

def test_toy_tables(toy_golden):
    d = toy_golden
    g, idx = toy_index(d)
    assert_labels(idx, d)
    for f in FAMS:
        np.testing.assert_array_equal(idx.export_words()[f][:, 0], d["exp_" + f])
    auto = E.build_index(g, E.IndexConfig(k=3, k_prime=4))
    assert_meta(auto, d, "auto_")
    assert_labels(auto, d, "auto_")


def test_toy_queries_all_flagsets(toy_golden):
    d = toy_golden
    g, idx = toy_index(d)
    for name, fl in FLAGSETS.items():
        out, stats = E.query_batch(g, idx, (d["qu"], d["qv"]), flags=fl)
        np.testing.assert_array_equal(out.codes, d[f"codes_{name}"], err_msg=name)
        bfs = np.isin(out.codes, (5, 6))
        np.testing.assert_array_equal(out.visited == 0, ~bfs)
        assert stats.label_answered == int((~bfs).sum())


def test_toy_single_queries(toy_golden):
    d = toy_golden
    g, idx = toy_index(d)
    # tests/test_queries.py:12-47 outcomes
    assert E.query(g, idx, 0, 9) == E.QueryOutcome(True, E.AnsweredBy.DL_POSITIVE, 0)
    assert E.query(g, idx, 3, 5).answered_by is E.AnsweredBy.BL_NEGATIVE
    o = E.query(g, idx, 2, 10)
    assert o.reachable and o.answered_by is E.AnsweredBy.BFS_POSITIVE and o.visited >= 1
    assert E.query(g, idx, 6, 6) == E.QueryOutcome(True, E.AnsweredBy.REFLEXIVE, 0)
    assert E.query(g, idx, 9, 7).answered_by is E.AnsweredBy.THM1_NEGATIVE
    assert E.query(g, idx, 4, 3, E.QueryFlags(use_bl=False)).answered_by is E.AnsweredBy.THM2_NEGATIVE
    out, st = E.query_batch(g, idx, [(0, 9), (3, 5), (2, 10)])
    assert [o.answered_by for o in out] == [E.AnsweredBy.DL_POSITIVE, E.AnsweredBy.BL_NEGATIVE,
                                            E.AnsweredBy.BFS_POSITIVE]
    assert st.rho == pytest.approx(2 / 3)


def test_toy_insertion_example(toy_golden):
    d = toy_golden
    g, idx = toy_index(d)
    st = E.insert_edge(g, idx, *map(int, d["ins_uv"]))
    exp = d["ins_stats"]
    assert (st.visited, st.labels_changed, st.early_terminated) == (int(exp[0]), int(exp[1]), bool(exp[2]))
    assert_labels(idx, d, "ins_")
    assert idx.labels_equal(E.rebuild_index(g, idx))
    g2, idx2 = toy_index(d)
    st2 = E.insert_edge(g2, idx2, *map(int, d["ins2_uv"]))
    assert st2.early_terminated and st2.visited == 0 and st2.labels_changed == 0
    assert g2.has_edge(*map(int, d["ins2_uv"]))
    # re-inserting a present edge changes nothing (tests/test_updates.py:58-65)
    m = g2.edge_count
    E.insert_edge(g2, idx2, 2, 6)
    assert g2.edge_count == m


def test_toy_errors(toy_golden):
    d = toy_golden
    g, idx = toy_index(d)
    with pytest.raises(E.VertexRangeError):
        E.query(g, idx, 0, 11)
    with pytest.raises(E.VertexRangeError):
        E.query_batch(g, idx, [(0, 1), (12, 3)])
    with pytest.raises(E.ConfigError):
        E.query_batch(g, idx, [(0, 1)], workers=0)
    with pytest.raises(E.ConfigError):
        E.build_index(g, E.IndexConfig(k=12))
    with pytest.raises(E.ConfigError):
        E.build_index(g, E.IndexConfig(k=3, k_prime=2), landmarks=[4, 5])
    with pytest.raises(E.ConfigError):
        E.select_leaves(g, 0, k_prime=2, bucket_override={0: 5})
    with pytest.raises(E.VertexRangeError):
        E.insert_edge(g, idx, 0, 99)
    g.add_vertex()
    with pytest.raises(E.IndexGraphMismatchError):
        E.query(g, idx, 0, 1)


def test_leaf_hash_kats():
    d = np.load(__import__("conftest").GOLDEN + "/leaf_hash.npz")
    for j, kp in enumerate(d["kprimes"]):
        for s, sd in enumerate(d["seeds"]):
            got = E.leaf_hash_batch(d["ids"], int(kp), int(sd))
            np.testing.assert_array_equal(got, d["buckets"][:, j, s])
    assert E.leaf_hash(1, 64, 0) == 47 and E.leaf_hash(12345, 64, 7) == 5


def test_landmark_and_leaf_kats():
    d = np.load(__import__("conftest").GOLDEN + "/landmarks.npz")
    for ci in range(4):
        g = E.DynamicGraph.from_edges(int(d[f"c{ci}_n"]), d[f"c{ci}_src"], d[f"c{ci}_dst"])
        for s in E.LandmarkStrategy:
            exp = d[f"c{ci}_{s.value}"]
            assert E.select_landmarks(g, len(exp), s).landmarks == tuple(exp.tolist())
        for thr in (0, 2, 6):
            ls = E.select_leaves(g, thr, k_prime=13, hash_seed=5)
            np.testing.assert_array_equal(ls.flags, d[f"c{ci}_leaf_flags_t{thr}"])
            m = ls.flags != 0
            np.testing.assert_array_equal(ls.bucket_array[m], d[f"c{ci}_bucket_t{thr}"][m])


# --------------------------------------------------------------- family --

def test_family_build_and_all_pairs(family_golden):
    d = family_golden
    bits = {"default": FLAGSETS["default"], "bl_only": FLAGSETS["bl_only"], "bare": FLAGSETS["bare"]}
    for i in range(int(d["count"])):
        p = f"f{i}_"
        g = graph_of(d, p)
        k = int(d[p + "k"])
        idx = E.build_index(g, E.IndexConfig(k=k, k_prime=k))
        assert_meta(idx, d, p)
        assert_labels(idx, d, p)
        n = int(d[p + "n"])
        qu = np.repeat(np.arange(n, dtype=np.uint32), n)
        qv = np.tile(np.arange(n, dtype=np.uint32), n)
        for name, fl in bits.items():
            out, _ = E.query_batch(g, idx, (qu, qv), flags=fl)
            np.testing.assert_array_equal(out.codes, d[p + f"codes_{name}"], err_msg=f"{i} {name}")
            np.testing.assert_array_equal(out.visited == 0, d[p + f"visited_{name}"] == 0)


def test_family_insert_sequence_exact_stats(family_golden):
    d = family_golden
    for i in range(int(d["count"])):
        p = f"f{i}_"
        g = graph_of(d, p)
        k = int(d[p + "k"])
        idx = E.build_index(g, E.IndexConfig(k=k, k_prime=k))
        for j, (u, v) in enumerate(zip(d[p + "ins_u"], d[p + "ins_v"])):
            st = E.insert_edge(g, idx, int(u), int(v))
            e = d[p + "ins_stats"][j]
            assert (st.visited, st.labels_changed, st.early_terminated) == \
                (int(e[0]), int(e[1]), bool(e[2])), (i, j)
        assert_labels(idx, d, p + "after_")
        assert idx.labels_equal(E.rebuild_index(g, idx))


def test_family_insert_batched(family_golden):
    d = family_golden
    for i in range(int(d["count"])):
        p = f"f{i}_"
        g = graph_of(d, p)
        k = int(d[p + "k"])
        idx = E.build_index(g, E.IndexConfig(k=k, k_prime=k))
        st = E.insert_edges(g, idx, d[p + "ins_u"], d[p + "ins_v"])
        assert st.inserted == len(d[p + "ins_u"])
        assert_labels(idx, d, p + "after_")


# ----------------------------------------------------------------- cfg1 --

def test_cfg1_build_query_insert(cfg1_golden):
    d = cfg1_golden
    src, dst = W.gen_random_graph(10_000, 5, seed=1)
    g = E.DynamicGraph.from_edges(10_000, src, dst)
    assert g.edge_count == 50_000
    idx = E.build_index(g)
    assert_meta(idx, d)
    assert_labels(idx, d)
    out, st = E.query_batch(g, idx, (d["qu"], d["qv"]))
    np.testing.assert_array_equal(out.codes, d["codes"])
    assert st.rho == pytest.approx(float(np.mean(d["visited"] == 0)))
    # batched insertion of the same 1000 edges == sequential reference result
    g2 = E.DynamicGraph.from_edges(10_000, src, dst)
    idx2 = E.build_index(g2)
    E.insert_edges(g2, idx2, d["ins_u"], d["ins_v"])
    assert_labels(idx2, d, "after_")
    # sequential exact stats on the first 200
    for j in range(200):
        s1 = E.insert_edge(g, idx, int(d["ins_u"][j]), int(d["ins_v"][j]))
        e = d["ins_stats"][j]
        assert (s1.visited, s1.labels_changed, s1.early_terminated) == (int(e[0]), int(e[1]), bool(e[2])), j


# ---------------------------------------------------- R-MAT vs the oracle --

def rmat_case(scale, ef, seed):
    src, dst = W.rmat_edges(scale, ef, seed)
    n = 1 << scale
    return n, src, dst


@pytest.mark.parametrize("scale,ef", [(12, 8), (16, 8), (16, 2)])
def test_rmat_build_and_queries_vs_oracle(scale, ef):
    n, src, dst = rmat_case(scale, ef, 7)
    g = E.DynamicGraph.from_edges(n, src, dst)
    og = O.OracleGraph(n, src, dst)
    assert g.edge_count == og.edge_count
    idx = E.build_index(g)
    oidx = og.build(64, 64, threads=8)
    np.testing.assert_array_equal(np.array(idx.landmark_set.landmarks), oidx.landmarks)
    np.testing.assert_array_equal(idx.leaf_sets.flags, oidx.leaf_flags)
    assert_labels_equal_oracle(idx, oidx)
    qu, qv = W.uniform_queries(n, 100_000, 3)
    pu, pv = W.positive_queries(n, src, dst, 50_000, 4)
    qu, qv = np.concatenate([qu, pu]), np.concatenate([qv, pv])
    for fl in (E.QueryFlags(), E.QueryFlags(use_dl=False), E.QueryFlags(prune_dl=False, prune_bl=False)):
        out, _ = E.query_batch(g, idx, (qu, qv), flags=fl)
        oc, ov = og.query_batch(oidx, qu, qv, fl.bits(), threads=8)
        np.testing.assert_array_equal(out.codes, oc)
        np.testing.assert_array_equal(out.visited == 0, ov == 0)


@pytest.mark.parametrize("k", [64, 256])
def test_large_graph_build_paths_vs_oracle(k):
    """2^21 vertices: the build paths that only large graphs take -- the
    has-predecessor bitmaps and sparse later pivot sweeps (n >= 2^21), the
    stand-alone record-apply kernel (records >= 256 MB at k = 256: 32-byte
    stores) -- against the oracle's labels, and against a rebuild (frozen
    metadata: dense sweeps, no prep degrees)."""
    n, src, dst = rmat_case(21, 4, 21)
    g = E.DynamicGraph.from_edges(n, src, dst)
    og = O.OracleGraph(n, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=k, k_prime=64))
    oidx = og.build(k, 64, threads=16)
    np.testing.assert_array_equal(np.array(idx.landmark_set.landmarks), oidx.landmarks)
    assert_labels_equal_oracle(idx, oidx)
    assert idx.labels_equal(E.rebuild_index(g, idx))


def test_rmat_insert_batches_vs_rebuild():
    n, src, dst = rmat_case(16, 8, 11)
    g = E.DynamicGraph.from_edges(n, src, dst)
    og = O.OracleGraph(n, src, dst)
    idx = E.build_index(g)
    oidx = og.build(64, 64, threads=8)
    prev = None
    for b in range(3):
        iu, iv = W.gen_insert_workload(src, dst, n, 2000, 100 + b, exclude=prev)
        prev = (iu, iv) if prev is None else (np.concatenate([prev[0], iu]), np.concatenate([prev[1], iv]))
        st = E.insert_edges(g, idx, iu, iv)
        assert st.inserted == 2000
        for u, v in zip(iu.tolist(), iv.tolist()):
            og.insert_edge(oidx, u, v)
        assert g.edge_count == og.edge_count
        assert_labels_equal_oracle(idx, oidx)
        assert idx.labels_equal(E.rebuild_index(g, idx))
    qu, qv = W.uniform_queries(n, 100_000, 9)
    out, _ = E.query_batch(g, idx, (qu, qv))
    oc, _ = og.query_batch(oidx, qu, qv, threads=8)
    np.testing.assert_array_equal(out.codes, oc)


@pytest.mark.parametrize("k", [64, 256])
def test_pivot_prune_after_growth(k):
    """The BFS prunes D(h) on one bitmap bit for queries whose dl_out[u] holds
    a landmark of the pivot's SCC.  After vertex growth and edge inserts the
    stored D(h) is a stale subset (and shorter than n): answers must still
    equal the reference BFS (queries.py:116-142) run on the same labels."""
    n, src, dst = rmat_case(13, 8, 21)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=k, k_prime=64))
    lm = list(idx.landmark_set.landmarks)
    rng = np.random.default_rng(3)
    new = []
    for j in range(24):   # new vertices wired into and out of the hub core
        outs = [int(lm[j % len(lm)])] if j % 3 else []
        ins = [int(x) for x in rng.integers(0, n, 2)] + ([int(new[-1])] if new else [])
        E.insert_vertex(g, idx, out_edges=outs, in_edges=ins)
        new.append(g.vertex_count - 1)
    iu, iv = W.gen_insert_workload(src, dst, n, 3000, 17)
    E.insert_edges(g, idx, iu, iv)
    assert idx.labels_equal(E.rebuild_index(g, idx))
    nn = g.vertex_count
    qu, qv = W.uniform_queries(nn, 60_000, 5)
    qu[:2000] = rng.choice(new, 2000)
    qv[2000:4000] = rng.choice(new, 2000)
    w = idx.export_words()
    ptr, col = g.adjacency(False)
    for fl in (E.QueryFlags(), E.QueryFlags(use_bl=False), E.QueryFlags(prune_bl=False)):
        out, _ = E.query_batch(g, idx, (qu, qv), flags=fl)
        oc = O.csr_query_batch(nn, ptr.astype(np.uint64), col, k, 64, w, qu, qv, fl.bits(), threads=8)
        np.testing.assert_array_equal(out.codes, oc)
    assert np.mean(out.codes >= 5) > 0   # the BFS ran


def test_dense_bfs_fallback_path():
    # k = 0 and a single bucket: many BFS queries explore cones larger than the
    # shared-memory table, exercising the dense re-run path.
    src, dst = W.gen_random_graph(6000, 1.3, seed=5, acyclic=True)
    g = E.DynamicGraph.from_edges(6000, src, dst)
    og = O.OracleGraph(6000, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=0, k_prime=1))
    oidx = og.build(0, 1)
    assert_labels_equal_oracle(idx, oidx)
    qu, qv = W.uniform_queries(6000, 20_000, 1)
    for fl in (E.QueryFlags(), E.QueryFlags(use_bl=False), E.QueryFlags(prune_dl=False, prune_bl=False)):
        out, _ = E.query_batch(g, idx, (qu, qv), flags=fl)
        oc, _ = og.query_batch(oidx, qu, qv, fl.bits(), threads=8)
        np.testing.assert_array_equal(out.codes, oc)


def test_wide_labels_k256():
    n, src, dst = rmat_case(14, 8, 21)
    g = E.DynamicGraph.from_edges(n, src, dst)
    og = O.OracleGraph(n, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=256, k_prime=64))
    oidx = og.build(256, 64, threads=8)
    assert_labels_equal_oracle(idx, oidx)
    qu, qv = W.uniform_queries(n, 50_000, 2)
    out, _ = E.query_batch(g, idx, (qu, qv))
    oc, _ = og.query_batch(oidx, qu, qv, threads=8)
    np.testing.assert_array_equal(out.codes, oc)
    iu, iv = W.gen_insert_workload(src, dst, n, 500, 3)
    E.insert_edges(g, idx, iu, iv)
    for u, v in zip(iu.tolist(), iv.tolist()):
        og.insert_edge(oidx, u, v)
    assert_labels_equal_oracle(idx, oidx)


def test_odd_widths_and_strategies():
    src, dst = W.gen_random_graph(700, 3, seed=8)
    g = E.DynamicGraph.from_edges(700, src, dst)
    og = O.OracleGraph(700, src, dst)
    for k, kp, strat, thr, seed in ((100, 96, "max", 0, 3), (0, 13, "sum", 2, 1), (640, 200, "min", 4, 9)):
        cfg = E.IndexConfig(k=k, k_prime=kp, landmark_strategy=E.LandmarkStrategy(strat),
                            leaf_threshold=thr, hash_seed=seed)
        idx = E.build_index(g, cfg)
        oidx = og.build(k, kp, strat, thr, seed, threads=4)
        np.testing.assert_array_equal(np.array(idx.landmark_set.landmarks, np.uint32), oidx.landmarks)
        assert_labels_equal_oracle(idx, oidx)
        qu, qv = W.uniform_queries(700, 20_000, k)
        out, _ = E.query_batch(g, idx, (qu, qv))
        oc, _ = og.query_batch(oidx, qu, qv, threads=4)
        np.testing.assert_array_equal(out.codes, oc)


def test_empty_and_edge_cases():
    g = E.DynamicGraph.from_edges(5, [], [])
    idx = E.build_index(g, E.IndexConfig(k=5, k_prime=3))
    out, st = E.query_batch(g, idx, [])
    assert len(out) == 0 and st.query_count == 0
    out, _ = E.query_batch(g, idx, [(0, 0), (1, 2)])
    assert [o.answered_by for o in out] == [E.AnsweredBy.REFLEXIVE, E.AnsweredBy.BL_NEGATIVE]
    # self-loops count toward degrees like the reference
    g2 = E.DynamicGraph.from_edges(3, [0, 0, 1, 1], [0, 1, 2, 2])
    assert g2.edge_count == 3
    ind, outd = g2.degrees()
    assert ind.tolist() == [1, 1, 1] and outd.tolist() == [2, 1, 0]
    # insert_vertex grows graph and index together
    g3 = E.DynamicGraph.from_edges(4, [0, 1, 2], [1, 2, 3])
    idx3 = E.build_index(g3, E.IndexConfig(k=2, k_prime=2))
    E.insert_vertex(g3, idx3, out_edges=[0], in_edges=[3])
    assert g3.vertex_count == 5
    assert E.query(g3, idx3, 3, 0).reachable
    assert idx3.labels_equal(E.rebuild_index(g3, idx3))


def test_graph_buffered_then_device_edges():
    g = E.DynamicGraph(6)
    assert g.add_edge(0, 1) and not g.add_edge(0, 1)
    g.add_edge(1, 2)
    idx = E.build_index(g, E.IndexConfig(k=2, k_prime=2))
    assert g.edge_count == 2
    assert g.add_edge(2, 3) and not g.add_edge(2, 3)
    assert g.edge_count == 3 and g.has_edge(2, 3)
    assert sorted(g.edges()) == [(0, 1), (1, 2), (2, 3)]
    with pytest.raises(E.VertexRangeError):
        g.add_edge(0, 6)
    del idx


@pytest.mark.parametrize("world", [2, 3, 8])
def test_word_sharded_build_single_process(world):
    """The sharded build's device pieces (dbl_index_create / build_words /
    pack / unpack), with the allgather done in-process: every emulated rank
    builds only its words into its own index; the exchanged tables must equal
    a full build."""
    import torch
    from paper_2101_09441_b200.parallel import DeviceWordEngine, create_index, sharded_exchange
    n, src, dst = rmat_case(13, 8, 5)
    g = E.DynamicGraph.from_edges(n, src, dst)
    full = E.build_index(g, E.IndexConfig(k=128, k_prime=64))
    engines = [DeviceWordEngine(g, create_index(g, E.IndexConfig(k=128, k_prime=64))) for _ in range(world)]
    from paper_2101_09441_b200.parallel import plan_words
    plan = plan_words(engines[0].rw, world)
    maxw = max(len(p) for p in plan)
    slabs = []
    for r, eng in enumerate(engines):
        if plan[r]:
            eng.build_words(plan[r])
        s = eng.empty_slab(maxw)
        if plan[r]:
            eng.pack(plan[r], s)
        slabs.append(s)
    gathered = torch.cat(slabs)
    per = maxw * n
    for r, eng in enumerate(engines):
        for p in range(world):
            if p != r and plan[p]:
                eng.unpack(plan[p], gathered[p * per:(p + 1) * per])
        assert eng.idx.labels_equal(full), r


# ------------------------------------------- device landmark top-k (prep) --

@pytest.mark.parametrize("strategy", ["product", "sum", "max", "min"])
def test_topk_flat_scores_fallback(strategy):
    """Every vertex of a directed cycle has score 1 (or 2): more candidates in
    the threshold bin than the on-chip sort holds, so the build re-selects
    with the radix-sort path.  Landmarks must be ids 0..k-1 (ties by id,
    labels.py:145-146) and the labels equal the oracle's."""
    n = 20_000
    src = np.arange(n, dtype=np.uint32)
    dst = ((src + 1) % n).astype(np.uint32)
    g = E.DynamicGraph.from_edges(n, src, dst)
    cfg = E.IndexConfig(k=64, landmark_strategy=E.LandmarkStrategy(strategy))
    idx = E.build_index(g, cfg)
    og = O.OracleGraph(n, src, dst)
    oidx = og.build(64, 64, strategy=strategy, threads=8)
    assert idx.landmark_set.landmarks == tuple(range(64))
    np.testing.assert_array_equal(np.array(idx.landmark_set.landmarks), oidx.landmarks)
    assert_labels_equal_oracle(idx, oidx)


@pytest.mark.parametrize("n_hot", [8000, 8300])
def test_topk_candidate_table_boundary(n_hot):
    """n_hot vertices share the top score bin (just under / just over the
    8192-entry on-chip candidate table): both paths give the oracle's
    landmarks and labels."""
    rng = np.random.default_rng(n_hot)
    n = 30_000
    # hot vertices: in = out = 3 (score 9, bin 4); the rest: degree <= 1
    hot = np.arange(n_hot, dtype=np.uint32)
    src, dst = [], []
    for j in range(3):
        src.append(hot)
        dst.append(((hot + 1 + j * 977) % n_hot).astype(np.uint32))
    cold = np.arange(n_hot, n, dtype=np.uint32)
    src.append(cold[:-1])
    dst.append(cold[1:])
    src = np.concatenate(src).astype(np.uint32)
    dst = np.concatenate(dst).astype(np.uint32)
    perm = rng.permutation(n).astype(np.uint32)   # scatter the hot ids
    src, dst = perm[src], perm[dst]
    g = E.DynamicGraph.from_edges(n, src, dst)
    og = O.OracleGraph(n, src, dst)
    for k in (64, 256):
        idx = E.build_index(g, E.IndexConfig(k=k))
        oidx = og.build(k, 64, threads=8)
        np.testing.assert_array_equal(np.array(idx.landmark_set.landmarks), oidx.landmarks)
        assert_labels_equal_oracle(idx, oidx)


# ------------------------------------------------------- pivot head start --

def _two_component_graph(seed):
    """Two R-MAT blocks (the second one smaller) with one-way bridges from the
    second into the first: the pivot (landmark 0, a hub of block 1) reaches
    only block 1, while block 2's seeds reach block 1 through the bridges."""
    s1, d1 = W.rmat_edges(13, 8, seed)
    s2, d2 = W.rmat_edges(11, 4, seed + 1)
    off = np.uint32(1 << 13)
    rng = np.random.default_rng(seed)
    bu = (rng.integers(0, 1 << 11, 300) + (1 << 13)).astype(np.uint32)
    bv = rng.integers(0, 1 << 13, 300).astype(np.uint32)
    src = np.concatenate([s1, s2 + off, bu]).astype(np.uint32)
    dst = np.concatenate([d1, d2 + off, bv]).astype(np.uint32)
    return (1 << 13) + (1 << 11), src, dst


@pytest.mark.parametrize("case", ["two_components", "dag", "reverse_dag"])
def test_pivot_head_start_partial_cover(case):
    """The head start covers only part of the graph (the pivot's SCC does not
    hold every seed, or the graph is acyclic): labels must still equal the
    oracle's word for word."""
    if case == "two_components":
        n, src, dst = _two_component_graph(5)
    else:
        n = 6000
        src, dst = W.gen_random_graph(n, 4, seed=9, acyclic=True)
        if case == "reverse_dag":
            src, dst = dst, src
    g = E.DynamicGraph.from_edges(n, src, dst)
    og = O.OracleGraph(n, src, dst)
    for k, kp in ((64, 64), (100, 13)):
        idx = E.build_index(g, E.IndexConfig(k=k, k_prime=kp))
        oidx = og.build(k, kp, threads=8)
        np.testing.assert_array_equal(np.array(idx.landmark_set.landmarks), oidx.landmarks)
        assert_labels_equal_oracle(idx, oidx)
        # rebuild (frozen metadata) after some inserts also starts from the pivot
        iu, iv = W.gen_insert_workload(src, dst, n, 500, 7)
        E.insert_edges(g, idx, iu, iv)
        assert idx.labels_equal(E.rebuild_index(g, idx))
        g = E.DynamicGraph.from_edges(n, src, dst)


@pytest.mark.parametrize("count", [1, 255, 256, 1000, 100_003])
def test_zero_copy_host_queries_match_device(count):
    """Pinned host buffers take the zero-copy path (pairs staged per CTA with
    16-byte loads over PCIe); codes and visited counts must equal the
    device-resident batch for ragged sizes."""
    import torch
    from paper_2101_09441_b200 import _native as N
    n, src, dst = rmat_case(14, 8, 21)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g)
    qu, qv = W.uniform_queries(n, count, 5)
    du = torch.from_numpy(qu.view(np.int32)).cuda()
    dv = torch.from_numpy(qv.view(np.int32)).cuda()
    dc, dvis = E.query_codes(g, idx, du, dv)
    hu = torch.from_numpy(qu.view(np.int32)).pin_memory()
    hv = torch.from_numpy(qv.view(np.int32)).pin_memory()
    hc = torch.empty(count, dtype=torch.uint8).pin_memory()
    hvis = torch.empty(count, dtype=torch.int32).pin_memory()
    N.call("dbl_query", idx.handle, g.handle, N.ptr(hu), N.ptr(hv), count, E.DEFAULT_FLAGS.bits(), N.ptr(hc),
           N.ptr(hvis), N.MEM_HOST)
    np.testing.assert_array_equal(hc.numpy(), dc.cpu().numpy())
    np.testing.assert_array_equal(hvis.numpy(), dvis.cpu().numpy())


@pytest.mark.parametrize("k,kp", [(64, 64), (640, 96)])
def test_pivot_capped_sweeps_deep_graph(k, kp):
    """A long cycle with sparse chords: the pivot's reachability needs far
    more bottom-up sweeps than the cap, so the partial sets are handed to the
    label fixpoint's frontier (with k = 640 the record has several word
    groups and only the first group's words get the head start)."""
    n = 12_000
    rng = np.random.default_rng(3)
    cyc_s = np.arange(n, dtype=np.uint32)
    cyc_d = ((cyc_s + 1) % n).astype(np.uint32)
    ch_s = rng.integers(0, n, 400).astype(np.uint32)
    ch_d = ((ch_s.astype(np.int64) + rng.integers(2, 50, 400)) % n).astype(np.uint32)
    tail_s = np.arange(n, n + 2000, dtype=np.uint32)          # a tail of leaves hanging off
    tail_d = rng.integers(0, n, 2000).astype(np.uint32)
    src = np.concatenate([cyc_s, ch_s, tail_s, tail_d]).astype(np.uint32)
    dst = np.concatenate([cyc_d, ch_d, tail_d, tail_s + 2000]).astype(np.uint32)
    nn = n + 4000
    g = E.DynamicGraph.from_edges(nn, src, dst)
    og = O.OracleGraph(nn, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=k, k_prime=kp))
    oidx = og.build(k, kp, threads=8)
    np.testing.assert_array_equal(np.array(idx.landmark_set.landmarks), oidx.landmarks)
    assert_labels_equal_oracle(idx, oidx)


def test_insert_batch_range_error_leaves_index_untouched():
    """A batch with one endpoint outside [0, n) raises VertexRangeError and
    inserts nothing (updates.py checks before mutating): the batch is aborted
    on the device, so edges, labels and the delta adjacency stay as they
    were, before and after some delta already exists."""
    n, src, dst = rmat_case(12, 8, 31)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g)
    for round_ in range(2):
        before_m = g.edge_count
        before = idx.export_words()
        iu, iv = W.gen_insert_workload(src, dst, n, 300, 40 + round_)
        bad_v = iv.copy()
        bad_v[137] = n + 5
        with pytest.raises(E.VertexRangeError):
            E.insert_edges(g, idx, iu, bad_v)
        assert g.edge_count == before_m
        after = idx.export_words()
        for f in FAMS:
            np.testing.assert_array_equal(after[f], before[f], err_msg=f)
        # a valid batch afterwards still matches a frozen-metadata rebuild
        st = E.insert_edges(g, idx, iu, iv)
        assert st.inserted == len(iu)
        assert idx.labels_equal(E.rebuild_index(g, idx))


def test_device_inputs_ordered_after_producer_stream():
    """Device edge/query arrays produced by still-running torch kernels (legacy
    default stream) must be read only after those kernels finish: the engine's
    non-blocking stream waits on them.  Before the fix, a graph built right
    after asynchronous torch work, with the engine's pool already warm (no
    implicit cudaMalloc sync), lost edges (cfg5 after cfg4: 1.06 B -> 0.29 B)."""
    import torch
    n, src, dst = rmat_case(20, 8, 3)
    keys = np.unique((src.astype(np.uint64) << np.uint64(32)) | dst.astype(np.uint64))
    keys = keys[(keys >> np.uint64(32)) != (keys & np.uint64(0xFFFFFFFF))]
    expected = len(keys)
    E.DynamicGraph.from_edges(n, torch.from_numpy(src.view(np.int32)).cuda(),
                              torch.from_numpy(dst.view(np.int32)).cuda())   # warms the pool
    s0 = torch.from_numpy(src.view(np.int32)).cuda()
    d0 = torch.from_numpy(dst.view(np.int32)).cuda()
    for trial in range(3):
        perm = torch.randperm(s0.numel(), device="cuda")
        inv = torch.argsort(perm)
        s2, d2 = s0[perm][inv], d0[perm][inv]   # same content, written by queued kernels
        g = E.DynamicGraph.from_edges(n, s2, d2)
        assert g.edge_count == expected, trial
        idx = E.build_index(g)
        qu = torch.randint(0, n, (1 << 20,), device="cuda", dtype=torch.int32)
        qv = torch.randint(0, n, (1 << 20,), device="cuda", dtype=torch.int32)
        qu2, qv2 = qu[perm[: 1 << 20] % (1 << 20)], qv[perm[: 1 << 20] % (1 << 20)]
        codes, _ = E.query_codes(g, idx, qu2, qv2)
        ref, _ = E.query_batch(g, idx, (qu2.cpu().numpy().view(np.uint32), qv2.cpu().numpy().view(np.uint32)))
        np.testing.assert_array_equal(codes.cpu().numpy(), ref.codes)


# ------------------------------------------------- dl_intersec / bl_contain --

def test_label_tests_kats(toy_golden):
    """dl_intersec / bl_contain (labels.py:315-327) on the device against the
    reference's answers for all pairs (tests/golden/label_tests.npz; the
    reference's KATs tests/test_labels.py:166-191 are rows of the toy set)."""
    from conftest import golden
    from paper_2101_09441_b200.labels import _label_tests
    d = golden("label_tests")
    g, idx = toy_index(toy_golden)
    dl, bl = _label_tests(idx, d["toy_x"], d["toy_y"])
    np.testing.assert_array_equal(dl, d["toy_dl"].astype(bool))
    np.testing.assert_array_equal(bl, d["toy_bl"].astype(bool))
    assert E.dl_intersec(idx, 0, 9) is True          # (V1, V10)
    assert E.dl_intersec(idx, 2, 10) is False        # (V3, V11): a miss, not a refutation
    assert E.dl_intersec(idx, 2, 2) is False
    assert E.bl_contain(idx, 3, 5) is False          # (V4, V6)
    assert E.bl_contain(idx, 4, 1) is True           # (V5, V2)
    assert all(E.bl_contain(idx, v, v) for v in range(11))
    with pytest.raises(E.VertexRangeError):
        E.dl_intersec(idx, 0, 11)
    for name in ("r64", "r130", "dag"):
        n = int(d[name + "_n"])
        gg = E.DynamicGraph.from_edges(n, d[name + "_src"], d[name + "_dst"])
        cfg = E.IndexConfig(k=int(d[name + "_k"]), k_prime=int(d[name + "_k_prime"]),
                            leaf_threshold=int(d[name + "_threshold"]))
        ix = E.build_index(gg, cfg)
        assert_labels(ix, d, name + "_")
        x, y = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        dl, bl = _label_tests(ix, x.ravel(), y.ravel())
        np.testing.assert_array_equal(dl, d[name + "_dl"].ravel().astype(bool), err_msg=name)
        np.testing.assert_array_equal(bl, d[name + "_bl"].ravel().astype(bool), err_msg=name)


@pytest.mark.parametrize("k,kp", [(64, 64), (256, 64), (100, 13)])
def test_label_tests_random_pairs_vs_oracle(k, kp):
    """10k random pairs on R-MAT 2^12 against the oracle formula on the oracle's words."""
    n = 1 << 12
    src, dst = W.rmat_edges(12, 8, seed=21)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=k, k_prime=kp))
    oidx = O.OracleGraph(n, src, dst).build(k, kp, threads=2)
    assert_labels_equal_oracle(idx, oidx)
    from paper_2101_09441_b200.labels import _label_tests
    x, y = W.uniform_queries(n, 10_000, seed=22)
    dl, bl = _label_tests(idx, x, y)
    odl, obl = O.label_tests({f: getattr(oidx, f) for f in FAMS}, x, y)
    np.testing.assert_array_equal(dl, odl)
    np.testing.assert_array_equal(bl, obl)


def test_dense_workspace_lazy_paths():
    """The dense BFS workspace is allocated on first need: a batch that needs it
    is re-run by whichever path issued it -- the staged small host batch, the
    chunked pageable pipeline (> 64k pairs), the device-resident synchronous
    call, and dbl_query_async completed by dbl_sync."""
    import torch
    from paper_2101_09441_b200 import _native as N
    # no labels to prune with, and targets with no in-edges: every such BFS
    # exhausts the giant component (thousands of vertices), overflowing the
    # 64-query groups' shared tables
    nn = 12_000
    src, dst = W.gen_random_graph(nn, 2.0, seed=5)
    og = O.OracleGraph(nn, src, dst)
    oidx = og.build(0, 1)
    qu, qv = W.uniform_queries(nn, 70_000, 3)
    sources = np.setdiff1d(np.arange(nn, dtype=np.uint32), dst)
    qv[::2] = sources[np.arange(len(qv[::2])) % len(sources)]
    fl = E.QueryFlags(prune_dl=False, prune_bl=False)   # unpruned cones outgrow the shared tables
    oc, _ = og.query_batch(oidx, qu, qv, fl.bits(), threads=8)
    for path in ("staged", "pipelined", "device", "async"):
        g = E.DynamicGraph.from_edges(nn, src, dst)   # fresh graph: no dense workspace yet
        idx = E.build_index(g, E.IndexConfig(k=0, k_prime=1))
        if path == "staged":
            codes, _ = E.query_codes(g, idx, qu[:30_000], qv[:30_000], fl)
            np.testing.assert_array_equal(codes, oc[:30_000], err_msg=path)
        elif path == "pipelined":
            codes, _ = E.query_codes(g, idx, qu, qv, fl)
            np.testing.assert_array_equal(codes, oc, err_msg=path)
        else:
            du = torch.from_numpy(qu.view(np.int32)).cuda()
            dv = torch.from_numpy(qv.view(np.int32)).cuda()
            if path == "device":
                codes, _ = E.query_codes(g, idx, du, dv, fl)
            else:
                torch.cuda.synchronize()
                codes = torch.empty(len(qu), dtype=torch.uint8, device="cuda")
                N.call("dbl_query_async", idx.handle, g.handle, N.ptr(du), N.ptr(dv), len(qu), fl.bits(),
                       N.ptr(codes), None)
                N.call("dbl_sync", g.handle)
            np.testing.assert_array_equal(codes.cpu().numpy(), oc, err_msg=path)
        qc = np.zeros(8, np.uint32)
        N.call("dbl_query_counters", g.handle, N.ptr(qc))
        assert qc[3] > 0, f"{path}: the batch did not need the dense kernel"
