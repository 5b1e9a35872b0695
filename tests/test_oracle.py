"""Pin the CPU oracle (oracle/dbl_oracle.c) to the reference's own outputs.

The golden vectors were produced by running the unmodified reference
(oracle/gen_golden.py); the oracle must reproduce every one of them before
any GPU parity claim rests on it.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O


def graph_from(d, p=""):
    return O.OracleGraph(int(d[p + "n"]), d[p + "src"], d[p + "dst"])


def assert_index_equal(idx, d, p=""):
    np.testing.assert_array_equal(idx.landmarks, d[p + "landmarks"])
    np.testing.assert_array_equal(idx.leaf_flags, d[p + "leaf_flags"])
    mask = idx.leaf_flags != 0
    np.testing.assert_array_equal(idx.bucket[mask], d[p + "bucket"][mask])
    for fam in ("dl_in", "dl_out", "bl_in", "bl_out"):
        np.testing.assert_array_equal(getattr(idx, fam), d[p + fam], err_msg=fam)


def test_leaf_hash_kats():
    d = golden("leaf_hash")
    for i, v in enumerate(d["ids"]):
        for j, kp in enumerate(d["kprimes"]):
            for s, sd in enumerate(d["seeds"]):
                assert O.leaf_hash(int(v), int(kp), int(sd)) == d["buckets"][i, j, s]
    # survey KATs (SURVEY.md §7 hard part 1)
    assert O.leaf_hash(1, 64, 0) == 47
    assert O.leaf_hash(12345, 64, 7) == 5
    assert O.leaf_hash(0, 64, 0) == 0


def test_landmarks_and_leaves_kats():
    d = golden("landmarks")
    for ci in range(4):
        g = O.OracleGraph(int(d[f"c{ci}_n"]), d[f"c{ci}_src"], d[f"c{ci}_dst"])
        for s in ("max", "min", "sum", "product"):
            exp = d[f"c{ci}_{s}"]
            np.testing.assert_array_equal(g.select_landmarks(len(exp), s), exp)
        for thr in (0, 2, 6):
            flags, bucket = g.select_leaves(thr, 13, 5)
            np.testing.assert_array_equal(flags, d[f"c{ci}_leaf_flags_t{thr}"])
            m = flags != 0
            np.testing.assert_array_equal(bucket[m], d[f"c{ci}_bucket_t{thr}"][m])


def test_toy_tables(toy_golden):
    d = toy_golden
    g = graph_from(d)
    ovr = {0: 0, 9: 0, 1: 1, 2: 1, 10: 1}  # pinned buckets, pkg/tests/conftest.py:23
    flags, bucket = g.select_leaves(0, 2, 0, ovr)
    idx = g.build(2, 2, landmarks=np.array([4, 7], np.uint32), leaf_flags=flags, bucket=bucket)
    assert_index_equal(idx, d)
    for fam in ("dl_in", "dl_out", "bl_in", "bl_out"):
        np.testing.assert_array_equal(getattr(idx, fam)[:, 0], d["exp_" + fam])
    auto = g.build(3, 4)
    assert_index_equal(auto, d, "auto_")


def test_toy_queries_all_flagsets(toy_golden):
    d = toy_golden
    g = graph_from(d)
    idx = g.build(2, 2, landmarks=d["landmarks"], leaf_flags=d["leaf_flags"], bucket=d["bucket"])
    for name in ("default", "dl_only", "bl_only", "no_early", "no_prune", "bare"):
        codes, visited = g.query_batch(idx, d["qu"], d["qv"], int(d[f"flagbits_{name}"]))
        np.testing.assert_array_equal(codes, d[f"codes_{name}"], err_msg=name)
        np.testing.assert_array_equal(visited, d[f"visited_{name}"], err_msg=name)


def test_toy_insertion_example(toy_golden):
    d = toy_golden
    g = graph_from(d)
    idx = g.build(2, 2, landmarks=d["landmarks"], leaf_flags=d["leaf_flags"], bucket=d["bucket"])
    st = g.insert_edge(idx, *map(int, d["ins_uv"]))
    assert st == tuple(int(x) for x in d["ins_stats"][:2]) + (bool(d["ins_stats"][2]),)
    for fam in ("dl_in", "dl_out", "bl_in", "bl_out"):
        np.testing.assert_array_equal(getattr(idx, fam), d["ins_" + fam])
    g2 = graph_from(d)
    idx2 = g2.build(2, 2, landmarks=d["landmarks"], leaf_flags=d["leaf_flags"], bucket=d["bucket"])
    st2 = g2.insert_edge(idx2, *map(int, d["ins2_uv"]))
    assert st2 == (0, 0, True)


def test_family_build_query_insert(family_golden):
    d = family_golden
    flagbits = {"default": 63, "bl_only": 0b111110, "bare": 0b000011}
    for i in range(int(d["count"])):
        p = f"f{i}_"
        g = graph_from(d, p)
        k = int(d[p + "k"])
        idx = g.build(k, k)
        assert_index_equal(idx, d, p)
        n = int(d[p + "n"])
        qu = np.repeat(np.arange(n, dtype=np.uint32), n)
        qv = np.tile(np.arange(n, dtype=np.uint32), n)
        for name, fb in flagbits.items():
            codes, visited = g.query_batch(idx, qu, qv, fb, threads=2)
            np.testing.assert_array_equal(codes, d[p + f"codes_{name}"], err_msg=f"{i} {name}")
            np.testing.assert_array_equal(visited, d[p + f"visited_{name}"], err_msg=f"{i} {name}")
        for j, (u, v) in enumerate(zip(d[p + "ins_u"], d[p + "ins_v"])):
            st = g.insert_edge(idx, int(u), int(v))
            exp = d[p + "ins_stats"][j]
            assert st == (int(exp[0]), int(exp[1]), bool(exp[2])), (i, j)
        for fam in ("dl_in", "dl_out", "bl_in", "bl_out"):
            np.testing.assert_array_equal(getattr(idx, fam), d[p + "after_" + fam])
        re = g.rebuild(idx)
        for fam in ("dl_in", "dl_out", "bl_in", "bl_out"):
            np.testing.assert_array_equal(getattr(re, fam), getattr(idx, fam))


def test_cfg1_full(cfg1_golden):
    d = cfg1_golden
    g = graph_from(d)
    idx = g.build(64, 64, threads=4)
    assert_index_equal(idx, d)
    codes, visited = g.query_batch(idx, d["qu"], d["qv"], threads=4)
    np.testing.assert_array_equal(codes, d["codes"])
    np.testing.assert_array_equal(visited, d["visited"])
    for j, (u, v) in enumerate(zip(d["ins_u"], d["ins_v"])):
        st = g.insert_edge(idx, int(u), int(v))
        e = d["ins_stats"][j]
        assert st == (int(e[0]), int(e[1]), bool(e[2])), j
    for fam in ("dl_in", "dl_out", "bl_in", "bl_out"):
        np.testing.assert_array_equal(getattr(idx, fam), d["after_" + fam])


def test_reach_batch_matches_codes(cfg1_golden):
    d = cfg1_golden
    g = graph_from(d)
    reach = g.reach_batch(d["qu"][:20000], d["qv"][:20000], threads=4)
    exp = np.isin(d["codes"][:20000], (0, 1, 5))
    np.testing.assert_array_equal(reach, exp)


def test_label_tests_kats():
    """dl_intersec / bl_contain: the restated formula against the reference's
    answers on all pairs (tests/golden/label_tests.npz), incl. the KATs of
    the reference's tests/test_labels.py:166-191 (worked example)."""
    from conftest import golden
    d = golden("label_tests")
    t = golden("toy")
    lab = {f: t[f] for f in ("dl_in", "dl_out", "bl_in", "bl_out")}
    dl, bl = O.label_tests(lab, d["toy_x"], d["toy_y"])
    np.testing.assert_array_equal(dl, d["toy_dl"].astype(bool))
    np.testing.assert_array_equal(bl, d["toy_bl"].astype(bool))
    pair = {(int(a), int(b)): i for i, (a, b) in enumerate(zip(d["toy_x"], d["toy_y"]))}
    V1, V2, V3, V4, V5, V6, V10, V11 = 0, 1, 2, 3, 4, 5, 9, 10
    assert d["toy_dl"][pair[V1, V10]] == 1
    assert d["toy_dl"][pair[V3, V11]] == 0
    assert d["toy_dl"][pair[V3, V3]] == 0
    assert d["toy_bl"][pair[V4, V6]] == 0
    assert d["toy_bl"][pair[V5, V2]] == 1
    assert all(d["toy_bl"][pair[v, v]] == 1 for v in range(11))
    for name in ("r64", "r130", "dag"):
        n = int(d[name + "_n"])
        lab = {f: d[f"{name}_{f}"] for f in ("dl_in", "dl_out", "bl_in", "bl_out")}
        x, y = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        dl, bl = O.label_tests(lab, x.ravel(), y.ravel())
        np.testing.assert_array_equal(dl, d[name + "_dl"].ravel().astype(bool), err_msg=name)
        np.testing.assert_array_equal(bl, d[name + "_bl"].ravel().astype(bool), err_msg=name)
        # the oracle's own build reproduces the reference labels of these graphs
        og = O.OracleGraph(n, d[name + "_src"], d[name + "_dst"])
        oidx = og.build(int(d[name + "_k"]), int(d[name + "_k_prime"]), leaf_threshold=int(d[name + "_threshold"]))
        for f in ("dl_in", "dl_out", "bl_in", "bl_out"):
            np.testing.assert_array_equal(getattr(oidx, f), lab[f], err_msg=f"{name} {f}")
