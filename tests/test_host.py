"""CPU-side checks: host logic, generators, and that the C-ABI library
loads and exports every symbol include/dbl_b200.h declares (no GPU calls)."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import _native as N
from paper_2101_09441_b200 import workload as W
from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "dbl_b200.h")).read()
    return sorted(set(re.findall(r"\b(dbl_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = N.lib()
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(N.exported_symbols())
    assert lib.dbl_version() == 1


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump -lelf {N.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_workload_reproduces_reference_cfg1(cfg1_golden):
    d = cfg1_golden
    s, t = W.gen_random_graph(10_000, 5, seed=1)
    assert len(s) == 50_000
    got = np.sort(s.astype(np.uint64) << np.uint64(32) | t)
    exp = np.sort(d["src"].astype(np.uint64) << np.uint64(32) | d["dst"])
    np.testing.assert_array_equal(got, exp)
    qu, qv = W.gen_random_queries(10_000, 100_000, seed=2)
    np.testing.assert_array_equal(qu, d["qu"])
    np.testing.assert_array_equal(qv, d["qv"])


def test_rmat_generator_shape():
    s, d = W.rmat_edges(12, 8, seed=1)
    assert len(s) == len(d) and len(s) <= 8 << 12
    assert (s != d).all() and s.max() < 4096 and d.max() < 4096
    s2, d2 = W.rmat_edges(12, 8, seed=1)
    np.testing.assert_array_equal(s, s2)
    # skew: vertex 0 is the top hub
    deg = np.bincount(s, minlength=4096)
    assert deg.argmax() == 0


def test_positive_queries_are_reachable_walks():
    from oracle import oracle as O
    s, d = W.rmat_edges(12, 4, seed=3)
    qu, qv = W.positive_queries(4096, s, d, 2000, seed=4)
    assert len(qu) == 2000 and (qu != qv).all()
    g = O.OracleGraph(4096, s, d)
    assert g.reach_batch(qu, qv).all()


def test_insert_workload_rule():
    s, d = W.rmat_edges(10, 4, seed=5)
    iu, iv = W.gen_insert_workload(s, d, 1024, 3000, seed=6)
    assert len(iu) == 3000 and (iu != iv).all()
    k = iu.astype(np.uint64) << np.uint64(32) | iv
    assert len(np.unique(k)) == 3000
    present = set(zip(s.tolist(), d.tolist()))
    assert not any((a, b) in present for a, b in zip(iu.tolist(), iv.tolist()))


def test_query_flags_bits_and_outcomes():
    assert E.DEFAULT_FLAGS.bits() == 63
    assert E.DL_ONLY.bits() == 63 & ~2
    assert E.BL_ONLY.bits() == 63 & ~1
    codes = np.array([0, 1, 2, 5, 6], np.uint8)
    vis = np.array([0, 0, 0, 3, 4], np.uint32)
    out = E.Outcomes(codes, vis)
    assert out[3] == E.QueryOutcome(True, E.AnsweredBy.BFS_POSITIVE, 3)
    assert list(out.reachable) == [True, True, False, True, False]
    assert out == [out[i] for i in range(5)]
    st = E.BatchStats.collect(out, 1.0)
    assert st.label_answered == 3 and st.rho == pytest.approx(0.6) and st.reachable_count == 3
    assert "4" in E.explain(out[4])


def test_pairs_parsing():
    from paper_2101_09441_b200.queries import _pairs_to_arrays
    u, v = _pairs_to_arrays([(1, 2), (3, 4)])
    assert u.tolist() == [1, 3] and v.tolist() == [2, 4]
    u, v = _pairs_to_arrays((np.array([5]), np.array([6])))
    assert u.tolist() == [5] and v.tolist() == [6]
    with pytest.raises(E.VertexRangeError):
        _pairs_to_arrays([(-1, 2)])


def test_leafsets_and_config_validation():
    ls = E.LeafSets({0, 2}, {1}, {0: 3, 1: 4, 2: 5})
    assert ls.leaves_in == {0, 2} and ls.leaves_out == {1}
    assert ls.in_bit(2) == 1 << 5 and ls.out_bit(2) == 0
    f, b = ls.for_vertex_count(5)
    assert f.tolist() == [1, 2, 1, 0, 0]
    with pytest.raises(E.ConfigError):
        E.IndexConfig(k=-1).validate(10)
    with pytest.raises(E.ConfigError):
        E.IndexConfig(k=11).validate(10)
    with pytest.raises(E.ConfigError):
        E.IndexConfig(k_prime=0).validate(10)
    with pytest.raises(E.ConfigError):
        E.LandmarkSet.of([1, 1])
    assert issubclass(E.VertexRangeError, IndexError) and issubclass(E.ConfigError, ValueError)


def test_no_silent_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(E.DeviceError):
        E.DynamicGraph.from_edges(4, [0, 1], [1, 2])
    with pytest.raises(E.DeviceError):
        E.leaf_hash(1, 64)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2101_09441_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\b(import|from)\s+oracle\b|oracle/|dbl_oracle|\borc_", text), f


def test_pairs_tuple_of_pairs_is_pairs():
    """A 2-tuple of (u, v) pairs means two queries, as in the reference; only a
    2-tuple of equal-length 1-D arrays is the column form."""
    from paper_2101_09441_b200.queries import _pairs_to_arrays
    u, v = _pairs_to_arrays(((0, 5), (3, 7)))
    assert u.tolist() == [0, 3] and v.tolist() == [5, 7]
    u, v = _pairs_to_arrays([(0, 5), (3, 7)])
    assert u.tolist() == [0, 3] and v.tolist() == [5, 7]
    u, v = _pairs_to_arrays((np.array([0, 3]), np.array([5, 7])))
    assert u.tolist() == [0, 3] and v.tolist() == [5, 7]
    # arrays of different lengths are not columns: read as pairs -> error
    with pytest.raises(Exception):
        _pairs_to_arrays((np.array([0, 3, 4]), np.array([5, 7])))
    u, v = _pairs_to_arrays(np.array([[1, 2], [3, 4]]))
    assert u.tolist() == [1, 3] and v.tolist() == [2, 4]
    # the fromiter fast path (a list of 2-tuples) equals np.array's on a large
    # list, on numpy scalars and on a generator; ragged pairs still raise
    rng = np.random.default_rng(0)
    big = [(int(a), int(b)) for a, b in rng.integers(0, 2**32, size=(5000, 2))]
    u, v = _pairs_to_arrays(big)
    ref = np.array(big, dtype=np.int64)
    assert np.array_equal(u, ref[:, 0]) and np.array_equal(v, ref[:, 1])
    u, v = _pairs_to_arrays((p for p in [(np.uint32(4), 5), (6, np.int64(7))]))
    assert u.tolist() == [4, 6] and v.tolist() == [5, 7]
    for bad in ([(1, 2), (3,)], [(1, 2, 3), (4,)], [(1, 2), 3]):
        with pytest.raises(Exception):
            _pairs_to_arrays(bad)
    with pytest.raises(Exception):
        _pairs_to_arrays([(0, 2**32)])


def test_slice_bounds_match_reference_pool():
    """Contiguous slices of ceil(q / parts) (queries.py:231-232)."""
    from paper_2101_09441_b200.parallel import slice_bounds
    for q in (0, 1, 7, 10, 1000, 1001):
        for parts in (1, 2, 3, 8):
            b = slice_bounds(q, parts)
            assert len(b) == parts
            chunk = -(-q // parts) if q else 1
            ref = [(i, min(i + chunk, q)) for i in range(0, q, chunk)]
            assert b[:len(ref)] == ref
            assert all(lo == hi == q for lo, hi in b[len(ref):])
            assert sum(hi - lo for lo, hi in b) == q
