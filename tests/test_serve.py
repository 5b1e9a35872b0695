"""Per-call query service (query.cu K6s): single query() calls answered by a
resident warp through a mailbox in pinned host memory.

Every single-call answer code must equal the batch path's answer for the
same pair (visited: zero for exactly the same pairs), under every flag set, across service
restarts caused by inserts, index switches, other graphs and idle exits.
"""
from __future__ import annotations

import time

import numpy as np
import pytest

from oracle import oracle as O
from paper_2101_09441_b200 import workload as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_09441_b200 as E
    return E


def code_of(E, outcome):
    return list(E.AnsweredBy).index(outcome.answered_by)


def test_single_calls_equal_batch_all_flagsets(E):
    n = 1 << 12
    src, dst = W.rmat_edges(12, 8, 31)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g)
    rng = np.random.default_rng(2)
    qu = rng.integers(0, n, 3000, dtype=np.uint32)
    qv = rng.integers(0, n, 3000, dtype=np.uint32)
    qu[:50] = qv[:50]                      # reflexive
    for flags in (E.QueryFlags(), E.QueryFlags(use_bl=False), E.QueryFlags(use_dl=False),
                  E.QueryFlags(use_thm1=False, use_thm2=False), E.QueryFlags(prune_dl=False, prune_bl=False),
                  E.QueryFlags(use_thm1=False, use_thm2=False, prune_dl=False, prune_bl=False)):
        bc, bv = E.query_codes(g, idx, qu, qv, flags)
        for i, (u, v) in enumerate(zip(qu.tolist(), qv.tolist())):
            o = E.query(g, idx, u, v, flags)
            assert code_of(E, o) == bc[i], (i, u, v, flags)
            # visited: 0 iff label-answered (the BFS variants may count differently)
            assert (o.visited == 0) == (bv[i] == 0), (i, u, v, flags)
    # the fallback share: BFS beyond the warp's bounds goes to the batch path
    fptr, fcol = g.adjacency(False)
    ref = O.csr_query_batch(n, fptr.astype(np.uint64), fcol, 64, 64, idx.export_words(), qu, qv)
    np.testing.assert_array_equal(E.query_codes(g, idx, qu, qv)[0], ref)


def test_single_calls_across_restarts(E):
    """Inserts (service stopped, pending log folded in at restart), a second
    graph and index (service moves), idle exits (service relaunched)."""
    n = 1 << 12
    src, dst = W.rmat_edges(12, 8, 32)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g)
    g2 = E.DynamicGraph.from_edges(n, *W.rmat_edges(12, 4, 33))
    idx2 = E.build_index(g2, E.IndexConfig(k=128, k_prime=64))
    rng = np.random.default_rng(5)
    for step in range(30):
        qu = rng.integers(0, n, 40, dtype=np.uint32)
        qv = rng.integers(0, n, 40, dtype=np.uint32)
        gg, ii = (g, idx) if step % 3 else (g2, idx2)
        bc, bv = E.query_codes(gg, ii, qu, qv)
        for i, (u, v) in enumerate(zip(qu.tolist(), qv.tolist())):
            o = E.query(gg, ii, u, v)
            assert code_of(E, o) == bc[i] and (o.visited == 0) == (bv[i] == 0), (step, i)
        if step % 4 == 1:   # single-edge inserts go to the pending log
            for _ in range(5):
                E.insert_edge(g, idx, int(rng.integers(0, n)), int(rng.integers(0, n)))
        if step % 7 == 2:
            time.sleep(0.005)   # longer than the service's idle timeout
    # labels after all of it still equal a rebuild, answers the oracle's
    assert idx.labels_equal(E.rebuild_index(g, idx))
    qu = rng.integers(0, n, 500, dtype=np.uint32)
    qv = rng.integers(0, n, 500, dtype=np.uint32)
    fptr, fcol = g.adjacency(False)
    ref = O.csr_query_batch(n, fptr.astype(np.uint64), fcol, 64, 64, idx.export_words(), qu, qv)
    got = np.array([code_of(E, E.query(g, idx, u, v)) for u, v in zip(qu.tolist(), qv.tolist())], np.uint8)
    np.testing.assert_array_equal(got, ref)


def test_single_call_range_error(E):
    n = 1 << 10
    g = E.DynamicGraph.from_edges(n, *W.rmat_edges(10, 4, 34))
    idx = E.build_index(g)
    E.query(g, idx, 1, 2)
    with pytest.raises(E.VertexRangeError):
        E.query(g, idx, 1, n)
    assert code_of(E, E.query(g, idx, 3, 3)) == 0


def test_single_calls_beside_other_threads(E):
    """Single queries on one thread while another thread builds and inserts on
    another graph (cooperative launches): the service never runs beside them
    (every other call blocks it), answers stay exact, nothing stalls."""
    import threading
    n = 1 << 12
    g = E.DynamicGraph.from_edges(n, *W.rmat_edges(12, 8, 35))
    idx = E.build_index(g)
    rng = np.random.default_rng(6)
    qu = rng.integers(0, n, 4000, dtype=np.uint32)
    qv = rng.integers(0, n, 4000, dtype=np.uint32)
    ref, _ = E.query_codes(g, idx, qu, qv)
    g2 = E.DynamicGraph.from_edges(n, *W.rmat_edges(12, 8, 36))
    errors = []

    def writer():
        try:
            r = np.random.default_rng(7)
            for _ in range(15):
                i2 = E.build_index(g2)
                E.insert_edges(g2, i2, r.integers(0, n, 500, dtype=np.uint32), r.integers(0, n, 500, dtype=np.uint32))
                assert i2.labels_equal(E.rebuild_index(g2, i2))
        except Exception as e:   # noqa: BLE001
            errors.append(e)

    t = threading.Thread(target=writer)
    t.start()
    got = np.array([code_of(E, E.query(g, idx, u, v)) for u, v in zip(qu.tolist(), qv.tolist())], np.uint8)
    t.join(timeout=120)
    assert not t.is_alive(), "writer thread stalled"
    assert not errors, errors
    np.testing.assert_array_equal(got, ref)


def test_single_calls_when_launches_block(E):
    """Under CUDA_LAUNCH_BLOCKING (as under a profiler or sanitizer, which
    serialise launches) a service kernel cannot see the request posted after
    its launch: the library notices the unanswered first request and answers
    single calls on the launch path from then on."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, paper_2101_09441_b200 as E\n"
        "from paper_2101_09441_b200 import workload as W\n"
        "n = 1 << 11\n"
        "g = E.DynamicGraph.from_edges(n, *W.rmat_edges(11, 8, 37))\n"
        "idx = E.build_index(g)\n"
        "r = np.random.default_rng(1)\n"
        "qu = r.integers(0, n, 300, dtype=np.uint32); qv = r.integers(0, n, 300, dtype=np.uint32)\n"
        "ref, _ = E.query_codes(g, idx, qu, qv)\n"
        "order = list(E.AnsweredBy)\n"
        "got = [order.index(E.query(g, idx, int(a), int(b)).answered_by) for a, b in zip(qu, qv)]\n"
        "E.insert_edge(g, idx, 5, 9)\n"
        "assert got == ref.tolist()\n"
        "print('ok')\n")
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
