"""Determinism stress (the race evidence this pool allows: compute-sanitizer
is not available here).  The engine's kernels use relaxed atomics, L2-coherent
reads of other CTAs' words, grid barriers and last-CTA counter closes; a race
in any of them shows up as run-to-run differences.  Labels are least
fixpoints and answers are order-independent, so every repetition must be
bit-identical: many builds (pivot head start + fixpoint), many query batches
(lean kernel, tail-launched BFS kernels), insert batches against rebuilds,
and concurrent multi-handle batches.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import parallel as P
from paper_2101_09441_b200 import workload as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("k,kp", [(64, 64), (256, 64)])
def test_repeated_builds_identical(k, kp):
    n = 1 << 16
    src, dst = W.rmat_edges(16, 8, seed=41)
    g = E.DynamicGraph.from_edges(n, src, dst)
    cfg = E.IndexConfig(k=k, k_prime=kp)
    first = E.build_index(g, cfg)
    for _ in range(25):
        assert E.build_index(g, cfg).labels_equal(first)
    assert E.verify_labels(g, first, exhaustive=False).ok


def test_repeated_query_batches_identical():
    n = 1 << 16
    src, dst = W.rmat_edges(16, 4, seed=42)
    g = E.DynamicGraph.from_edges(n, src, dst)
    for cfg in (E.IndexConfig(), E.IndexConfig(k=256, k_prime=64), E.IndexConfig(k=4, k_prime=2)):
        idx = E.build_index(g, cfg)
        qu, qv = W.uniform_queries(n, 200_000, seed=43)
        c0, v0 = E.query_codes(g, idx, qu, qv)
        assert c0.max() <= 6
        for _ in range(40):
            c, v = E.query_codes(g, idx, qu, qv)
            assert np.array_equal(c, c0)
            assert np.array_equal(v == 0, v0 == 0)


def test_insert_batches_match_rebuild_repeatedly():
    n = 1 << 15
    src, dst = W.rmat_edges(15, 4, seed=44)
    for rep in range(3):
        g = E.DynamicGraph.from_edges(n, src, dst)
        idx = E.build_index(g)
        prev = None
        for b in range(5):
            iu, iv = W.gen_insert_workload(src, dst, n, 5000, 45 + b, exclude=prev)
            prev = (iu, iv) if prev is None else (np.concatenate([prev[0], iu]), np.concatenate([prev[1], iv]))
            E.insert_edges(g, idx, iu, iv)
            assert idx.labels_equal(E.rebuild_index(g, idx)), (rep, b)


def test_concurrent_handles_identical():
    n = 1 << 14
    src, dst = W.rmat_edges(14, 8, seed=46)
    reps = P.replicate(n, src, dst, [0, 0, 0])
    qu, qv = W.uniform_queries(n, 300_000, seed=47)
    ref, _ = E.query_batch(reps[0][0], reps[0][1], (qu, qv))
    for _ in range(20):
        out, _ = P.query_batch_sharded(reps, (qu, qv))
        assert np.array_equal(out.codes, ref.codes)
