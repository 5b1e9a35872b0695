"""`visited` of BFS-answered queries (queries.py:116-142 counts dequeues).

The engine's BFS stages (bounded warp BFS, 32-query bit-parallel warp BFS,
64-query group and dense kernels) all count the vertices of every BFS level
the query expands: all reached vertices for BFS_NEGATIVE -- exactly the
reference's count, since the FIFO dequeues every reached, unpruned vertex --
and the levels up to the one holding the target's predecessor for
BFS_POSITIVE (>= the reference's FIFO position, which depends on adjacency
order).  So pruning never increases `visited` (the reference's acceptance
criterion 7), whichever kernel answers, and label-answered queries keep 0.
"""
from __future__ import annotations

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


@pytest.mark.parametrize("scale,deg,k", [(12, 4, 64), (12, 2, 8), (11, 8, 256)])
def test_visited_against_the_reference_count(E, scale, deg, k):
    n = 1 << scale
    src, dst = W.rmat_edges(scale, deg, 41)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=k, k_prime=64))
    og = O.OracleGraph(n, src, dst)
    oidx = og.build(k, 64, threads=4)
    rng = np.random.default_rng(3)
    qu = rng.integers(0, n, 60_000, dtype=np.uint32)
    qv = rng.integers(0, n, 60_000, dtype=np.uint32)
    D = O.DEFAULT_FLAGS
    NP = O.F_PRUNE_DL | O.F_PRUNE_BL
    runs = {}
    for name, fl, of in (("default", E.QueryFlags(), D),
                         ("no_prune", E.QueryFlags(prune_dl=False, prune_bl=False), D & ~NP),
                         ("bl_only", E.QueryFlags(use_dl=False), D & ~O.F_USE_DL),
                         ("bl_only_no_prune", E.QueryFlags(use_dl=False, prune_bl=False),
                          D & ~O.F_USE_DL & ~O.F_PRUNE_BL)):
        codes, vis = E.query_codes(g, idx, qu, qv, fl)
        ocodes, ovis = og.query_batch(oidx, qu, qv, flags=of, threads=4)
        np.testing.assert_array_equal(codes, ocodes, err_msg=name)
        neg, pos, lab = codes == 6, codes == 5, codes < 5
        if name.startswith("bl_only"):   # without rule 1 the BFS answers the positives too
            assert neg.any() and pos.any(), name
        np.testing.assert_array_equal(vis[neg], ovis[neg], err_msg=f"{name}: BFS_NEGATIVE counts")
        assert np.all(vis[pos] >= ovis[pos]), name
        assert np.all(vis[lab] == 0), name
        runs[name] = (codes, vis)
    assert np.all(runs["default"][1] <= runs["no_prune"][1]), "pruning increased a visited count"
    assert np.all(runs["bl_only"][1] <= runs["bl_only_no_prune"][1]), "BL pruning increased a visited count"
    codes, vis = runs["bl_only_no_prune"]
    # the single-call service counts the same way
    for i in np.flatnonzero(codes >= 5)[:200].tolist():
        o = E.query(g, idx, int(qu[i]), int(qv[i]), E.QueryFlags(use_dl=False, prune_bl=False))
        assert o.visited == vis[i], i
