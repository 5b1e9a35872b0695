"""Workload for compute-sanitizer runs (memcheck / racecheck / synccheck /
initcheck): the worked example, config 1 (build, 100k queries, batched and
single-edge inserts), an R-MAT 2^12 pivot build with k = 256, forced BFS
fallbacks (k = 0: every non-trivial query takes the BFS kernels, incl. the
group kernel), and the pending-log path.  Compares with the golden fixtures
so a sanitizer run also checks the answers.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py [small]
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2101_09441_b200 as E  # noqa: E402
from paper_2101_09441_b200 import workload as W  # noqa: E402
from conftest import golden  # noqa: E402

FAMS = ("dl_in", "dl_out", "bl_in", "bl_out")
small = len(sys.argv) > 1 and sys.argv[1] == "small"


def check(idx, d, p=""):
    w = idx.export_words()
    for f in FAMS:
        assert np.array_equal(w[f], d[p + f]), p + f


# worked example
t = golden("toy")
g = E.DynamicGraph.from_edges(11, t["src"], t["dst"])
leaves = E.select_leaves(g, 0, k_prime=2, bucket_override={0: 0, 9: 0, 1: 1, 2: 1, 10: 1})
idx = E.build_index(g, E.IndexConfig(k=2, k_prime=2), landmarks=[4, 7], leaf_sets=leaves)
check(idx, t)
out, _ = E.query_batch(g, idx, (t["qu"], t["qv"]))
assert np.array_equal(out.codes, t["codes_default"])
st = E.insert_edge(g, idx, *map(int, t["ins_uv"]))
assert (st.visited, st.labels_changed, st.early_terminated) == tuple(int(x) for x in t["ins_stats"][:2]) + (False,)
print("toy ok", flush=True)

# config 1
d = golden("cfg1")
src, dst = W.gen_random_graph(10_000, 5, seed=1)
g = E.DynamicGraph.from_edges(10_000, src, dst)
idx = E.build_index(g)
check(idx, d)
nq = 20_000 if small else 100_000
out, _ = E.query_batch(g, idx, (d["qu"][:nq], d["qv"][:nq]))
assert np.array_equal(out.codes, d["codes"][:nq])
ni = 100 if small else 300
for j in range(ni):
    s1 = E.insert_edge(g, idx, int(d["ins_u"][j]), int(d["ins_v"][j]))
    e = d["ins_stats"][j]
    assert (s1.visited, s1.labels_changed, s1.early_terminated) == (int(e[0]), int(e[1]), bool(e[2])), j
E.insert_edges(g, idx, d["ins_u"][ni:], d["ins_v"][ni:])
check(idx, d, "after_")
print("cfg1 ok", flush=True)

# R-MAT 2^12, k = 256 (padded records, quad gather kernel), pivot head start
src, dst = W.rmat_edges(12, 8, seed=1)
g = E.DynamicGraph.from_edges(1 << 12, src, dst)
idx = E.build_index(g, E.IndexConfig(k=256, k_prime=64))
qu, qv = W.uniform_queries(1 << 12, 20_000, seed=2)
out, _ = E.query_batch(g, idx, (qu, qv))
rep = E.verify_labels(g, idx, exhaustive=True)
assert rep.ok
print("rmat k256 ok", flush=True)

# k = 0: every non-reflexive query is a BFS (warp, group and dense kernels)
idx0 = E.build_index(g, E.IndexConfig(k=0, k_prime=1))
out0, _ = E.query_batch(g, idx0, (qu[:4000], qv[:4000]))
assert np.array_equal(out0.reachable, out.reachable[:4000])
print("bfs paths ok", flush=True)
