import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W
n = 1 << 20
src, dst = W.rmat_edges(20, 8, 1)
g = E.DynamicGraph.from_edges(n, src, dst)
idx = E.build_index(g)
su, sv = W.gen_insert_workload(src, dst, n, 2300, 90)
for u, v in zip(su[:300].tolist(), sv[:300].tolist()):
    E.insert_edge(g, idx, u, v)
t0 = time.perf_counter()
for u, v in zip(su[300:].tolist(), sv[300:].tolist()):
    E.insert_edge(g, idx, u, v)
print("single insert_edge:", 2000 / (time.perf_counter() - t0), "edges/s")
