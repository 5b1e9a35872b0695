import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W
n = 1 << 20
src, dst = W.rmat_edges(20, 8, 1)
g = E.DynamicGraph.from_edges(n, src, dst)
idx = E.build_index(g)
qu, qv = W.uniform_queries(n, 200000, 9)
pairs = list(zip(qu.tolist(), qv.tolist()))
for u, v in pairs[:2000]: E.query(g, idx, u, v)
t = time.perf_counter()
for u, v in pairs: E.query(g, idx, u, v)
print("single query()", len(pairs) / (time.perf_counter() - t), "q/s")
