"""Where query_batch(g, idx, (u, v)) on pageable numpy arrays spends its time (cfg2, 1M pairs)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W, _native as N
n = 1 << 20
src, dst = W.rmat_edges(20, 8, 1)
g = E.DynamicGraph.from_edges(n, src, dst)
idx = E.build_index(g)
qu, qv = W.uniform_queries(n, 1_000_000, 2)
codes = np.zeros(len(qu), np.uint8)
vis = np.zeros(len(qu), np.uint32)
flags = E.DEFAULT_FLAGS.bits()


def t(fn, reps=15):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts) * 1e6, 1)


print("dbl_query pageable, codes+visited  us:", t(lambda: N.call("dbl_query", idx.handle, g.handle, N.ptr(qu), N.ptr(qv), len(qu), flags, N.ptr(codes), N.ptr(vis), N.MEM_HOST)))
print("dbl_query pageable, codes only     us:", t(lambda: N.call("dbl_query", idx.handle, g.handle, N.ptr(qu), N.ptr(qv), len(qu), flags, N.ptr(codes), None, N.MEM_HOST)))
print("query_codes(numpy)                 us:", t(lambda: E.query_codes(g, idx, qu, qv)))
print("query_batch(g, idx, (u, v))        us:", t(lambda: E.query_batch(g, idx, (qu, qv))))
print("np.copy of 8 MB of pairs           us:", t(lambda: (qu.copy(), qv.copy())))
