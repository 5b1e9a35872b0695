"""e2e of a 1M-query batch from pinned host memory through dbl_query (zero-copy), as bench.py times it."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W, _native as N
n = 1 << 20
src, dst = W.rmat_edges(20, 8, 1)
g = E.DynamicGraph.from_edges(n, src, dst)
idx = E.build_index(g)
B = 1_000_000
qu, qv = W.uniform_queries(n, B, 2)
hu = torch.from_numpy(qu.view(np.int32)).pin_memory(); hv = torch.from_numpy(qv.view(np.int32)).pin_memory()
hc = torch.empty(B, dtype=torch.uint8).pin_memory()
hvis = torch.empty(B, dtype=torch.int32).pin_memory()
flags = E.DEFAULT_FLAGS.bits()
ref, _ = E.query_codes(g, idx, qu, qv, with_visited=False)
out = []
for vis in (False, True):
    fn = lambda: N.call("dbl_query", idx.handle, g.handle, N.ptr(hu), N.ptr(hv), B, flags, N.ptr(hc),
                        N.ptr(hvis) if vis else None, N.MEM_HOST)
    for _ in range(5): fn()
    assert np.array_equal(hc.numpy(), ref)
    ts = []
    for _ in range(30):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    out.append(f"{'codes+visited' if vis else 'codes'} {B / statistics.mean(ts) / 1e9:.3f} G q/s ({statistics.mean(ts)*1e6:.0f} us)")
print(" | ".join(out))
