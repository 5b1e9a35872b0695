"""Fixed cost of one insert_edges batch: tiny graph + tiny batch (GPU work ~0),
so the time is host enqueue + launch + sync overhead; plus a 100k batch on cfg2
for comparison.  DBL_TRACE builds print per-phase host times."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W

for scale, batch in ((10, 100), (20, 100), (20, 100_000)):
    n = 1 << scale
    src, dst = W.rmat_edges(scale, 8, 1)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g)
    prev = None
    ts = []
    for b in range(8):
        iu, iv = W.gen_insert_workload(src, dst, n, batch, 50 + b, exclude=prev)
        prev = (iu, iv) if prev is None else (np.concatenate([prev[0], iu]), np.concatenate([prev[1], iv]))
        du = torch.from_numpy(iu.view(np.int32)).cuda(); dv = torch.from_numpy(iv.view(np.int32)).cuda()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        E.insert_edges(g, idx, du, dv)
        ts.append(time.perf_counter() - t0)
    print(f"scale {scale} batch {batch}: median {statistics.median(ts[2:])*1e6:.0f} us  (all: {[round(t*1e6) for t in ts]})")
