"""Wall time of one synchronous dbl_query call for tiny batches (API + launch
+ sync overhead), pinned host and device buffers."""
import os, sys, time, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W, _native as N
n = 1 << 20
src, dst = W.rmat_edges(20, 8, 1)
g = E.DynamicGraph.from_edges(n, src, dst)
idx = E.build_index(g)
flags = E.DEFAULT_FLAGS.bits()
out = {}
for B in (1, 1024, 1 << 16):
    qu, qv = W.uniform_queries(n, B, 2)
    hu = torch.from_numpy(qu.view(np.int32)).pin_memory(); hv = torch.from_numpy(qv.view(np.int32)).pin_memory()
    hc = torch.empty(B, dtype=torch.uint8).pin_memory()
    du, dv = hu.cuda(), hv.cuda(); dc = torch.empty(B, dtype=torch.uint8, device="cuda")
    for name, args in (("host", (hu, hv, hc, N.MEM_HOST)), ("device", (du, dv, dc, N.MEM_DEVICE))):
        a, b, c, mem = args
        ts = []
        for i in range(60):
            t0 = time.perf_counter()
            N.call("dbl_query", idx.handle, g.handle, N.ptr(a), N.ptr(b), B, flags, N.ptr(c), None, mem)
            ts.append(time.perf_counter() - t0)
        out[f"{name}_{B}"] = round(statistics.median(ts[10:]) * 1e6, 1)
print(json.dumps({"us_per_call": out}))
