"""e2e (pinned host in/out) timing of dbl_query for one 1M-query cfg2 batch:
wall time per call (the API syncs), median of 30, codes checked against the
device-resident path."""
import os, sys, time, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W, _native as N
n = 1 << 20
src, dst = W.rmat_edges(20, 8, 1)
g = E.DynamicGraph.from_edges(n, src, dst)
idx = E.build_index(g)
B = int(os.environ.get("E2E_BATCH", 1_000_000))
qu, qv = W.uniform_queries(n, B, 2)
hu = torch.from_numpy(qu.view(np.int32)).pin_memory(); hv = torch.from_numpy(qv.view(np.int32)).pin_memory()
hc = torch.empty(B, dtype=torch.uint8).pin_memory()
hvis = torch.empty(B, dtype=torch.int32).pin_memory()
ref, _ = E.query_codes(g, idx, torch.from_numpy(qu.view(np.int32)).cuda(), torch.from_numpy(qv.view(np.int32)).cuda())
ref = ref.cpu().numpy()
flags = E.DEFAULT_FLAGS.bits()
out = {}
for with_vis in (False, True):
    ts = []
    for i in range(33):
        t0 = time.perf_counter()
        N.call("dbl_query", idx.handle, g.handle, N.ptr(hu), N.ptr(hv), B, flags, N.ptr(hc),
               N.ptr(hvis) if with_vis else None, N.MEM_HOST)
        t1 = time.perf_counter()
        if i >= 3:
            ts.append(t1 - t0)
    assert np.array_equal(hc.numpy(), ref)
    out["with_visited" if with_vis else "codes"] = round(B / statistics.median(ts) / 1e9, 3)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("DBL_")}, "Gq_s": out}))

# component timings (wall, median of 20): torch H2D copies of the pairs, the
# device-resident query, and both
du = torch.empty(B, dtype=torch.int32, device="cuda"); dv = torch.empty_like(du)
dc = torch.empty(B, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def med(fn, k=20):
    ts = []
    for i in range(k + 3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        if i >= 3: ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts) * 1e6, 1)
def copies1():
    du.copy_(hu, non_blocking=True); dv.copy_(hv, non_blocking=True)
def copies2():
    with torch.cuda.stream(s1): du.copy_(hu, non_blocking=True)
    with torch.cuda.stream(s2): dv.copy_(hv, non_blocking=True)
def kern():
    N.call("dbl_query_async", idx.handle, g.handle, N.ptr(du), N.ptr(dv), B, flags, N.ptr(dc), None)
print(json.dumps({"us": {"h2d_1stream": med(copies1), "h2d_2streams": med(copies2), "kernel_async": med(kern),
                        "is_pinned": bool(hu.is_pinned())}}))
