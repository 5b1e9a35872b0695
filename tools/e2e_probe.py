"""e2e variants for a 1M-query batch from pinned host memory (experiment)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W, _native as N
n = 1 << 20
src, dst = W.rmat_edges(20, 8, 1)
g = E.DynamicGraph.from_edges(n, src, dst)
idx = E.build_index(g)
sp = N.ctypes.c_void_p(); N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
st = torch.cuda.ExternalStream(sp.value)
B = 1_000_000
qu, qv = W.uniform_queries(n, B, 2)
hu = torch.from_numpy(qu.view(np.int32)).pin_memory(); hv = torch.from_numpy(qv.view(np.int32)).pin_memory()
hc = torch.empty(B, dtype=torch.uint8).pin_memory()
du = torch.empty(B, dtype=torch.int32, device="cuda"); dv = torch.empty_like(du)
dc = torch.empty(B, dtype=torch.uint8, device="cuda")
flags = E.DEFAULT_FLAGS.bits()
def zc():
    N.call("dbl_query", idx.handle, g.handle, N.ptr(hu), N.ptr(hv), B, flags, N.ptr(hc), None, N.MEM_HOST)
def dma(chunks):
    with torch.cuda.stream(st):
        c = B // chunks
        for k in range(chunks):
            lo, hi = k * c, (k + 1) * c if k < chunks - 1 else B
            du[lo:hi].copy_(hu[lo:hi], non_blocking=True); dv[lo:hi].copy_(hv[lo:hi], non_blocking=True)
            N.call("dbl_query_async", idx.handle, g.handle, N.ptr(du[lo:hi]), N.ptr(dv[lo:hi]), hi - lo, flags,
                   N.ptr(dc[lo:hi]), None)
            hc[lo:hi].copy_(dc[lo:hi], non_blocking=True)
    st.synchronize()
for name, fn in (("zero-copy", zc), ("dma x1", lambda: dma(1)), ("dma x2", lambda: dma(2)), ("dma x4", lambda: dma(4))):
    for _ in range(3): fn()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    print(f"{name:10s} {B / statistics.mean(ts) / 1e9:.2f} G q/s  ({statistics.mean(ts)*1e6:.0f} us)")
