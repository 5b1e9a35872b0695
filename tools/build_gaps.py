"""Host wall time vs device (event) time of a cfg2 build, and the host time
of the build's enqueue alone (everything before the final sync is async)."""
import os, sys, time, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W, _native as N
n = 1 << 20
src, dst = W.rmat_edges(20, 8, 1)
g = E.DynamicGraph.from_edges(n, src, dst)
sp = N.ctypes.c_void_p(); N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
stream = torch.cuda.ExternalStream(sp.value)
idx = None
wall, dev = [], []
for i in range(12):
    idx = None
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    idx = E.build_index(g)
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    if i >= 2:
        wall.append((t1 - t0) * 1e3); dev.append(e0.elapsed_time(e1))
print(json.dumps({"wall_ms": round(statistics.mean(wall), 4), "device_ms": round(statistics.mean(dev), 4)}))
