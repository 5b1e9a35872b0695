set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/qbench.py 2>&1 | tail -1
timeout 300 python - <<'PY'
import time, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W, _native as N
src, dst = W.rmat_edges(20, 8, 1)
g = E.DynamicGraph.from_edges(1 << 20, src, dst)
sp = N.ctypes.c_void_p(); N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
st = torch.cuda.ExternalStream(sp.value)
idx = E.build_index(g)
ts = []
for i in range(8):
    idx = None
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(st)
    idx = E.build_index(g)
    e1.record(st); t1 = time.perf_counter(); torch.cuda.synchronize()
    fx = N.ctypes.c_float(); N.call("dbl_last_timings", g.handle, N.ctypes.byref(fx), None, None)
    ts.append((e0.elapsed_time(e1), fx.value, (t1 - t0) * 1e3))
for t in ts[2:]: print("event %.4f ms  lib-span %.4f ms  host-call %.4f ms" % t)
PY
