"""cfg4-style insertion timing: R-MAT 2^SCALE d=8, 3 batches of 100k edges (device inputs)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W
scale = int(os.environ.get("DBL_SCALE", 20))
n = 1 << scale
src, dst = W.rmat_edges(scale, 8, 1)
g = E.DynamicGraph.from_edges(n, src, dst)
idx = E.build_index(g)
prev = None
for b in range(int(os.environ.get("DBL_BATCHES", 3))):
    iu, iv = W.gen_insert_workload(src, dst, n, 100_000, 50 + b, exclude=prev)
    prev = (iu, iv) if prev is None else (np.concatenate([prev[0], iu]), np.concatenate([prev[1], iv]))
    du = torch.from_numpy(iu.view(np.int32)).cuda(); dv = torch.from_numpy(iv.view(np.int32)).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = E.insert_edges(g, idx, du, dv)
    dt = time.perf_counter() - t0
    print(f"batch {b}: {dt*1e3:.2f} ms  {st.inserted/dt/1e6:.2f} M edges/s  {st}", flush=True)
