"""One cfg3-shaped (R-MAT 2^22, d = 8) 1M-query batch on device-resident pairs,
after a warm-up batch (for ncu captures of the label kernel beyond L2 size)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import run_configs as R
import numpy as np
E, torch, W = R.E, R.torch, R.W
g = R.device_graph(22, 8, 38)
idx = E.build_index(g)
qu, qv = W.uniform_queries(g.vertex_count, 1_000_000, 48)
du = torch.from_numpy(qu.view(np.int32)).cuda(); dv = torch.from_numpy(qv.view(np.int32)).cuda()
E.query_codes(g, idx, du, dv)
E.query_codes(g, idx, du, dv)
print("ok")
