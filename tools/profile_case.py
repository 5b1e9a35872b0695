"""Small fixed workload for ncu captures (cfg2 shape: R-MAT 2^20, d = 8).

Builds the graph and index, runs the 1M uniform query batch three times and
one 100k insertion batch.  Used as:
  python tools/profile_case.py && ncu ... python tools/profile_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2101_09441_b200 as E  # noqa: E402
from paper_2101_09441_b200 import workload as W  # noqa: E402

scale = int(os.environ.get("DBL_SCALE", 20))
n = 1 << scale
src, dst = W.rmat_edges(scale, 8, 1)
g = E.DynamicGraph.from_edges(n, src, dst)
idx = E.build_index(g)
idx = E.build_index(g)
qu, qv = W.uniform_queries(n, 1_000_000, 2)
import torch  # noqa: E402
du = torch.from_numpy(qu.view(np.int32)).cuda()   # device-resident 1M batch, as bench.py times it
dv = torch.from_numpy(qv.view(np.int32)).cuda()
for _ in range(3):
    codes, _ = E.query_codes(g, idx, du, dv)
codes = codes.cpu().numpy()
iu, iv = W.gen_insert_workload(src, dst, n, 100_000, 50)
st = E.insert_edges(g, idx, iu, iv)
print("ok", g.edge_count, int(np.count_nonzero(codes >= 5)), st)
