"""One cfg2 label build after a warm-up build (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W
scale = int(os.environ.get("DBL_SCALE", 20))
src, dst = W.rmat_edges(scale, 8, 1)
g = E.DynamicGraph.from_edges(1 << scale, src, dst)
idx = E.build_index(g)
idx = None
idx = E.build_index(g)
print("ok")
