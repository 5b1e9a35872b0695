import sys, os
sys.path.insert(0, os.getcwd())
import paper_2101_09441_b200 as E
from paper_2101_09441_b200 import workload as W
src, dst = W.gen_random_graph(10_000, 5, seed=1)
g = E.DynamicGraph.from_edges(10_000, src, dst)
E.build_index(g)
E.build_index(g)
