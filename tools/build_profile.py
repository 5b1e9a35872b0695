"""Label-build timing on a device-generated R-MAT graph (cfg2 / cfg5 shapes).

  python tools/build_profile.py --scale 26 --ef 16 --k 256          # event-timed builds
  python tools/build_profile.py --scale 26 --ef 16 --k 256 --once   # one build (for ncu)

Prints one JSON line: mean/min build ms over --reps builds (engine stream, CUDA
events; the previous index freed first) and the executed-work counters of an
instrumented build.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_09441_b200 as E  # noqa: E402
from paper_2101_09441_b200 import _native as N  # noqa: E402
from paper_2101_09441_b200 import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ef", type=int, default=8)
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--kp", type=int, default=64)
    ap.add_argument("--seed", type=int, default=55)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--once", action="store_true")
    a = ap.parse_args()
    s, d = W.rmat_edges_device(a.scale, a.ef, a.seed)
    g = E.DynamicGraph.from_edges(1 << a.scale, s, d)
    del s, d
    cfg = E.IndexConfig(k=a.k, k_prime=a.kp)
    torch.cuda.synchronize()
    if a.once:
        idx = E.build_index(g, cfg)
        torch.cuda.synchronize()
        print(json.dumps({"scale": a.scale, "once": True}))
        return
    sp = N.ctypes.c_void_p()
    N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    idx, ts = E.build_index(g, cfg), []
    for _ in range(a.reps):
        idx = None
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        idx = E.build_index(g, cfg)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ref = idx
    idx = None
    N.call("dbl_graph_instrument", g.handle, 1)
    idx = E.build_index(g, cfg)
    bw = N.BuildWorkC()
    N.call("dbl_build_work_stats", g.handle, N.ctypes.byref(bw))
    N.call("dbl_graph_instrument", g.handle, 0)
    same = idx.labels_equal(ref)
    work = {f: int(getattr(bw, f)) for f, _ in N.BuildWorkC._fields_}
    print(json.dumps({"scale": a.scale, "ef": a.ef, "n": g.vertex_count, "m": g.edge_count, "k": a.k,
                      "k_prime": a.kp, "build_ms": ts, "mean_ms": sum(ts) / len(ts), "min_ms": min(ts),
                      "instrumented_equal": bool(same), "work": work}))


if __name__ == "__main__":
    main()
