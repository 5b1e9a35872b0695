"""Quick timing of the cfg2 hot path for experiments (no parity assertions).

    DBL_LIB_PATH=... python tools/qbench.py [--scale 20] [--reps 30]

Prints one line: step / kernel medians of the 1M uniform query batch (L2
flushed before each), the label build (total and fixpoint), and a 100k-edge
insertion batch.  Used to compare library variants built with
paper_2101_09441_b200.build.build_variant; bench.py is the measurement of record.
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_09441_b200 as E  # noqa: E402
from paper_2101_09441_b200 import _native as N  # noqa: E402
from paper_2101_09441_b200 import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--novis", action="store_true", help="codes only (visited = NULL)")
    ap.add_argument("--plain", action="store_true", help="no per-launch library events (as bench.py times)")
    a = ap.parse_args()
    n = 1 << a.scale
    src, dst = W.rmat_edges(a.scale, 8, seed=1)
    g = E.DynamicGraph.from_edges(n, src, dst)
    if not a.plain:
        N.call("dbl_graph_instrument", g.handle, 1)   # per-launch events for label_us
    sp = N.ctypes.c_void_p()
    N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    bt, ft = [], []
    idx = None
    for i in range(6):
        idx = None
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        idx = E.build_index(g)
        e1.record(stream)
        torch.cuda.synchronize()
        fx = N.ctypes.c_float()
        N.call("dbl_last_timings", g.handle, N.ctypes.byref(fx), None, None)
        if i:
            bt.append(e0.elapsed_time(e1))
            ft.append(fx.value)
    qu_h, qv_h = W.uniform_queries(n, a.batch, seed=2)
    qu = torch.from_numpy(qu_h.view(np.int32)).cuda()
    qv = torch.from_numpy(qv_h.view(np.int32)).cuda()
    codes = torch.empty(a.batch, dtype=torch.uint8, device="cuda")
    vis = torch.empty(a.batch, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flags = E.DEFAULT_FLAGS.bits()
    step, kern, lab = [], [], []
    tl, tb = N.ctypes.c_float(), N.ctypes.c_float()
    with torch.cuda.stream(stream):
        for i in range(a.reps + 3):
            flush.fill_(1)
            flush2.max()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            N.call("dbl_query_async", idx.handle, g.handle, N.ptr(qu), N.ptr(qv), a.batch, flags,
                   N.ptr(codes), None if a.novis else N.ptr(vis))
            e1.record(stream)
            e1.synchronize()
            N.call("dbl_last_timings", g.handle, None, N.ctypes.byref(tl), N.ctypes.byref(tb))
            if i >= 3:
                step.append(e0.elapsed_time(e1))
                kern.append(tl.value + tb.value)
                lab.append(tl.value)
    c = codes.cpu().numpy()
    vv = vis.cpu().numpy()
    import hashlib
    chash = hashlib.sha1(c.tobytes() + (b"" if a.novis else vv.tobytes())).hexdigest()[:12]
    iu, iv = W.gen_insert_workload(src, dst, n, 100_000, 50)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = E.insert_edges(g, idx, iu, iv)
    ins = time.perf_counter() - t0
    print(json.dumps({
        "step_us": round(1e3 * statistics.mean(step), 2), "kernel_us": round(1e3 * statistics.mean(kern), 2),
        "label_us": round(1e3 * statistics.mean(lab), 2),
        "Gq_s": round(a.batch / statistics.mean(step) / 1e6, 2),
        "build_ms": round(statistics.mean(bt), 4), "fixpoint_ms": round(statistics.mean(ft), 4),
        "insert_edges_s": round(st.inserted / ins / 1e6, 1),
        "unanswered": int(np.count_nonzero(c > 6)), "bfs_frac": float(np.mean((c >= 5) & (c <= 6))),
        "codes_sha1": chash}))


if __name__ == "__main__":
    main()
