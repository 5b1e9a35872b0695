"""A/B timing of the query batch with and without the label digest.

    DBL_LIB_PATH=... python tools/digest_ab.py [--scales 20 22 24] [--tag name]

Per scale (R-MAT 2^s, d = 8, device generator, k = k' = 64): the build time,
then 1M and 16M uniform batches, each timed with CUDA events on the engine
stream after a 256 MB L2-flushing write (as bench.py times), plus the same
1M batch back to back without a flush (steady-state serving), and an md5 of
the codes so two library variants can be checked for identical answers.
"""
import argparse
import hashlib
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_09441_b200 as E  # noqa: E402
from paper_2101_09441_b200 import _native as N  # noqa: E402
from paper_2101_09441_b200 import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scales", type=int, nargs="+", default=[20, 22, 24])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("DBL_LIB_PATH", "product")))
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for scale in a.scales:
        n = 1 << scale
        s, d = W.rmat_edges_device(scale, 8, 24)
        g = E.DynamicGraph.from_edges(n, s, d)
        del s, d
        sp = N.ctypes.c_void_p()
        N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
        stream = torch.cuda.ExternalStream(sp.value, device=dev)
        bms = []
        idx = None
        for rep in range(4):
            idx = None
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            idx = E.build_index(g)
            e1.record(stream)
            torch.cuda.synchronize()
            if rep:
                bms.append(e0.elapsed_time(e1))
        flags = E.DEFAULT_FLAGS.bits()
        out = {"tag": a.tag, "scale": scale, "build_ms": statistics.median(bms)}
        for cnt in (1 << 20, 16 << 20):
            qu, qv = W.uniform_queries(n, cnt, 7)
            du = torch.from_numpy(qu.view(np.int32)).to(dev)
            dv = torch.from_numpy(qv.view(np.int32)).to(dev)
            codes = torch.empty(cnt, dtype=torch.uint8, device=dev)
            for fl in (True, False):
                if cnt > (1 << 20) and not fl:
                    continue
                ms = []
                with torch.cuda.stream(stream):
                    for i in range(3 + a.reps):
                        if fl:
                            flush.fill_(1)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        N.call("dbl_query_async", idx.handle, g.handle, N.ptr(du), N.ptr(dv), cnt, flags,
                               N.ptr(codes), None)
                        e1.record(stream)
                        e1.synchronize()
                        if i >= 3:
                            ms.append(e0.elapsed_time(e1))
                N.call("dbl_sync", g.handle)
                key = f"q{cnt >> 20}M" + ("_flushed" if fl else "_warm")
                med = statistics.median(ms)
                out[key + "_us"] = round(med * 1e3, 2)
                out[key + "_Gqps"] = round(cnt / med / 1e6, 2)
            c = codes.cpu().numpy()
            out[f"q{cnt >> 20}M_md5"] = hashlib.md5(c.tobytes()).hexdigest()[:12]
            out[f"q{cnt >> 20}M_hist"] = np.bincount(c, minlength=7).tolist()
        print(json.dumps(out), flush=True)
        del idx, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
