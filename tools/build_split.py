"""Replicated vs word-sharded label build, measured on one GPU.

For N = 2, 4, 8 ranks: the slowest rank's share of the word-sharded build
(dbl_index_build_words on its round-robin words, after the shared metadata
step), the pack and unpack of the word slabs, and the allgather volume; the
replicated build is one full build.  The NVLink allgather is modelled at
--nvlink-gbs per GPU (received bytes / bandwidth; NCCL all_gather on
NVSwitch moves (N-1)/N of the gathered slab into every GPU).

    python tools/build_split.py [--scale 20 --ef 8 --k 64] [--nvlink-gbs 700]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_09441_b200 as E  # noqa: E402
from paper_2101_09441_b200 import _native as N  # noqa: E402
from paper_2101_09441_b200 import parallel as P  # noqa: E402
from paper_2101_09441_b200 import workload as W  # noqa: E402


def timed(stream, fn, reps=5):
    ts = []
    for i in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    return statistics.mean(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ef", type=int, default=8)
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--kp", type=int, default=64)
    ap.add_argument("--nvlink-gbs", type=float, default=700.0)
    a = ap.parse_args()
    n = 1 << a.scale
    if a.scale <= 22:
        src, dst = W.rmat_edges(a.scale, a.ef, 1)
    else:
        src, dst = W.rmat_edges_device(a.scale, a.ef, 55)
    g = E.DynamicGraph.from_edges(n, src, dst)
    del src, dst
    cfg = E.IndexConfig(k=a.k, k_prime=a.kp)
    sp = N.ctypes.c_void_p()
    N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    full = [None]

    def build():
        full[0] = None
        full[0] = E.build_index(g, cfg)
    t_full = timed(stream, build)
    ref = full[0]
    idx = P.create_index(g, cfg)
    eng = P.DeviceWordEngine(g, idx)
    rw = eng.rw
    t_create = timed(stream, lambda: P.create_index(g, cfg))
    out = {"n": n, "m": g.edge_count, "k": a.k, "k_prime": a.kp, "record_words": rw,
           "replicated_build_ms": t_full, "create_ms": t_create, "nvlink_gbs_model": a.nvlink_gbs, "ranks": {}}
    for world in (2, 4, 8):
        plan = P.plan_words(rw, world)
        shares = []
        for words in plan:
            if not words:
                continue
            shares.append(timed(stream, lambda w=words: eng.build_words(w), reps=3))
        maxw = max(len(p) for p in plan)
        slab = eng.empty_slab(maxw)
        gathered = eng.empty_slab(maxw * world)
        t_pack = timed(stream, lambda: eng.pack(plan[0], slab), reps=3)
        t_unpack = timed(stream, lambda: [eng.unpack(plan[r], gathered[r * maxw * n:(r + 1) * maxw * n])
                                          for r in range(1, world) if plan[r]], reps=3)
        recv = (world - 1) * maxw * n * 8
        t_ag = recv / (a.nvlink_gbs * 1e9) * 1e3
        total = t_create + max(shares) + t_pack + t_ag + t_unpack
        out["ranks"][world] = {"words_per_rank": maxw, "idle_ranks": sum(1 for p in plan if not p),
                               "slowest_share_ms": max(shares), "pack_ms": t_pack, "unpack_ms": t_unpack,
                               "allgather_bytes_per_gpu": recv, "allgather_ms_model": t_ag,
                               "sharded_total_ms": total, "replicated_ms": t_full,
                               "faster": "replicated" if t_full <= total else "words"}
        del slab, gathered
    # the sharded exchange itself reproduces the full build (in-process check)
    idx2 = P.create_index(g, cfg)
    eng2 = P.DeviceWordEngine(g, idx2)
    eng2.build_words(list(range(rw)))
    out["words_build_equals_full"] = bool(idx2.labels_equal(ref))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
