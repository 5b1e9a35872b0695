"""cfg5 query-path experiment: build the 2^26 R-MAT index once, time the
64M-query batch, and print codes/visited digests so that variants selected by
environment toggles (DBL_NO_PIVOT_PRUNE, DBL_LEAN_WIDE, ...) run in separate
processes can be compared for bit-identical answers.

    python tools/cfg5_query.py [--scale 26] [--nq 64000000] [--label NAME]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import run_configs as R  # noqa: E402

E = R.E
torch = R.torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--nq", type=int, default=64_000_000)
    ap.add_argument("--label", default="")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--builds", type=int, default=1, help="builds before the timed one (warm allocations)")
    args = ap.parse_args()
    g = R.device_graph(args.scale, 16, 55)
    n = g.vertex_count
    for _ in range(args.builds - 1):
        E.build_index(g, E.IndexConfig(k=256, k_prime=64))
    idx, tb = R.build_time(g, E.IndexConfig(k=256, k_prime=64), reps=1)
    rng = np.random.default_rng(56)
    qu = rng.integers(0, n, args.nq, dtype=np.uint32)
    qv = rng.integers(0, n, args.nq, dtype=np.uint32)
    du = torch.from_numpy(qu.view(np.int32)).cuda()
    dv = torch.from_numpy(qv.view(np.int32)).cuda()
    E.query_codes(g, idx, du, dv)
    (codes, vis), t = R.timed(lambda: E.query_codes(g, idx, du, dv), args.reps)
    c = codes.cpu().numpy()
    v = vis.cpu().numpy() if vis is not None else np.zeros(0, np.uint32)
    qc = np.zeros(8, np.uint32)
    R.N.call("dbl_query_counters", g.handle, R.N.ptr(qc))
    print(json.dumps({"label": args.label, "n": n, "m": g.edge_count, "build_s": tb, "query_s": t, "Gq_s": args.nq / t / 1e9,
                      "bfs_fraction": float(np.mean(c >= 5)), "hard_path": int(qc[0]),
                      "visited_total": int(v.astype(np.uint64).sum()),
                      "codes_md5": hashlib.md5(c.tobytes()).hexdigest(),
                      "visited_md5": hashlib.md5(v.tobytes()).hexdigest()}), flush=True)


if __name__ == "__main__":
    main()
