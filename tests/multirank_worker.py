"""One rank of the multi-rank GPU tests (tests/test_multirank.py).

Every rank runs on cuda:0 with the gloo backend (NCCL refuses two ranks on
one device); the ranks' kernels never wait on one another -- the only
exchange is gloo's host-side allgather -- so sharing one GPU is safe
(B200_PROFILING.md: only kernels that wait on other ranks must not share).

    python tests/multirank_worker.py RANK WORLD PORT OUT.json
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, world, port, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2101_09441_b200 as E
    from paper_2101_09441_b200 import parallel as P
    from paper_2101_09441_b200 import workload as W
    from oracle import oracle as O

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    res = {"rank": rank, "ok": True, "checks": {}}
    try:
        n = 1 << 12
        src, dst = W.rmat_edges(12, 8, seed=5)
        g = E.DynamicGraph.from_edges(n, src, dst, device=0)
        og = O.OracleGraph(n, src, dst)
        for k, kp in ((64, 64), (128, 64), (256, 64)):
            cfg = E.IndexConfig(k=k, k_prime=kp)
            full = E.build_index(g, cfg)
            sh = P.build_index_distributed(g, cfg, rank, world, mode="words")
            eq = bool(sh.labels_equal(full))
            oidx = og.build(k, kp, threads=2)
            w = sh.export_words()
            orc = all(np.array_equal(w[f], getattr(oidx, f)) for f in ("dl_in", "dl_out", "bl_in", "bl_out"))
            res["checks"][f"words_k{k}"] = {"equal_full": eq, "equal_oracle": bool(orc)}
            res["ok"] &= eq and orc
        idx = E.build_index(g)
        qu, qv = W.uniform_queries(n, 30_001, seed=6)
        whole, _ = E.query_codes(g, idx, qu, qv, with_visited=False)
        split = P.query_batch_split(g, idx, qu, qv, rank, world, gather=True)
        qeq = bool(np.array_equal(split, whole))
        res["checks"]["query_split"] = qeq
        res["ok"] &= qeq
        dist.barrier()
    except Exception as e:  # reported to the test, which fails on it
        res["ok"] = False
        res["error"] = repr(e)
    finally:
        with open(out, "w") as f:
            json.dump(res, f)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
