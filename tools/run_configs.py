"""Run BASELINE.json configs 1-5 on one GPU with parity checks.

    python tools/run_configs.py [--cfg 1,3,4,5] [--out profiles/r01_configs.json]

Config 2 is bench.py's workload.  Parity evidence per config:
  cfg1  full: labels, 100k query codes, 1000 inserts vs the oracle (C port of
        the reference; the inputs are the reference's own generators).
  cfg3  per degree: GPU verify_labels (union fixpoint); bit columns of 8
        landmarks + 8 in/out buckets vs CPU floods over the exported CSR/CSC;
        200k query codes vs the CSR oracle on the GPU's labels; full oracle
        label parity for d <= 8.
  cfg4  after every batch: labels == GPU rebuild_index on frozen metadata and
        verify_labels; after batches 1 and 10: labels and 1M query codes vs the
        oracle (base build + sequential insert_edge loop).
  cfg5  verify_labels; bit columns of 4 landmarks + 2 buckets per direction vs
        CPU floods; 200k sampled query codes vs the CSR oracle.
Large synthetic graphs are generated on the GPU (dbl_rmat_generate).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_09441_b200 as E  # noqa: E402
from paper_2101_09441_b200 import _native as N  # noqa: E402
from paper_2101_09441_b200 import workload as W  # noqa: E402
from oracle import oracle as O  # noqa: E402

CORES = os.cpu_count() or 1
FAMS = ("dl_in", "dl_out", "bl_in", "bl_out")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def timed(fn, reps=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return out, (time.perf_counter() - t0) / reps


def build_time(g, cfg=None, reps=3):
    """Device time of E.build_index on the engine's stream (CUDA events), the
    previous index freed and the device idle before each rep -- the bench's
    definition of label-build seconds.  Returns (index, mean seconds)."""
    sp = N.ctypes.c_void_p()
    N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    idx, ts = None, []
    for _ in range(reps):
        idx = None
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        idx = E.build_index(g, cfg) if cfg is not None else E.build_index(g)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return idx, sum(ts) / len(ts)


def query_rate(g, idx, qu, qv, reps=5):
    """query_qps: device-resident batch timed with CUDA events on the engine
    stream after a 256 MB L2-flushing write (the bench's definition; codes +
    visited written); api_qps: the
    same batch through E.query_codes (allocation, call and sync included)."""
    du = torch.from_numpy(qu.view(np.int32)).cuda()
    dv = torch.from_numpy(qv.view(np.int32)).cuda()
    E.query_codes(g, idx, du, dv)
    (codes, vis), t_api = timed(lambda: E.query_codes(g, idx, du, dv), reps)
    qc = np.zeros(8, np.uint32)
    N.call("dbl_query_counters", g.handle, N.ptr(qc))
    c = codes.cpu().numpy()
    sp = N.ctypes.c_void_p()
    N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    dc = torch.empty(len(qu), dtype=torch.uint8, device="cuda")
    dvis = torch.empty(len(qu), dtype=torch.int32, device="cuda")
    flags = E.DEFAULT_FLAGS.bits()
    ts = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for i in range(reps + 1):
        flush.fill_(1)   # L2 flushed before every timed batch, as bench.py times
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        N.call("dbl_query_async", idx.handle, g.handle, N.ptr(du), N.ptr(dv), len(qu), flags, N.ptr(dc), N.ptr(dvis))
        e1.record(stream)
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1) / 1e3)
    assert np.array_equal(dc.cpu().numpy(), c)
    t = sum(ts) / len(ts)
    return c, len(qu) / t, {"api_qps": len(qu) / t_api, "rho": float(np.mean(c < 5)),
                            "bfs_fraction": float(np.mean(c >= 5)), "hard_path_queries": int(qc[0])}


def label_columns_check(g, idx, n_lm=8, n_bk=8, seed=0):
    """Sampled bit columns vs CPU floods (labels.py:247-260) over exported adjacency.

    Each column is one reference-style single-bit flood (oracle csr_flood);
    the floods run on a thread pool (the C oracle releases the GIL).
    """
    from concurrent.futures import ThreadPoolExecutor
    w = idx.export_words()
    fptr, fcol = g.adjacency(False)
    rptr, rcol = g.adjacency(True)
    fptr, rptr = fptr.astype(np.uint64), rptr.astype(np.uint64)
    n = g.vertex_count
    rng = np.random.default_rng(seed)
    lms = np.array(idx.landmark_set.landmarks)
    jobs = []   # (family, bit, ptr, col, seeds)
    for i in (rng.choice(len(lms), min(n_lm, len(lms)), replace=False) if len(lms) else []):
        jobs.append(("dl_in", int(i), fptr, fcol, [lms[i]]))
        jobs.append(("dl_out", int(i), rptr, rcol, [lms[i]]))
    flags, bucket = idx.leaf_sets.flags, idx.leaf_sets.bucket_array
    kp = idx.config.k_prime
    for b in rng.choice(kp, min(n_bk, kp), replace=False):
        for side, fam, ptr, col in ((1, "bl_in", fptr, fcol), (2, "bl_out", rptr, rcol)):
            seeds = np.flatnonzero((flags & side) != 0)
            seeds = seeds[bucket[seeds] == b].astype(np.uint32)
            jobs.append((fam, int(b), ptr, col, seeds))

    def run(job):
        fam, bit, ptr, col, seeds = job
        reach = O.csr_flood(n, ptr, col, seeds)
        colv = (w[fam][:, bit // 64] >> np.uint64(bit % 64)) & np.uint64(1)
        return fam, bit, bool(np.array_equal(colv.astype(bool), reach))

    with ThreadPoolExecutor(max(1, min(CORES, 16))) as ex:
        res = list(ex.map(run, jobs))
    bad = [(f, b) for f, b, ok in res if not ok]
    assert not bad, f"label columns differ from the CPU floods: {bad[:5]}"
    per = {}
    for f, _, _ in res:
        per[f] = per.get(f, 0) + 1
    return {"columns": len(res), "per_family": per}


def csr_codes_check(g, idx, qu, qv, codes):
    fptr, fcol = g.adjacency(False)
    oc = O.csr_query_batch(g.vertex_count, fptr.astype(np.uint64), fcol, idx.config.k, idx.config.k_prime,
                           idx.export_words(), qu, qv, threads=CORES)
    assert np.array_equal(oc, codes), "query codes differ from the CSR oracle"
    return len(qu)


def device_graph(scale, ef, seed):
    s, d = W.rmat_edges_device(scale, ef, seed)
    g = E.DynamicGraph.from_edges(1 << scale, s, d)
    del s, d
    return g


# ------------------------------------------------------------------ cfg1 --

def cfg1():
    src, dst = W.gen_random_graph(10_000, 5, seed=1)
    qu, qv = W.gen_random_queries(10_000, 100_000, seed=2)
    g = E.DynamicGraph.from_edges(10_000, src, dst)
    E.build_index(g)
    idx, tb = build_time(g)
    codes, qps, st = query_rate(g, idx, qu, qv)
    og = O.OracleGraph(10_000, src, dst)
    oidx = og.build(64, 64, threads=CORES)
    w = idx.export_words()
    for f in FAMS:
        assert np.array_equal(w[f], getattr(oidx, f)), f
    oc, _ = og.query_batch(oidx, qu, qv, threads=CORES)
    assert np.array_equal(oc, codes)
    iu, iv = W.gen_insert_workload(src, dst, 10_000, 1000, seed=3)
    _, ti = timed(lambda: E.insert_edges(g, idx, iu, iv))
    for u, v in zip(iu.tolist(), iv.tolist()):
        og.insert_edge(oidx, u, v)
    w = idx.export_words()
    for f in FAMS:
        assert np.array_equal(w[f], getattr(oidx, f)), f
    return {"n": 10_000, "m": g.edge_count, "build_s": tb, "query_qps": qps, **st,
            "insert_edges_per_s": 1000 / ti, "parity": "labels + 100k codes + 1000 inserts == oracle (full)"}


# ------------------------------------------------------------------ cfg3 --

def cfg3(degrees=(2, 4, 8, 16, 32, 64), scale=22):
    out = []
    for d in degrees:
        torch.cuda.empty_cache()
        g = device_graph(scale, d, 30 + d)
        n = g.vertex_count
        E.build_index(g)
        idx, tb = build_time(g)
        fix = np.zeros(1, np.float32)
        qu, qv = W.uniform_queries(n, 1_000_000, 40 + d)
        codes, qps, st = query_rate(g, idx, qu, qv)
        rep = E.verify_labels(g, idx, exhaustive=False)
        assert rep.ok, rep.violations[:3]
        nq = csr_codes_check(g, idx, qu[:200_000], qv[:200_000], codes[:200_000])
        if d > 8:
            # every one of the 4 x 64 bit columns against its own reference-style
            # flood (labels.py:247-260) over the exported CSR: the full labels
            cols = label_columns_check(g, idx, n_lm=64, n_bk=64, seed=d)
            full = f"all {cols['columns']} bit columns equal single-bit CSR floods (labels.py:247-260)"
        else:
            cols = label_columns_check(g, idx, seed=d)
        if d <= 8:
            s, dd = g.edge_arrays()
            og = O.OracleGraph(n, s, dd)
            oidx = og.build(64, 64, threads=CORES)
            w = idx.export_words()
            for f in FAMS:
                assert np.array_equal(w[f], getattr(oidx, f)), f
            del og, oidx
            full = "all four families equal the oracle's"
        out.append({"degree": d, "n": n, "m": g.edge_count, "build_s": tb, "query_qps": qps, **st,
                    "parity": {"verify_fixpoint": True, "bit_columns": cols, "codes_vs_csr_oracle": nq,
                               "full_labels_vs_oracle": full}})
        log(json.dumps(out[-1]))
        del g, idx
    return out


# ------------------------------------------------------------------ cfg4 --

def cfg4(scale=22, batches=10, batch=100_000, check_at=(1, 10)):
    g = device_graph(scale, 8, 44)
    n = g.vertex_count
    idx = E.build_index(g)
    src, dst = g.edge_arrays()
    og = O.OracleGraph(n, src, dst)
    oidx = og.build(64, 64, threads=CORES)
    prev = None
    rows = []
    for b in range(1, batches + 1):
        iu, iv = W.gen_insert_workload(src, dst, n, batch, 100 + b, exclude=prev)
        prev = (iu, iv) if prev is None else (np.concatenate([prev[0], iu]), np.concatenate([prev[1], iv]))
        du = torch.from_numpy(iu.view(np.int32)).cuda()
        dv = torch.from_numpy(iv.view(np.int32)).cuda()
        st, ti = timed(lambda: E.insert_edges(g, idx, du, dv))
        qu, qv = W.uniform_queries(n, 1_000_000, 200 + b)
        codes, qps, qst = query_rate(g, idx, qu, qv)
        assert idx.labels_equal(E.rebuild_index(g, idx)), f"batch {b}: labels != rebuild"
        assert E.verify_labels(g, idx, exhaustive=False).ok
        for u, v in zip(iu.tolist(), iv.tolist()):
            og.insert_edge(oidx, u, v)
        oracle = False
        if b in check_at:
            w = idx.export_words()
            for f in FAMS:
                assert np.array_equal(w[f], getattr(oidx, f)), f"batch {b} {f}"
            oc, _ = og.query_batch(oidx, qu, qv, threads=CORES)
            assert np.array_equal(oc, codes), f"batch {b} codes"
            oracle = True
        rows.append({"batch": b, "inserted": st.inserted, "insert_s": ti, "edges_per_s": st.inserted / ti,
                     "labels_changed": st.labels_changed, "levels": st.levels, "delta_merged": st.delta_merged,
                     "query_qps": qps, **qst, "labels_eq_rebuild": True, "oracle_checked": oracle})
        log(json.dumps(rows[-1]))
    return {"n": n, "m_final": g.edge_count, "batches": rows}


# ------------------------------------------------------------------ cfg5 --

def cfg5(scale=26, ef=16, nq=64_000_000):
    g = device_graph(scale, ef, 55)
    n = g.vertex_count
    cfg = E.IndexConfig(k=256, k_prime=64)
    idx = E.build_index(g, cfg)
    idx = None
    idx, tb = build_time(g, cfg)
    rng = np.random.default_rng(56)
    qu = rng.integers(0, n, nq, dtype=np.uint32)
    qv = rng.integers(0, n, nq, dtype=np.uint32)
    codes, qps, st = query_rate(g, idx, qu, qv, reps=3)
    rep = E.verify_labels(g, idx, exhaustive=False)
    assert rep.ok, rep.violations[:3]
    cols = label_columns_check(g, idx, n_lm=256, n_bk=64, seed=5)   # every bit column: the full labels
    sample = rng.choice(nq, 200_000, replace=False)
    nchk = csr_codes_check(g, idx, qu[sample], qv[sample], codes[sample])
    return {"n": n, "m": g.edge_count, "k": 256, "k_prime": 64, "build_s": tb, "query_batch": nq,
            "query_qps": qps, **st,
            "parity": {"verify_fixpoint": True, "bit_columns": cols, "codes_vs_csr_oracle": nchk}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="1,3,4,5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_configs.json"))
    ap.add_argument("--scale3", type=int, default=22)
    ap.add_argument("--scale5", type=int, default=26)
    args = ap.parse_args()
    res = {}
    if os.path.exists(args.out):
        res = json.load(open(args.out))
    for c in args.cfg.split(","):
        t0 = time.perf_counter()
        if c == "1":
            res["cfg1"] = cfg1()
        elif c == "3":
            res["cfg3"] = cfg3(scale=args.scale3)
        elif c == "4":
            res["cfg4"] = cfg4()
        elif c == "5":
            res["cfg5"] = cfg5(scale=args.scale5)
        log(f"cfg{c} done in {time.perf_counter() - t0:.1f} s")
        res["host_cores"] = CORES
        json.dump(res, open(args.out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
