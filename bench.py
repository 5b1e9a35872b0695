"""Benchmark: reach queries/s on a 1M-query batch (+ label build s, edge inserts/s).

BASELINE.json metric "reach queries/sec (1M-query batch) + label build sec and
edge-inserts/sec, 1/2/4/8 B200"; workload = configs[1]: directed R-MAT 2^20,
average out-degree 8, (a, b, c, d) = (.57, .19, .19, .05), duplicates
removed, seeded (numpy PCG64 seed 1, ids unpermuted); default IndexConfig
(k = k' = 64).

One step = one pass of the query hot path (K6 label check + K7 pruned-BFS
fallback) over a batch of 1M uniform random pairs resident in HBM; L2 is
flushed (256 MB write, then 256 MB read) before every timed step; each step
is bracketed by CUDA events on the engine's stream.  `e2e` times the same
batch through the public C-ABI call dbl_query with pinned HOST buffers (the
pairs cross PCIe host->device and the answer codes device->host inside the
timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Multi-GPU (torchrun, one rank per GPU; DBL_BENCH_GLOO=1 puts every rank on
cuda:0 over gloo, for testing the N > 1 code path on one GPU): the graph and
the labels are replicated -- each rank runs the whole label build, the
measured-faster mode -- and every rank answers its own 1M-query
batch (weak scaling, no collective on the query path); the word-sharded build
(NCCL allgather of label words) is timed beside it and checked equal.  The
`whole_box_2^24` block is the north_star's number: R-MAT 2^24, d = 8, 1M
uniform pairs per GPU, plus one 16M batch split across the GPUs.  Times are
the max over ranks.

--impl reference times the reference algorithm's CPU implementation on the
host cores instead: the oracle port (oracle/dbl_oracle.c, a restatement of the
Python reference, which cannot travel to the GPU box) on the same graph and
query batches, all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SCALE, EDGE_FACTOR, GRAPH_SEED = 20, 8, 1
BATCH = 1_000_000
METRIC = "reach queries/sec (1M-query batch)"
FAMS = ("dl_in", "dl_out", "bl_in", "bl_out")


def workload_name(scale: int) -> str:
    return (f"cfg2: directed R-MAT 2^{scale}, avg out-degree {EDGE_FACTOR}, a/b/c/d=.57/.19/.19/.05, dedup, "
            f"seed {GRAPH_SEED} (numpy PCG64, unpermuted ids); k=64 landmarks (product), k'=64 BL; "
            f"1M uniform random (u,v) pairs per step")


def bench_config(n: int, m: int, scale: int, world: int) -> dict:
    """The `config` of both arms (identical dicts, so the driver sees the same config)."""
    return {"workload": workload_name(scale), "n": n, "m": m, "queries_per_step": BATCH,
            "k": 64, "k_prime": 64,
            "l2": "flushed before every timed step (256 MB write, then 256 MB read so no dirty lines remain)",
            "parallelism": f"replicated graph+labels (each GPU builds), one 1M batch per GPU x{world}"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for nm, val in zip(names, p[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


# L2 request ceiling of a random 32-byte gather (8 CTAs/SM, 64 MB table, warm):
# 205.3 G requests/s, tools/ubench_gather.cu -> profiles/r01_ubench_gather.txt
L2_REQ_CEILING_G = 205.3


def ncu_l2req(kernel: str):
    """SM->L2 requests per launch of `kernel` from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_l2req.json")) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


def make_workload(rank: int, scale: int):
    from paper_2101_09441_b200 import workload as W
    src, dst = W.rmat_edges(scale, EDGE_FACTOR, GRAPH_SEED)
    n = 1 << scale
    qu, qv = W.uniform_queries(n, BATCH, 2 + 1000 * rank)
    return n, src, dst, qu, qv


# ------------------------------------------------------ algorithmic bytes --

def build_exec_bytes(w) -> dict:
    """Bytes of the build work the kernels actually executed (dbl_build_work_stats).

    prep: per vertex 4 row-pointer words (in- and out-degree) 16 B + score 8 B
    + leaf flag and bucket 5 B, + the seeded record when prep writes it;
    pivot reach: per sweep both directions' bitmaps (n/8 B each), per
    bottom-up test 2 row pointers (8 B), per neighbour probe a column id and
    a bitmap word (8 B); per top-down vertex 8 B and edge 8 B; the union pass
    5 B/vertex of metadata plus each touched record read and written (or every
    record written once in write mode); label fixpoint: 16 B per frontier item
    + 12 B per relaxed edge (SURVEY.md §8(d) unit costs).
    """
    n, R = w.n, w.record_bytes
    prep = n * (16 + 8 + 5) + (n * R if w.flags & 1 else 0)
    reach = (w.sweeps * 2 * n // 8 + 8 * w.bu_tests + 8 * w.bu_probes + 8 * w.td_vertices
             + 8 * w.td_edges + 5 * n)
    if w.flags & 2:
        reach += n * R
    elif w.flags & 4:
        reach += 2 * R * w.union_records
    fix = 16 * w.fix_items + 12 * w.fix_edges
    return {"prep": int(prep), "pivot_reach": int(reach), "fixpoint": int(fix),
            "total": int(prep + reach + fix)}


def digest_undecided(dig: np.ndarray, u: np.ndarray, v: np.ndarray) -> float:
    """Fraction of pairs (u != v) whose digests decide neither rule 1 nor rule 2
    under the default flags (query.cu digest_decide): these read both records."""
    du, dv = dig[u], dig[v]
    dl = du & (dv >> np.uint32(2)) & np.uint32(3)
    fi_u, fi_v = (du >> np.uint32(4)) & np.uint32(0x3FFF), (dv >> np.uint32(4)) & np.uint32(0x3FFF)
    blneg = ((fi_u & ~fi_v) | ((dv >> np.uint32(18)) & ~(du >> np.uint32(18)))) != 0
    decided = ((dl & np.uint32(1)) != 0) | ((dl == 0) & blneg) | (u == v)
    return float(1.0 - decided.mean())


def work_dict(w) -> dict:
    return {k: int(getattr(w, k)) for k, _ in w._fields_}


# ----------------------------------------------------------------- ours --

def run_ours(args, rank, world, local_rank, gloo):
    import torch
    import torch.distributed as dist

    import paper_2101_09441_b200 as E
    from paper_2101_09441_b200 import _native as N
    from paper_2101_09441_b200 import workload as W
    from paper_2101_09441_b200.parallel import build_index_distributed

    devi = 0 if gloo else local_rank
    torch.cuda.set_device(devi)
    dev = torch.device("cuda", devi)
    scale = args.scale
    n, src, dst, qu_h, qv_h = make_workload(rank, scale)
    g = E.DynamicGraph.from_edges(n, src, dst, device=devi)
    m = g.edge_count
    sp = N.ctypes.c_void_p()
    N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_ranks(x: float) -> float:
        return _max_over_ranks(torch, dist, world, x, gloo)

    def ev_pair():
        return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    # ---- label build (device time, CSR/CSC resident -> final AoS table)
    cfg = E.IndexConfig()
    # executed work of this build: one instrumented build (the pivot kernel
    # variant with work counters), not timed
    N.call("dbl_graph_instrument", g.handle, 1)
    idx = E.build_index(g, cfg)
    bw = N.BuildWorkC()
    N.call("dbl_build_work_stats", g.handle, N.ctypes.byref(bw))
    N.call("dbl_graph_instrument", g.handle, 0)
    exec_bytes = build_exec_bytes(bw)

    def timed_builds(mode: str, reps: int = 8) -> tuple[float, object]:
        ms, out = [], None
        for rep in range(reps):   # rep 0 warms the allocator cache; the previous index is dropped first
            out = None
            barrier()
            torch.cuda.synchronize()
            e0, e1 = ev_pair()
            e0.record(stream)
            out = build_index_distributed(g, cfg, rank, world, mode=mode)
            e1.record(stream)
            torch.cuda.synchronize()
            if rep:
                ms.append(e0.elapsed_time(e1))
        return max_ranks(statistics.mean(ms)), out

    idx = None
    build_ms_max, idx = timed_builds("replicated")
    want_cpu = rank == 0 and world == 1 and not args.no_cpu_baseline
    built_words = idx.export_words() if want_cpu else None   # checked against the oracle below
    fix_ms = N.ctypes.c_float()
    N.call("dbl_last_timings", g.handle, N.ctypes.byref(fix_ms), None, None)
    sharded = None
    if world > 1:
        sh_ms, sidx = timed_builds("words", reps=4)
        sharded = {"value_s": sh_ms / 1e3, "labels_equal_replicated": bool(sidx.labels_equal(idx)),
                   "mode": "word-sharded build + allgather of record words ("
                           + ("gloo, host-staged" if gloo else "NCCL over NVLink") + ")"}
        del sidx

    # SURVEY.md §8(d) level-synchronous work model (the work a plain
    # Jacobi fixpoint would do), reported beside the executed bytes
    rw = 2 * (idx.wdl + idx.wbl)
    V = np.zeros(rw, np.uint64)
    Ecnt = np.zeros(rw, np.uint64)
    L = np.zeros(rw, np.uint32)
    N.call("dbl_work_model", idx.handle, g.handle, N.ptr(V), N.ptr(Ecnt), N.ptr(L))
    rec_bytes = 8 * rw
    model_bytes = int(sum(16 * int(v) + 12 * int(e) for v, e in zip(V, Ecnt)) + n * (8 * rw + rec_bytes))

    # ---- queries: device-resident batch
    qu = torch.from_numpy(qu_h.view(np.int32)).to(dev)
    qv = torch.from_numpy(qv_h.view(np.int32)).to(dev)
    codes = torch.empty(BATCH, dtype=torch.uint8, device=dev)
    vis = torch.empty(BATCH, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flags = E.DEFAULT_FLAGS.bits()

    def l2_flush():
        # write 256 MB (evicts everything), then read 256 MB so the write-back of
        # the dirty flush lines happens here rather than inside the timed step
        flush.fill_(1)
        flush2.max()

    def step(u_t, v_t):
        N.call("dbl_query_async", idx.handle, g.handle, N.ptr(u_t), N.ptr(v_t), BATCH, flags,
               N.ptr(codes), N.ptr(vis))

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            l2_flush()
            step(qu, qv)
    N.call("dbl_sync", g.handle)
    c = codes.cpu().numpy()
    assert c.max() <= 6, "unanswered queries in the batch"
    rho = float(np.mean(c < 5))

    sampler = ClockSampler(devi)
    sampler.start()
    barrier()
    torch.cuda.synchronize()
    launches0 = N.kernel_launches()
    # a step is one launch (the query kernel; BFS stages are tail-launched
    # from the device only when needed) between the two events, so the step
    # time is also the kernel's event-timed duration used by the roofline
    step_ms = []
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            l2_flush()
            e0, e1 = ev_pair()
            e0.record(stream)
            step(qu, qv)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    barrier()
    launches = N.kernel_launches() - launches0
    qcnt = np.zeros(8, np.uint32)
    N.call("dbl_query_counters", g.handle, N.ptr(qcnt))
    total_ms = max_ranks(sum(step_ms))
    ms_per_step = total_ms / args.steps
    value = world * BATCH * args.steps / (total_ms / 1e3)
    assert np.array_equal(codes.cpu().numpy(), c), "codes changed between identical batches"

    # positives batch (cfg2's second query set), same measurement
    pu_h, pv_h = W.positive_queries(n, src, dst, BATCH, 3 + 1000 * rank)
    pu = torch.from_numpy(pu_h.view(np.int32)).to(dev)
    pv = torch.from_numpy(pv_h.view(np.int32)).to(dev)
    pos_ms = []
    with torch.cuda.stream(stream):
        for i in range(args.warmup + max(5, args.steps // 4)):
            l2_flush()
            e0, e1 = ev_pair()
            e0.record(stream)
            step(pu, pv)
            e1.record(stream)
            e1.synchronize()
            if i >= args.warmup:
                pos_ms.append(e0.elapsed_time(e1))
    N.call("dbl_sync", g.handle)
    pos_codes = codes.cpu().numpy()
    pos_rho = float(np.mean(pos_codes < 5))
    pos_total = max_ranks(sum(pos_ms))
    pos_qps = world * BATCH * len(pos_ms) / (pos_total / 1e3)

    # ---- e2e through the public C-ABI call with pinned host buffers: H2D of
    # the pairs and D2H of the answer codes (the step's result) every step
    hu = torch.from_numpy(qu_h.view(np.int32)).pin_memory()
    hv = torch.from_numpy(qv_h.view(np.int32)).pin_memory()
    hc = torch.empty(BATCH, dtype=torch.uint8).pin_memory()
    hvis = torch.empty(BATCH, dtype=torch.int32).pin_memory()

    def e2e_run(with_visited: bool) -> float:
        # the C-ABI call as a host program makes it: bound once, then called
        # per batch (each call copies the pairs in and the codes out)
        fn = N.lib().dbl_query
        call_args = (idx.handle, g.handle, N.ptr(hu), N.ptr(hv), BATCH, flags, N.ptr(hc),
                     N.ptr(hvis) if with_visited else None, N.MEM_HOST)
        for _ in range(args.warmup):
            N.check(fn(*call_args))
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            N.check(fn(*call_args))
        return max_ranks(time.perf_counter() - t0)

    e2e_s = e2e_run(False)
    assert np.array_equal(hc.numpy(), c), "host-path codes differ from device-path codes"
    e2e_value = world * BATCH * args.steps / e2e_s
    e2e_vis_value = world * BATCH * args.steps / e2e_run(True)
    clocks = sampler.stop()

    # ---- the reference-shaped API a user calls (queries.py:94-142, 210-249)
    api = api_paths(E, W, N, g, idx, qu_h, qv_h, c, n, args, max_ranks, barrier, world)

    # ---- incremental insertion: batches of 100k new edges (cfg4 batch size);
    # batch 0 is a warm-up (first-use kernel loading), batches 1-3 are timed
    # with CUDA events on the engine stream (graph update + propagation)
    ins_ms, ins_rates, ins_stats, prev = [], [], [], None
    for b in range(4):
        iu, iv = W.gen_insert_workload(src, dst, n, 100_000, 50 + b, exclude=prev)
        prev = (iu, iv) if prev is None else (np.concatenate([prev[0], iu]), np.concatenate([prev[1], iv]))
        du = torch.from_numpy(iu.view(np.int32)).to(dev)
        dv = torch.from_numpy(iv.view(np.int32)).to(dev)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = ev_pair()
        e0.record(stream)
        st = E.insert_edges(g, idx, du, dv)
        e1.record(stream)
        e1.synchronize()
        dt = max_ranks(e0.elapsed_time(e1))
        if b:
            ins_ms.append(dt)
            ins_rates.append(st.inserted / (dt / 1e3))
            ins_stats.append(st)
    peak, peak_src = measured_peak()
    ins_bytes = [s.inserted * (8 + 2 * rec_bytes) + 16 * s.inserted + 16 * s.fix_items + 12 * s.fix_edges
                 for s in ins_stats]
    ins_achieved = statistics.mean(b / (t / 1e3) / 1e9 for b, t in zip(ins_bytes, ins_ms))

    # single-edge insert_edge (updates.py:112-137) through the shim, per call
    su, sv = W.gen_insert_workload(src, dst, n, 2020, 90, exclude=prev)
    for u_, v_ in zip(su[:20].tolist(), sv[:20].tolist()):
        E.insert_edge(g, idx, u_, v_)
    barrier()
    t0 = time.perf_counter()
    for u_, v_ in zip(su[20:].tolist(), sv[20:].tolist()):
        E.insert_edge(g, idx, u_, v_)
    single_ins = (len(su) - 20) / max_ranks(time.perf_counter() - t0)

    # ---- whole-box R-MAT 2^24 (north_star)
    box = whole_box(args, E, W, N, torch, dist, rank, world, devi, dev, max_ranks, barrier, gloo)

    # algorithmic bytes of the digest algorithm: pair + code + visited count +
    # both endpoints' digests, plus both records for the pairs the digest
    # leaves undecided (counted exactly from the device digest of this index)
    f_rec = digest_undecided(idx.digest(g), qu_h, qv_h)
    q_bytes = 8 + 1 + 4 + 2 * 4 + f_rec * 2 * rec_bytes
    k6_ms = statistics.mean(step_ms)   # average launch duration (the event timer is quantized)
    achieved = BATCH * q_bytes / (k6_ms / 1e3) / 1e9
    traffic = ncu_traffic("label_lean_kernel")
    l2req = ncu_l2req("label_lean_kernel")
    build_achieved = exec_bytes["total"] / (build_ms_max / 1e3) / 1e9
    model_achieved = model_bytes / (build_ms_max / 1e3) / 1e9
    result = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded R-MAT; no dataset)",
        "config": bench_config(n, m, scale, world),
        "roofline": {"bound": "hbm", "kernel": "label_lean_kernel<1,1> (K6 digest check, records for the undecided pairs, deferred per-CTA K7 warp BFS; one launch)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_query": q_bytes, "kernel_ms": k6_ms,
                     "digest_undecided_fraction": f_rec,
                     "bytes_per_query_without_digest": 8 + 1 + 4 + 2 * rec_bytes,
                     # SURVEY.md §8(d)'s B_q (+4 B visited) over the same launch time: a
                     # work-equivalent rate (the digest skips most record reads), not a
                     # bandwidth claim -- as the build's survey_model below
                     "survey_model": {"bytes_per_query": 8 + 1 + 4 + 2 * rec_bytes,
                                      "achieved": BATCH * (13 + 2 * rec_bytes) / (k6_ms / 1e3) / 1e9,
                                      "frac": BATCH * (13 + 2 * rec_bytes) / (k6_ms / 1e3) / 1e9 / peak,
                                      "basis": "SURVEY.md §8(d) B_q = 8 + 1 + 2R, plus the 4-byte visited store"},
                     # what binds this kernel: SM->L2 requests (ncu count per launch) per
                     # event-timed launch against the random-gather request ceiling
                     "l2_requests": None if not l2req else {
                         "per_launch": l2req, "achieved_G_per_s": l2req / (k6_ms / 1e3) / 1e9,
                         "ceiling_G_per_s": L2_REQ_CEILING_G,
                         "frac": l2req / (k6_ms / 1e3) / 1e9 / L2_REQ_CEILING_G,
                         "ceiling_source": "tools/ubench_gather.cu, profiles/r01_ubench_gather.txt"}},
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": 8 * BATCH,
                "d2h_bytes_per_step": BATCH, "api": "dbl_query(mem=DBL_MEM_HOST) on pinned buffers: the kernels "
                "read the pairs and write the codes over PCIe (zero-copy); answer codes returned",
                "with_visited_counts": {"value": e2e_vis_value, "d2h_bytes_per_step": 5 * BATCH}},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "kernel_ms": {"query_kernel": k6_ms, "step": statistics.mean(step_ms),
                      "note": "one launch per step (hard-path BFS kernels are device tail launches)"},
        "rho": rho,
        "bfs_hard_path_queries": int(qcnt[0]),
        "positive_batch": {"value": pos_qps, "unit": "queries/s", "rho": pos_rho},
        "api_paths": api,
        "build": {"value_s": build_ms_max / 1e3, "fixpoint_ms": fix_ms.value, "mode": "replicated",
                  "roofline": {"bound": "hbm", "achieved": build_achieved, "peak": peak, "unit": "GB/s",
                               "frac": build_achieved / peak, "bytes": exec_bytes,
                               "basis": "bytes of the executed work (instrumented build's counters)"},
                  "survey_model": {"bytes": model_bytes, "achieved": model_achieved,
                                   "frac": model_achieved / peak,
                                   "basis": "SURVEY.md §8(d) level-synchronous work model (work-equivalent rate)",
                                   "V": V.tolist(), "E": Ecnt.tolist(), "levels": L.tolist()},
                  "executed_work": work_dict(bw)},
        "inserts": {"value": statistics.median(ins_rates), "unit": "edges/s", "batch": 100_000,
                    "rates": ins_rates, "ms": ins_ms,
                    "roofline": {"bound": "hbm", "achieved": ins_achieved, "peak": peak, "unit": "GB/s",
                                 "frac": ins_achieved / peak, "bytes_per_batch": ins_bytes,
                                 "basis": "b(8 + 2R) + 16b + 16 items + 12 edges of the delta fixpoint"},
                    "fixpoint_work": [{"items": s.fix_items, "edges": s.fix_edges, "levels": s.levels}
                                      for s in ins_stats],
                    "single_insert_edge": {"value": single_ins, "unit": "edges/s",
                                           "api": "insert_edge(g, idx, u, v) per call (updates.py:112-137)"}},
        "whole_box_2^24": box,
    }
    if sharded is not None:
        result["build_sharded"] = sharded
    if want_cpu:
        result["cpu_baseline"] = cpu_baseline(args, n, src, dst, qu_h, qv_h, c, built_words, pu_h, pv_h, pos_codes)
    return result


def api_paths(E, W, N, g, idx, qu_h, qv_h, codes, n, args, max_ranks, barrier, world) -> dict:
    """Rates of the reference-shaped calls: query_batch on pageable numpy
    arrays and on a Python list of pairs, single query() calls."""
    out = {}
    for _ in range(2):
        E.query_batch(g, idx, (qu_h, qv_h))
    barrier()
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        res, _ = E.query_batch(g, idx, (qu_h, qv_h))
    dt = max_ranks(time.perf_counter() - t0)
    assert np.array_equal(res.codes, codes)
    out["query_batch_numpy"] = {"value": world * reps * BATCH / dt, "unit": "queries/s",
                                "api": "query_batch(g, idx, (u, v)) on pageable numpy arrays -> Outcomes"}
    pairs = list(zip(qu_h[:100_000].tolist(), qv_h[:100_000].tolist()))
    barrier()
    t0 = time.perf_counter()
    res, _ = E.query_batch(g, idx, pairs)
    dt = max_ranks(time.perf_counter() - t0)
    assert np.array_equal(res.codes, codes[:100_000])
    out["query_batch_list"] = {"value": world * len(pairs) / dt, "unit": "queries/s",
                               "api": "query_batch(g, idx, [(u, v), ...]) on a 100k-pair Python list"}
    sample = list(zip(qu_h[:2000].tolist(), qv_h[:2000].tolist()))
    for u_, v_ in sample[:100]:
        E.query(g, idx, u_, v_)
    barrier()
    t0 = time.perf_counter()
    for u_, v_ in sample:
        E.query(g, idx, u_, v_)
    dt = max_ranks(time.perf_counter() - t0)
    out["single_query"] = {"value": len(sample) / dt, "unit": "queries/s", "us_per_call": 1e6 * dt / len(sample),
                           "api": "query(g, idx, u, v) per call (queries.py:94-142)"}
    return out


def whole_box(args, E, W, N, torch, dist, rank, world, devi, dev, max_ranks, barrier, gloo) -> dict:
    """North_star: whole-box queries/s on R-MAT 2^24 (d = 8), 1M uniform pairs per GPU,
    plus one 16M batch split over the GPUs (the reference pool's contiguous slices)."""
    from paper_2101_09441_b200.parallel import slice_bounds
    scale = args.box_scale
    n = 1 << scale
    s, d = W.rmat_edges_device(scale, EDGE_FACTOR, 24, device=devi)
    g = E.DynamicGraph.from_edges(n, s, d, device=devi)
    del s, d
    sp = N.ctypes.c_void_p()
    N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value, device=dev)
    bms = []
    idx = None
    for rep in range(4):
        idx = None
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        idx = E.build_index(g)
        e1.record(stream)
        torch.cuda.synchronize()
        if rep:
            bms.append(e0.elapsed_time(e1))
    build_ms = max_ranks(statistics.mean(bms))
    flags = E.DEFAULT_FLAGS.bits()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(u_t, v_t, cnt, steps):
        codes = torch.empty(max(cnt, 1), dtype=torch.uint8, device=dev)
        ms = []
        with torch.cuda.stream(stream):
            for i in range(args.warmup + steps):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                N.call("dbl_query_async", idx.handle, g.handle, N.ptr(u_t), N.ptr(v_t), cnt, flags,
                       N.ptr(codes), None)
                e1.record(stream)
                e1.synchronize()
                if i >= args.warmup:
                    ms.append(e0.elapsed_time(e1))
        N.call("dbl_sync", g.handle)
        return ms, codes

    # weak: 1M uniform pairs per GPU
    qu, qv = W.uniform_queries(n, BATCH, 24 + 1000 * rank)
    du = torch.from_numpy(qu.view(np.int32)).to(dev)
    dv = torch.from_numpy(qv.view(np.int32)).to(dev)
    barrier()
    ms, codes = timed(du, dv, BATCH, args.steps)
    weak_ms = max_ranks(sum(ms)) / len(ms)
    wc = codes.cpu().numpy()
    assert wc.max() <= 6
    # strong: one 16M batch, contiguous slices (queries.py:231-232)
    total = 16 * BATCH
    lo, hi = slice_bounds(total, world)[rank]
    gu, gv = W.uniform_queries(n, total, 4242)
    su = torch.from_numpy(gu[lo:hi].view(np.int32)).to(dev)
    sv = torch.from_numpy(gv[lo:hi].view(np.int32)).to(dev)
    barrier()
    ms2, _ = timed(su, sv, hi - lo, max(3, args.steps // 5))
    strong_ms = max_ranks(sum(ms2)) / len(ms2)
    out = {"workload": f"R-MAT 2^{scale}, avg out-degree {EDGE_FACTOR}, a/b/c/d=.57/.19/.19/.05, dedup, "
                       f"device generator seed 24; k=k'=64",
           "n": n, "m": g.edge_count,
           "build_s": build_ms / 1e3,
           "weak": {"value": world * BATCH / (weak_ms / 1e3), "unit": "queries/s", "ms_per_step": weak_ms,
                    "queries_per_gpu": BATCH, "rho": float(np.mean(wc < 5))},
           "strong": {"value": total / (strong_ms / 1e3), "unit": "queries/s", "ms_per_step": strong_ms,
                      "global_batch": total, "split": "contiguous slices of ceil(q/N) (queries.py:231-232)"},
           "l2": "256 MB write before every timed step (the 512 MB label table exceeds L2)"}
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        # parity at this size: 100k of the batch's codes against the CSR oracle
        # on the GPU's own labels (the oracle build is minutes at 2^24)
        from oracle import oracle as O
        fptr, fcol = g.adjacency(False)
        k = 100_000
        oc = O.csr_query_batch(n, fptr.astype(np.uint64), fcol, 64, 64, idx.export_words(), qu[:k], qv[:k],
                               threads=os.cpu_count() or 1)
        assert np.array_equal(oc, wc[:k]), "2^24 codes differ from the CSR oracle"
        out["parity"] = f"{k} codes equal the CSR oracle's on the exported labels"
    del idx, g
    return out


def _max_over_ranks(torch, dist, world, x: float, gloo: bool = False) -> float:
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if gloo else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# -------------------------------------------------------- CPU baselines --

def cpu_baseline(args, n, src, dst, qu, qv, gpu_codes, words, pu, pv, pos_codes) -> dict:
    """The oracle port on the host cores: same graph, same 1M batch, all threads,
    warmed up and timed over the same step count as the reference arm.  It also
    checks the GPU's labels (all four families) and both batches' codes."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    og = O.OracleGraph(n, src, dst)
    t0 = time.perf_counter()
    oidx = og.build(64, 64, threads=cores)
    build_s = time.perf_counter() - t0
    labels_equal = all(np.array_equal(words[f], getattr(oidx, f)) for f in FAMS)
    assert labels_equal, "GPU labels differ from the oracle's at the bench config"
    for _ in range(max(1, args.warmup)):
        oc, _ = og.query_batch(oidx, qu, qv, threads=cores)
    assert np.array_equal(oc, gpu_codes), "GPU codes differ from the oracle on the bench batch"
    steps = max(3, min(args.steps, 10))
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        og.query_batch(oidx, qu, qv, threads=cores)
        times.append(time.perf_counter() - t0)
    opc, _ = og.query_batch(oidx, pu, pv, threads=cores)
    assert np.array_equal(opc, pos_codes), "GPU codes differ from the oracle on the positive batch"
    t0 = time.perf_counter()
    og.query_batch(oidx, qu, qv, threads=1)
    one = time.perf_counter() - t0
    return {"value": BATCH * steps / sum(times), "unit": "queries/s", "cores": cores, "kind": "port",
            "sample": f"full 1M-query batch x{steps} after warm-up, oracle/dbl_oracle.c query_batch, "
                      f"{cores} threads; build {build_s:.2f} s on {cores} threads",
            "single_thread_value": BATCH / one, "build_s": build_s,
            "parity": {"labels_equal_oracle": labels_equal, "uniform_codes_equal": True,
                       "positive_codes_equal": True}}


def run_reference(args):
    from oracle import oracle as O
    from paper_2101_09441_b200 import workload as W
    n, src, dst, qu, qv = make_workload(0, args.scale)
    cores = os.cpu_count() or 1
    og = O.OracleGraph(n, src, dst)
    m = og.edge_count
    t0 = time.perf_counter()
    oidx = og.build(64, 64, threads=cores)
    build_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        og.query_batch(oidx, qu, qv, threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        og.query_batch(oidx, qu, qv, threads=cores)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = BATCH * args.steps / total
    # sequential insert_edge loop (updates.py:112-137) on a bounded sample
    iu, iv = W.gen_insert_workload(src, dst, n, 20_000, 50)
    t0 = time.perf_counter()
    for u, v in zip(iu.tolist(), iv.tolist()):
        og.insert_edge(oidx, u, v)
    ins_rate = len(iu) / (time.perf_counter() - t0)
    sample = (f"1M-query batch per step, oracle/dbl_oracle.c (port of queries.py:94-142), "
              f"{cores} threads; build {build_s:.2f} s; inserts: sequential insert_edge x20000")
    pyref = python_reference(n, src, dst, oidx, qu, qv, cores)
    return {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded R-MAT; no dataset)", "impl": "reference",
            "config": bench_config(n, m, args.scale, args.gpus),
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "build": {"value_s": build_s, "threads": cores},
            "inserts": {"value": ins_rate, "unit": "edges/s", "threads": 1},
            "python_reference": pyref}


def python_reference(n, src, dst, oidx, qu, qv, cores) -> dict:
    """Context only: the unmodified Python reference (dblreach, pip-installed
    into baseline/_ref) answering the same batch.  Its own build takes ~640 s
    at this size, so it loads the labels from a DBLIDX01 snapshot of the
    port's index (the format both engines read; snapshot.py:104-148), then
    query_batch with workers = 1 on a 100k sample and workers = cpu_count on
    the whole batch (queries.py:210-249).  Codes are checked against the port."""
    import io
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(ref_dir):
        return {"unavailable": "baseline/_ref not installed"}
    sys.path.insert(0, ref_dir)
    try:
        import dblreach as R
    except ImportError as e:
        return {"unavailable": f"import dblreach failed: {e}"}
    finally:
        sys.path.remove(ref_dir)
    from oracle import oracle as O
    from paper_2101_09441_b200.labels import IndexConfig
    from paper_2101_09441_b200.snapshot import encode_snapshot
    t0 = time.perf_counter()
    g = R.DynamicGraph(n)
    for u, v in zip(src.tolist(), dst.tolist()):
        g.add_edge(u, v)
    load_s = time.perf_counter() - t0
    blob = encode_snapshot(IndexConfig(), n, oidx.landmarks.astype(np.uint64), oidx.leaf_flags, oidx.bucket,
                           oidx.dl_in, oidx.dl_out, oidx.bl_in, oidx.bl_out)
    idx = R.load_index(io.BytesIO(blob))
    pairs = list(zip(qu.tolist(), qv.tolist()))
    k = 100_000
    t0 = time.perf_counter()
    outs1, _ = R.query_batch(g, idx, pairs[:k], workers=1)
    one = k / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    outs, _ = R.query_batch(g, idx, pairs, workers=cores)
    many = len(pairs) / (time.perf_counter() - t0)
    names = [a.value for a in R.AnsweredBy]
    codes = np.array([names.index(o.answered_by.value) for o in outs], np.uint8)
    oc, _ = O.OracleGraph(n, src, dst).query_batch(oidx, qu, qv, threads=cores)
    # the per-call API: query() and insert_edge() one call at a time (the
    # engine's api_paths.single_query / inserts.single_insert_edge), at most
    # ~10 s each; the inserts come last (they change the reference's graph)
    t0 = time.perf_counter()
    nq = 0
    for u, v in pairs[:50_000]:
        R.query(g, idx, u, v)
        nq += 1
        if nq % 1000 == 0 and time.perf_counter() - t0 > 10:
            break
    single_q = nq / (time.perf_counter() - t0)
    from paper_2101_09441_b200 import workload as W
    su, sv = W.gen_insert_workload(src, dst, n, 2300, 90)
    t0 = time.perf_counter()
    ni = 0
    for u, v in zip(su.tolist(), sv.tolist()):
        R.insert_edge(g, idx, u, v)
        ni += 1
        if time.perf_counter() - t0 > 10:
            break
    single_ins = ni / (time.perf_counter() - t0)
    return {"value_workers_1": one, "value_workers_all": many, "unit": "queries/s", "cores": cores,
            "single_query": {"value": single_q, "unit": "queries/s", "calls": nq,
                             "api": "dblreach.query(g, idx, u, v) per call"},
            "single_insert_edge": {"value": single_ins, "unit": "edges/s", "calls": ni,
                                   "api": "dblreach.insert_edge(g, idx, u, v) per call, edges of "
                                          "workload.gen_insert_workload(seed 90) on the base cfg2 graph"},
            "codes_equal_port": bool(np.array_equal(codes, oc)),
            "sample": f"dblreach 0.1.0 (unmodified, baseline/_ref): query_batch workers=1 on {k} pairs, "
                      f"workers={cores} on the 1M batch; labels via load_index of a DBLIDX01 snapshot of "
                      f"the port's build (graph load {load_s:.1f} s not timed)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scale", type=int, default=SCALE, help="cfg2 R-MAT scale (20; smaller only for tests)")
    ap.add_argument("--box-scale", type=int, default=24, help="whole-box R-MAT scale (24)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    gloo = os.environ.get("DBL_BENCH_GLOO") == "1"
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if gloo:
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_ours(args, rank, world, local_rank, gloo)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
