"""Benchmark: reach queries/s on a 1M-query batch (+ label build s, edge inserts/s).

BASELINE.json metric "reach queries/sec (1M-query batch) + label build sec and
edge-inserts/sec"; workload = configs[1]: directed R-MAT 2^20, average
out-degree 8, (a, b, c, d) = (.57, .19, .19, .05), duplicates removed, seeded
(numpy PCG64 seed 1, ids unpermuted); default IndexConfig (k = k' = 64).

One step = one pass of the query hot path (K6 label check + K7 pruned-BFS
fallback) over a batch of 1M uniform random pairs resident in HBM; L2 is
flushed (256 MB write) before every timed step; each step is bracketed by
CUDA events on the engine's stream.  `e2e` times the same batch through the
public C-ABI call dbl_query with pinned HOST buffers (H2D of the pairs and
D2H of codes + visited inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Multi-GPU (torchrun, one rank per GPU): graph + labels are replicated, the
label build is sharded by record word with an NCCL allgather, and every rank
answers its own 1M-query batch (weak scaling, no collective on the query
path); times are the max over ranks.

--impl reference times the reference algorithm's CPU implementation on the
host cores instead: the oracle port (oracle/dbl_oracle.c, a restatement of
the Python reference, which cannot travel to the GPU box) on the same graph
and query batches, all host threads.
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
WORKLOAD = ("cfg2: directed R-MAT 2^20, avg out-degree 8, a/b/c/d=.57/.19/.19/.05, dedup, "
            "seed 1 (numpy PCG64, unpermuted ids); k=64 landmarks (product), k'=64 BL; "
            "1M uniform random (u,v) pairs per step")
METRIC = "reach queries/sec (1M-query batch)"


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


def make_workload(rank: int):
    from paper_2101_09441_b200 import workload as W
    src, dst = W.rmat_edges(SCALE, EDGE_FACTOR, GRAPH_SEED)
    n = 1 << SCALE
    qu, qv = W.uniform_queries(n, BATCH, 2 + 1000 * rank)
    return n, src, dst, qu, qv


# ----------------------------------------------------------------- ours --

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2101_09441_b200 as E
    from paper_2101_09441_b200 import _native as N
    from paper_2101_09441_b200 import workload as W
    from paper_2101_09441_b200.parallel import sharded_build

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n, src, dst, qu_h, qv_h = make_workload(rank)
    g = E.DynamicGraph.from_edges(n, src, dst, device=local_rank)
    m = g.edge_count
    sp = N.ctypes.c_void_p()
    N.call("dbl_stream", g.handle, N.ctypes.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- label build (device time, CSR/CSC resident -> final AoS table)
    cfg = E.IndexConfig()
    build_ms = []
    idx = None
    for rep in range(8):   # rep 0 warms the allocator cache; the previous index is dropped first
        idx = None
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if world > 1:
            idx = sharded_build(g, cfg, rank, world)
        else:
            idx = E.build_index(g, cfg)
        e1.record(stream)
        torch.cuda.synchronize()
        if rep:
            build_ms.append(e0.elapsed_time(e1))
    build_ms_max = _max_over_ranks(torch, dist, world, statistics.mean(build_ms))
    fix_ms = N.ctypes.c_float()
    N.call("dbl_last_timings", g.handle, N.ctypes.byref(fix_ms), None, None)

    # work model -> algorithmic build bytes
    rw = 2 * (idx.wdl + idx.wbl)
    V = np.zeros(rw, np.uint64)
    Ecnt = np.zeros(rw, np.uint64)
    L = np.zeros(rw, np.uint32)
    N.call("dbl_work_model", idx.handle, g.handle, N.ptr(V), N.ptr(Ecnt), N.ptr(L))
    rec_bytes = 8 * rw
    build_bytes = int(sum(16 * int(v) + 12 * int(e) for v, e in zip(V, Ecnt)) + n * (8 * rw + rec_bytes))

    # ---- queries: device-resident batch
    qu = torch.from_numpy(qu_h.view(np.int32)).to(dev)
    qv = torch.from_numpy(qv_h.view(np.int32)).to(dev)
    codes = torch.empty(BATCH, dtype=torch.uint8, device=dev)
    vis = torch.empty(BATCH, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flags = E.DEFAULT_FLAGS.bits()

    flush2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def l2_flush():
        # write 256 MB (evicts everything), then read 256 MB so the write-back of
        # the dirty flush lines happens here rather than inside the timed step
        flush.fill_(1)
        flush2.max()

    def step():
        N.call("dbl_query_async", idx.handle, g.handle, N.ptr(qu), N.ptr(qv), BATCH, flags,
               N.ptr(codes), N.ptr(vis))

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            l2_flush()
            step()
    torch.cuda.synchronize()
    # correctness guard: the timed batch is fully answered
    c = codes.cpu().numpy()
    assert c.max() <= 6, "unanswered queries in the batch"
    rho = float(np.mean(c < 5))

    sampler = ClockSampler(local_rank)
    sampler.start()
    barrier()
    torch.cuda.synchronize()
    launches0 = N.kernel_launches()
    step_ms, label_ms, bfs_ms = [], [], []
    tl, tb = N.ctypes.c_float(), N.ctypes.c_float()
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            l2_flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            N.call("dbl_last_timings", g.handle, None, N.ctypes.byref(tl), N.ctypes.byref(tb))
            label_ms.append(tl.value)
            bfs_ms.append(tb.value)
    torch.cuda.synchronize()
    barrier()
    launches = N.kernel_launches() - launches0
    qcnt = np.zeros(8, np.uint32)
    N.call("dbl_query_counters", g.handle, N.ptr(qcnt))
    total_ms = _max_over_ranks(torch, dist, world, sum(step_ms))
    ms_per_step = total_ms / args.steps
    value = world * BATCH * args.steps / (total_ms / 1e3)

    # positives batch (cfg2's second query set), same measurement
    pu_h, pv_h = W.positive_queries(n, src, dst, BATCH, 3 + 1000 * rank)
    pu = torch.from_numpy(pu_h.view(np.int32)).to(dev)
    pv = torch.from_numpy(pv_h.view(np.int32)).to(dev)
    pos_ms = []
    with torch.cuda.stream(stream):
        for i in range(args.warmup + max(5, args.steps // 4)):
            l2_flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            N.call("dbl_query_async", idx.handle, g.handle, N.ptr(pu), N.ptr(pv), BATCH, flags,
                   N.ptr(codes), N.ptr(vis))
            e1.record(stream)
            e1.synchronize()
            if i >= args.warmup:
                pos_ms.append(e0.elapsed_time(e1))
    pos_rho = float(np.mean(codes.cpu().numpy() < 5))
    pos_total = _max_over_ranks(torch, dist, world, sum(pos_ms))
    pos_qps = world * BATCH * len(pos_ms) / (pos_total / 1e3)

    # ---- e2e through the public C-ABI call with pinned host buffers: H2D of
    # the pairs and D2H of the answer codes (the step's result) every step
    hu = torch.from_numpy(qu_h.view(np.int32)).pin_memory()
    hv = torch.from_numpy(qv_h.view(np.int32)).pin_memory()
    hc = torch.empty(BATCH, dtype=torch.uint8).pin_memory()
    hvis = torch.empty(BATCH, dtype=torch.int32).pin_memory()

    def e2e_run(with_visited: bool) -> float:
        vptr = N.ptr(hvis) if with_visited else None
        for _ in range(args.warmup):
            N.call("dbl_query", idx.handle, g.handle, N.ptr(hu), N.ptr(hv), BATCH, flags, N.ptr(hc), vptr,
                   N.MEM_HOST)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            N.call("dbl_query", idx.handle, g.handle, N.ptr(hu), N.ptr(hv), BATCH, flags, N.ptr(hc), vptr,
                   N.MEM_HOST)
        return _max_over_ranks(torch, dist, world, time.perf_counter() - t0)

    e2e_s = e2e_run(False)
    assert np.array_equal(hc.numpy(), c), "host-path codes differ from device-path codes"
    e2e_value = world * BATCH * args.steps / e2e_s
    e2e_vis_value = world * BATCH * args.steps / e2e_run(True)
    clocks = sampler.stop()

    # ---- incremental insertion: batches of 100k new edges (cfg4 batch size);
    # batch 0 is a warm-up (first-use kernel loading), batches 1-3 are timed
    ins_rates, prev = [], None
    for b in range(4):
        iu, iv = W.gen_insert_workload(src, dst, n, 100_000, 50 + b, exclude=prev)
        prev = (iu, iv) if prev is None else (np.concatenate([prev[0], iu]), np.concatenate([prev[1], iv]))
        du = torch.from_numpy(iu.view(np.int32)).to(dev)
        dv = torch.from_numpy(iv.view(np.int32)).to(dev)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        st = E.insert_edges(g, idx, du, dv)
        dt = _max_over_ranks(torch, dist, world, time.perf_counter() - t0)
        if b:
            ins_rates.append(st.inserted / dt)

    peak, peak_src = measured_peak()
    q_bytes = 8 + 1 + 4 + 2 * rec_bytes
    k6_ms = statistics.mean(label_ms)   # average launch duration (the event timer is quantized)
    achieved = BATCH * q_bytes / (k6_ms / 1e3) / 1e9
    traffic = ncu_traffic("label_lean_kernel")
    build_achieved = build_bytes / (build_ms_max / 1e3) / 1e9
    result = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded R-MAT; no dataset)",
        "config": {"workload": WORKLOAD, "n": n, "m": m, "queries_per_step": BATCH,
                   "k": 64, "k_prime": 64,
                   "l2": "flushed before every timed step (256 MB write, then 256 MB read so no dirty lines remain)",
                   "parallelism": f"replicated graph+labels, word-sharded build + NCCL allgather, "
                                  f"one 1M batch per GPU x{world}"},
        "roofline": {"bound": "hbm", "kernel": "label_lean_kernel<1,1> (K6 label check + deferred per-lane K7 BFS, one launch)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_query": q_bytes, "kernel_ms": k6_ms},
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": 8 * BATCH,
                "d2h_bytes_per_step": BATCH, "api": "dbl_query(mem=DBL_MEM_HOST) on pinned buffers: the kernels "
                "read the pairs and write the codes over PCIe (zero-copy); answer codes returned",
                "with_visited_counts": {"value": e2e_vis_value, "d2h_bytes_per_step": 5 * BATCH}},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "kernel_ms": {"query_kernel": k6_ms, "separate_bfs_kernels": statistics.mean(bfs_ms),
                      "step": statistics.mean(step_ms)},
        "rho": rho,
        "bfs_hard_path_queries": int(qcnt[0]),
        "positive_batch": {"value": pos_qps, "unit": "queries/s", "rho": pos_rho},
        "build": {"value_s": build_ms_max / 1e3, "fixpoint_ms": fix_ms.value,
                  "algorithmic_bytes": build_bytes,
                  "roofline": {"bound": "hbm", "achieved": build_achieved, "peak": peak, "unit": "GB/s",
                               "frac": build_achieved / peak},
                  "work_model": {"V": V.tolist(), "E": Ecnt.tolist(), "levels": L.tolist()}},
        "inserts": {"value": statistics.median(ins_rates), "unit": "edges/s", "batch": 100_000,
                    "rates": ins_rates},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(n, src, dst, qu_h, qv_h, c)
    return result


def _max_over_ranks(torch, dist, world, x: float) -> float:
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# -------------------------------------------------------- CPU baselines --

def cpu_baseline(n, src, dst, qu, qv, gpu_codes=None) -> dict:
    """The oracle port on the host cores: same graph, same 1M batch, all threads."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    og = O.OracleGraph(n, src, dst)
    t0 = time.perf_counter()
    oidx = og.build(64, 64, threads=cores)
    build_s = time.perf_counter() - t0
    times = []
    for _ in range(5):
        t0 = time.perf_counter()
        oc, _ = og.query_batch(oidx, qu, qv, threads=cores)
        times.append(time.perf_counter() - t0)
    if gpu_codes is not None:
        assert np.array_equal(oc, gpu_codes), "GPU codes differ from the oracle on the bench batch"
    t0 = time.perf_counter()
    oc1, _ = og.query_batch(oidx, qu, qv, threads=1)
    one = time.perf_counter() - t0
    return {"value": BATCH / statistics.median(times), "unit": "queries/s", "cores": cores,
            "kind": "port",
            "sample": f"full 1M-query batch x5 (median), oracle/dbl_oracle.c query_batch, {cores} threads; "
                      f"build {build_s:.2f} s on {cores} threads",
            "single_thread_value": BATCH / one, "build_s": build_s}


def run_reference(args):
    from oracle import oracle as O
    from paper_2101_09441_b200 import workload as W
    n, src, dst, qu, qv = make_workload(0)
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
    return {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded R-MAT; no dataset)", "impl": "reference",
            "config": {"workload": WORKLOAD, "n": n, "m": m, "queries_per_step": BATCH,
                       "k": 64, "k_prime": 64},
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "build": {"value_s": build_s, "threads": cores},
            "inserts": {"value": ins_rate, "unit": "edges/s", "threads": 1}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
