"""Multi-rank device paths with real kernels: 2 and 3 ranks
share cuda:0 over gloo and run the word-sharded label build (allgather of
record words) and the split query batch end to end; every rank's labels must
equal a single-GPU build and the oracle, and the gathered codes the
single-call answers.  Plus the single-process multi-handle split
(dbl_query_multi) against query_batch.
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_word_sharded_build_and_split_queries_multirank(world, tmp_path):
    port = _free_port()
    outs = [tmp_path / f"r{r}.json" for r in range(world)]
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "multirank_worker.py"),
                               str(r), str(world), str(port), str(outs[r])], cwd=ROOT)
             for r in range(world)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    for r in range(world):
        res = json.loads(outs[r].read_text())
        assert res["ok"], res


def test_query_multi_two_handles_one_gpu():
    import paper_2101_09441_b200 as E
    from paper_2101_09441_b200 import parallel as P
    from paper_2101_09441_b200 import workload as W
    n = 1 << 14
    src, dst = W.rmat_edges(14, 8, seed=7)
    reps = P.replicate(n, src, dst, [0, 0])
    qu, qv = W.uniform_queries(n, 100_003, seed=8)
    one, s1 = E.query_batch(reps[0][0], reps[0][1], (qu, qv))
    for k in (1, 2):
        out, st = P.query_batch_sharded(reps[:k], (qu, qv))
        assert np.array_equal(out.codes, one.codes)
        assert np.array_equal(out.visited == 0, one.visited == 0)
        assert st.query_count == s1.query_count and st.label_answered == s1.label_answered
    # a batch resident on the GPU (the peer-access path; one device here)
    import torch
    du = torch.from_numpy(qu.view(np.int32)).cuda()
    dv = torch.from_numpy(qv.view(np.int32)).cuda()
    for k in (1, 2):
        out, _ = P.query_batch_sharded(reps[:k], (du, dv))
        assert np.array_equal(out.codes, one.codes)
    # tiny and empty batches take the serial path
    out, _ = P.query_batch_sharded(reps, [(0, 1), (2, 2), (5, 3)])
    assert np.array_equal(out.codes, E.query_batch(reps[0][0], reps[0][1], [(0, 1), (2, 2), (5, 3)])[0].codes)
    out, _ = P.query_batch_sharded(reps, [])
    assert len(out) == 0


def test_query_multi_errors():
    import paper_2101_09441_b200 as E
    from paper_2101_09441_b200 import parallel as P
    n = 100
    src = np.arange(99, dtype=np.uint32)
    dst = src + 1
    reps = P.replicate(n, src, dst, [0, 0])
    with pytest.raises(E.VertexRangeError):
        P.query_batch_sharded(reps, [(0, 1)] * 10 + [(0, 100)])
    g2 = E.DynamicGraph.from_edges(101, src, dst)
    with pytest.raises(E.IndexGraphMismatchError):
        P.query_batch_sharded([reps[0], (g2, reps[1][1])], [(0, 1)] * 10)
    with pytest.raises(TypeError):   # one handle twice would be driven from two threads (DBL_E_ARG)
        P.query_batch_sharded([reps[0], reps[0]], [(0, 1)] * 10)


def _bench_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_small():
    """bench.py's whole N = 1 code path (incl. the CPU-port parity leg) at small scales."""
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--scale", "15",
                        "--box-scale", "17"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = _bench_json(r.stdout)
    assert res["n_gpus"] == 1 and res["value"] > 0 and res["e2e"]["value"] > 0
    assert res["cpu_baseline"]["parity"]["labels_equal_oracle"]
    assert res["whole_box_2^24"]["weak"]["value"] > 0 and "parity" in res["whole_box_2^24"]
    assert res["build"]["roofline"]["bytes"]["total"] > 0
    assert res["gpu_launches"] >= res["steps"]


def test_bench_two_ranks_gloo():
    """bench.py --gpus 2 under torchrun with both ranks on cuda:0 (gloo):
    the N > 1 path incl. the word-sharded build, checked equal."""
    env = dict(os.environ, DBL_BENCH_GLOO="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--scale", "15", "--box-scale", "17"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    res = _bench_json(r.stdout)
    assert res["n_gpus"] == 2
    assert res["build_sharded"]["labels_equal_replicated"]
    assert res["whole_box_2^24"]["strong"]["value"] > 0
