"""Multi-rank host logic of the sharded label build, on CPU with gloo
(world_size 2 and 3): word plan, slab packing, allgather, record interleave.

Each rank's "build" fills its assigned record words from the oracle's labels
(the oracle being the checker); after the exchange every rank must hold the
complete record table, identical to the oracle's.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_09441_b200.parallel import plan_words, sharded_exchange


def test_plan_words_covers_every_word_once():
    for rw in (2, 4, 10, 28):
        for world in (1, 2, 3, 4, 8):
            plan = plan_words(rw, world)
            flat = sorted(w for p in plan for w in p)
            assert flat == list(range(rw))
            sizes = [len(p) for p in plan]
            assert max(sizes) - min(sizes) <= 1


def oracle_records(n_scale=10, k=128, kp=64):
    from oracle import oracle as O
    from paper_2101_09441_b200 import workload as W
    src, dst = W.rmat_edges(n_scale, 8, seed=4)
    n = 1 << n_scale
    idx = O.OracleGraph(n, src, dst).build(k, kp, threads=2)
    # AoS record {dl_in | bl_in | dl_out | bl_out} as in csrc/internal.cuh
    rec = np.concatenate([idx.dl_in, idx.bl_in, idx.dl_out, idx.bl_out], axis=1)
    return n, rec


class NumpyEngine:
    def __init__(self, n, truth):
        self.n, self.rw = n, truth.shape[1]
        self.truth = truth
        self.rec = np.zeros_like(truth)

    def build_words(self, words):
        for w in words:
            self.rec[:, w] = self.truth[:, w]

    def empty_slab(self, nwords):
        return torch.zeros(max(nwords, 1) * self.n, dtype=torch.int64)

    def pack(self, words, out):
        o = out.numpy().view(np.uint64)
        for j, w in enumerate(words):
            o[j * self.n:(j + 1) * self.n] = self.rec[:, w]

    def unpack(self, words, slab):
        s = slab.numpy().view(np.uint64)
        for j, w in enumerate(words):
            self.rec[:, w] = s[j * self.n:(j + 1) * self.n]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, truth = oracle_records()
        eng = NumpyEngine(n, truth)

        def allgather(out, inp):
            parts = [torch.empty_like(inp) for _ in range(world)]
            dist.all_gather(parts, inp)
            out.copy_(torch.cat(parts))

        sharded_exchange(eng, rank, world, allgather)
        q.put((rank, bool(np.array_equal(eng.rec, truth))))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    results = sorted(q.get() for _ in range(world))
    assert results == [(r, True) for r in range(world)]
