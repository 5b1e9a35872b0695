"""ctypes wrapper for the CPU oracle (oracle/dbl_oracle.c).

TEST INFRASTRUCTURE ONLY: the checker for the CUDA engine and the "port"
CPU baseline timed by bench.py.  The product package
(paper_2101_09441_b200/) never imports this module.

The C file restates the reference's algorithm function by function (see its
header for the file:line map); this wrapper only marshals numpy arrays.
Parity of the restatement against the reference itself is pinned by
tests/test_oracle.py over the golden vectors in tests/golden/ (written by
oracle/gen_golden.py, which imports /root/reference).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "dbl_oracle.c")
LIB = os.path.join(HERE, "_build", "libdbl_oracle.so")

STRATEGY_CODES = {"max": 0, "min": 1, "sum": 2, "product": 3}
# AnsweredBy order, queries.py:40-47
ANSWER_NAMES = ("REFLEXIVE", "DL_POSITIVE", "BL_NEGATIVE", "THM1_NEGATIVE",
                "THM2_NEGATIVE", "BFS_POSITIVE", "BFS_NEGATIVE")
F_USE_DL, F_USE_BL, F_THM1, F_THM2, F_PRUNE_DL, F_PRUNE_BL = 1, 2, 4, 8, 16, 32
DEFAULT_FLAGS = 63


def build_oracle(force: bool = False) -> str:
    """Compile dbl_oracle.c with gcc into oracle/_build/ (idempotent)."""
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread",
                               SRC, "-o", tmp])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build_oracle()
        L = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        u32, u64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
        L.orc_leaf_hash.restype = u32
        L.orc_leaf_hash.argtypes = [u64, u32, u64]
        L.orc_graph_new.restype = P
        L.orc_graph_new.argtypes = [u32]
        L.orc_graph_free.argtypes = [P]
        L.orc_graph_add_edge.restype = i32
        L.orc_graph_add_edge.argtypes = [P, u32, u32]
        L.orc_graph_add_edges.restype = i32
        L.orc_graph_add_edges.argtypes = [P, P, P, u64]
        L.orc_graph_edge_count.restype = u64
        L.orc_graph_edge_count.argtypes = [P]
        L.orc_graph_has_edge.restype = i32
        L.orc_graph_has_edge.argtypes = [P, u32, u32]
        L.orc_graph_degrees.argtypes = [P, P, P]
        L.orc_select_landmarks.restype = i32
        L.orc_select_landmarks.argtypes = [P, u32, i32, P]
        L.orc_select_leaves.restype = i32
        L.orc_select_leaves.argtypes = [P, u64, u32, u64, P, P, P]
        L.orc_build.restype = i32
        L.orc_build.argtypes = [P, u32, u32, P, P, P, P, P, P, P, i32]
        L.orc_query_batch.restype = i32
        L.orc_query_batch.argtypes = [P, u32, u32, P, P, P, P, P, P, u64, u32, P, P, i32]
        L.orc_insert_edge.restype = i32
        L.orc_insert_edge.argtypes = [P, u32, u32, P, P, P, P, u32, u32, P]
        L.orc_reach_batch.restype = i32
        L.orc_reach_batch.argtypes = [P, P, P, u64, P, i32]
        L.orc_csr_flood.restype = i32
        L.orc_csr_flood.argtypes = [u32, P, P, P, u64, P]
        L.orc_csr_query_batch.restype = i32
        L.orc_csr_query_batch.argtypes = [u32, P, P, u32, u32, P, P, P, P, P, P, u64, u32, P, i32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def leaf_hash(v: int, k_prime: int, seed: int = 0) -> int:
    return int(lib().orc_leaf_hash(v, k_prime, seed))


@dataclass
class OracleIndex:
    k: int
    k_prime: int
    landmarks: np.ndarray        # u32[k]
    leaf_flags: np.ndarray       # u8[n]: bit0 leaves_in, bit1 leaves_out
    bucket: np.ndarray           # u32[n]
    dl_in: np.ndarray            # u64[n, ceil(k/64)]
    dl_out: np.ndarray
    bl_in: np.ndarray            # u64[n, ceil(k'/64)]
    bl_out: np.ndarray


class OracleGraph:
    """Reference DynamicGraph restated in C: insertion-ordered adjacency."""

    def __init__(self, n: int, src=None, dst=None):
        self.n = int(n)
        self._h = lib().orc_graph_new(self.n)
        if src is not None and len(src):
            s = np.ascontiguousarray(src, dtype=np.uint32)
            d = np.ascontiguousarray(dst, dtype=np.uint32)
            rc = lib().orc_graph_add_edges(self._h, _p(s), _p(d), len(s))
            if rc:
                raise IndexError(f"oracle add_edges failed rc={rc}")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_graph_free(self._h)
            self._h = None

    @property
    def edge_count(self) -> int:
        return int(lib().orc_graph_edge_count(self._h))

    def add_edge(self, u: int, v: int) -> bool:
        r = lib().orc_graph_add_edge(self._h, u, v)
        if r < 0:
            raise IndexError("vertex out of range")
        return bool(r)

    def has_edge(self, u: int, v: int) -> bool:
        return bool(lib().orc_graph_has_edge(self._h, u, v))

    def degrees(self):
        ind = np.zeros(self.n, np.uint32)
        outd = np.zeros(self.n, np.uint32)
        lib().orc_graph_degrees(self._h, _p(ind), _p(outd))
        return ind, outd

    def select_landmarks(self, k: int, strategy: str = "product") -> np.ndarray:
        out = np.zeros(max(k, 1), np.uint32)
        rc = lib().orc_select_landmarks(self._h, k, STRATEGY_CODES[strategy], _p(out))
        if rc:
            raise ValueError("k out of range")
        return out[:k]

    def select_leaves(self, threshold: int = 0, k_prime: int = 64, seed: int = 0,
                      override: dict | None = None):
        flags = np.zeros(self.n, np.uint8)
        bucket = np.zeros(self.n, np.uint32)
        ovr = None
        if override:
            ovr = np.full(self.n, 0xFFFFFFFF, np.uint32)
            for v, b in override.items():
                ovr[v] = b
        rc = lib().orc_select_leaves(self._h, threshold, k_prime, seed, _p(ovr),
                                     _p(flags), _p(bucket))
        if rc:
            raise ValueError("bad leaf config")
        return flags, bucket

    def build(self, k: int = 64, k_prime: int = 64, strategy: str = "product",
              leaf_threshold: int = 0, hash_seed: int = 0, landmarks=None,
              leaf_flags=None, bucket=None, override=None, threads: int = 1) -> OracleIndex:
        if landmarks is None:
            landmarks = self.select_landmarks(k, strategy)
        landmarks = np.ascontiguousarray(landmarks, dtype=np.uint32)
        if leaf_flags is None:
            leaf_flags, bucket = self.select_leaves(leaf_threshold, k_prime, hash_seed, override)
        wdl, wbl = (k + 63) // 64, (k_prime + 63) // 64
        n = self.n
        dl_in = np.zeros((n, wdl), np.uint64)
        dl_out = np.zeros((n, wdl), np.uint64)
        bl_in = np.zeros((n, wbl), np.uint64)
        bl_out = np.zeros((n, wbl), np.uint64)
        rc = lib().orc_build(self._h, k, k_prime, _p(landmarks), _p(leaf_flags), _p(bucket),
                             _p(dl_in), _p(dl_out), _p(bl_in), _p(bl_out), threads)
        if rc:
            raise ValueError(f"oracle build failed rc={rc}")
        return OracleIndex(k, k_prime, landmarks, leaf_flags, bucket, dl_in, dl_out, bl_in, bl_out)

    def rebuild(self, idx: OracleIndex, threads: int = 1) -> OracleIndex:
        """rebuild_index, labels.py:309-312: frozen landmarks and leaves."""
        return self.build(idx.k, idx.k_prime, landmarks=idx.landmarks,
                          leaf_flags=idx.leaf_flags, bucket=idx.bucket, threads=threads)

    def query_batch(self, idx: OracleIndex, qu, qv, flags: int = DEFAULT_FLAGS,
                    threads: int = 1):
        qu = np.ascontiguousarray(qu, dtype=np.uint32)
        qv = np.ascontiguousarray(qv, dtype=np.uint32)
        codes = np.zeros(len(qu), np.uint8)
        visited = np.zeros(len(qu), np.uint32)
        rc = lib().orc_query_batch(self._h, idx.k, idx.k_prime, _p(idx.dl_in), _p(idx.dl_out),
                                   _p(idx.bl_in), _p(idx.bl_out), _p(qu), _p(qv), len(qu),
                                   flags, _p(codes), _p(visited), threads)
        if rc:
            raise IndexError(f"oracle query failed rc={rc}")
        return codes, visited

    def insert_edge(self, idx: OracleIndex, u: int, v: int):
        """Returns (visited, labels_changed, early_terminated)."""
        st = np.zeros(3, np.uint32)
        rc = lib().orc_insert_edge(self._h, idx.k, idx.k_prime, _p(idx.dl_in), _p(idx.dl_out),
                                   _p(idx.bl_in), _p(idx.bl_out), u, v, _p(st))
        if rc:
            raise IndexError(f"oracle insert failed rc={rc}")
        return int(st[0]), int(st[1]), bool(st[2])

    def reach_batch(self, qu, qv, threads: int = 1) -> np.ndarray:
        qu = np.ascontiguousarray(qu, dtype=np.uint32)
        qv = np.ascontiguousarray(qv, dtype=np.uint32)
        out = np.zeros(len(qu), np.uint8)
        rc = lib().orc_reach_batch(self._h, _p(qu), _p(qv), len(qu), _p(out), threads)
        if rc:
            raise IndexError("vertex out of range")
        return out.astype(bool)


def csr_from_edges(n: int, src, dst):
    """Deduplicated CSR (u64 row pointers) of an edge list, for the CSR oracles."""
    key = np.unique(np.asarray(src, np.uint64) << np.uint64(32) | np.asarray(dst, np.uint64))
    s = (key >> np.uint64(32)).astype(np.int64)
    col = np.ascontiguousarray((key & np.uint64(0xFFFFFFFF)).astype(np.uint32))
    ptr = np.zeros(n + 1, np.uint64)
    ptr[1:] = np.cumsum(np.bincount(s, minlength=n))
    return ptr, col


def csr_flood(n: int, ptr, col, seeds) -> np.ndarray:
    """Vertices reachable from `seeds` along (ptr, col) (labels.py:247-260)."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint32)
    out = np.zeros(n, np.uint8)
    rc = lib().orc_csr_flood(n, _p(ptr), _p(col), _p(seeds), len(seeds), _p(out))
    if rc:
        raise MemoryError("oracle flood failed")
    return out.astype(bool)


def csr_query_batch(n: int, ptr, col, k: int, k_prime: int, labels: dict, qu, qv, flags: int = DEFAULT_FLAGS,
                    threads: int = 1) -> np.ndarray:
    """query (queries.py:94-142) over CSR arrays with given labels."""
    qu = np.ascontiguousarray(qu, dtype=np.uint32)
    qv = np.ascontiguousarray(qv, dtype=np.uint32)
    codes = np.zeros(len(qu), np.uint8)
    lab = [np.ascontiguousarray(labels[f], dtype=np.uint64) for f in ("dl_in", "dl_out", "bl_in", "bl_out")]
    rc = lib().orc_csr_query_batch(n, _p(ptr), _p(col), k, k_prime, *[_p(a) for a in lab], _p(qu), _p(qv),
                                   len(qu), flags, _p(codes), threads)
    if rc:
        raise IndexError("oracle query failed")
    return codes


def label_tests(labels: dict, x, y) -> tuple[np.ndarray, np.ndarray]:
    """dl_intersec (labels.py:315-319) and bl_contain (labels.py:322-327) over
    u64 word arrays: dl_out[x] & dl_in[y] != 0; bl_in[x] subset of bl_in[y]
    and bl_out[y] subset of bl_out[x]."""
    x = np.asarray(x, np.int64)
    y = np.asarray(y, np.int64)
    dl = (labels["dl_out"][x] & labels["dl_in"][y]).any(axis=1) if labels["dl_in"].shape[1] else \
        np.zeros(len(x), bool)
    bl = ~((labels["bl_in"][x] & ~labels["bl_in"][y]).any(axis=1)
           | (labels["bl_out"][y] & ~labels["bl_out"][x]).any(axis=1))
    return dl, bl
