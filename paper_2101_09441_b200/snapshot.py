"""Binary index snapshots, byte-compatible with the reference's DBLIDX01 files.

Reference: snapshot.py:1-148 and pkg/docs/snapshot-format.md:1-45.  The
labels come off the GPU through dbl_index_export (u64 words, least
significant word first) and are laid out per vertex as dl_in, dl_out, bl_in,
bl_out; the metadata (landmarks in bit order, ascending leaf sets, ascending
bucket table) is formatted with numpy.  A file written here is identical,
byte for byte, to the reference's save_index of the same index
(tests/test_snapshot.py), and either side can load the other's files.
"""
from __future__ import annotations

import ctypes
import struct
from typing import IO, Union

import numpy as np

from . import _native as N
from .errors import DblError
from .graph import DynamicGraph, as_device_graph
from .labels import DblIndex, IndexConfig, LandmarkStrategy

MAGIC = b"DBLIDX01"
VERSION = 1
_HEADER = struct.Struct("<IQIIQIB")
_STRATEGY_CODES = {LandmarkStrategy.MAX: 0, LandmarkStrategy.MIN: 1, LandmarkStrategy.SUM: 2,
                   LandmarkStrategy.PRODUCT: 3}
_STRATEGY_BY_CODE = {c: s for s, c in _STRATEGY_CODES.items()}


class SnapshotFormatError(DblError, ValueError):
    """The file is not a valid index snapshot (snapshot.py:45-46)."""


def encode_snapshot(config: IndexConfig, n: int, landmarks, leaf_flags, bucket, dl_in, dl_out, bl_in,
                    bl_out) -> bytes:
    """Serialise metadata + labels in the reference layout (snapshot.py:76-101)."""
    parts = [MAGIC, _HEADER.pack(VERSION, n, config.k, config.k_prime, config.hash_seed,
                                 config.leaf_threshold,
                                 _STRATEGY_CODES[LandmarkStrategy(config.landmark_strategy)])]
    parts.append(np.asarray(landmarks, dtype="<u8").tobytes())
    flags = np.asarray(leaf_flags, dtype=np.uint8)
    for side in (1, 2):
        ids = np.flatnonzero(flags & side).astype("<u8")
        parts.append(struct.pack("<Q", len(ids)))
        parts.append(ids.tobytes())
    leaves = np.flatnonzero(flags)
    table = np.zeros(len(leaves), dtype=np.dtype([("v", "<u8"), ("b", "<u4")], align=False))
    table["v"] = leaves
    table["b"] = np.asarray(bucket)[leaves]
    parts.append(struct.pack("<Q", len(leaves)))
    parts.append(table.tobytes())
    rec = np.concatenate([np.asarray(a, dtype="<u8").reshape(n, -1) for a in (dl_in, dl_out, bl_in, bl_out)],
                         axis=1)
    parts.append(rec.tobytes())
    return b"".join(parts)


def decode_snapshot(data: bytes) -> dict:
    """Parse a snapshot (snapshot.py:104-148), with the reference's checks."""
    if data[:len(MAGIC)] != MAGIC:
        raise SnapshotFormatError("bad magic; not an index snapshot")
    off = len(MAGIC)
    if len(data) < off + _HEADER.size:
        raise SnapshotFormatError("truncated header")
    version, n, k, kp, seed, thr, code = _HEADER.unpack_from(data, off)
    off += _HEADER.size
    if version != VERSION:
        raise SnapshotFormatError(f"unsupported snapshot version {version}")
    if code not in _STRATEGY_BY_CODE:
        raise SnapshotFormatError(f"unknown strategy code {code}")
    cfg = IndexConfig(k=k, k_prime=kp, landmark_strategy=_STRATEGY_BY_CODE[code], leaf_threshold=thr,
                      hash_seed=seed)
    try:
        landmarks = np.frombuffer(data, "<u8", k, off).astype(np.uint64)
        off += 8 * k
        sides = []
        for _ in range(2):
            (cnt,) = struct.unpack_from("<Q", data, off)
            off += 8
            sides.append(np.frombuffer(data, "<u8", cnt, off).astype(np.uint64))
            off += 8 * cnt
        (cnt,) = struct.unpack_from("<Q", data, off)
        off += 8
        table = np.frombuffer(data, np.dtype([("v", "<u8"), ("b", "<u4")], align=False), cnt, off)
        off += 12 * cnt
        wdl, wbl = (k + 63) // 64, (kp + 63) // 64
        rw = 2 * (wdl + wbl)
        rec = np.frombuffer(data, "<u8", n * rw, off).reshape(n, rw) if rw else np.zeros((n, 0), np.uint64)
        off += 8 * n * rw
    except (struct.error, ValueError) as e:
        raise SnapshotFormatError(f"truncated snapshot: {e}") from None
    if off != len(data):
        raise SnapshotFormatError(f"trailing bytes: expected {off}, file has {len(data)}")
    flags = np.zeros(n, np.uint8)
    bucket = np.zeros(n, np.uint32)
    flags[sides[0].astype(np.int64)] |= 1
    flags[sides[1].astype(np.int64)] |= 2
    bucket[table["v"].astype(np.int64)] = table["b"]
    return {"config": cfg, "n": n, "landmarks": landmarks, "leaf_flags": flags, "bucket": bucket,
            "dl_in": np.ascontiguousarray(rec[:, :wdl]), "dl_out": np.ascontiguousarray(rec[:, wdl:2 * wdl]),
            "bl_in": np.ascontiguousarray(rec[:, 2 * wdl:2 * wdl + wbl]),
            "bl_out": np.ascontiguousarray(rec[:, 2 * wdl + wbl:])}


def snapshot_bytes(idx: DblIndex) -> bytes:
    lm, leaves = idx._metadata()
    w = idx.export_words()
    return encode_snapshot(idx.config, idx.vertex_count, np.array(lm.landmarks, dtype=np.uint64),
                           leaves.flags, leaves.bucket_array, w["dl_in"], w["dl_out"], w["bl_in"], w["bl_out"])


def save_index(idx: DblIndex, sink: Union[str, IO[bytes]]) -> None:
    """Write idx as a DBLIDX01 snapshot (snapshot.py:76-101)."""
    data = snapshot_bytes(idx)
    if isinstance(sink, str):
        with open(sink, "wb") as fh:
            fh.write(data)
    else:
        sink.write(data)


def load_index(source: Union[str, IO[bytes]], g=None) -> DblIndex:
    """Load a snapshot onto g's device (snapshot.py:104-148).

    g (optional) must have the snapshot's vertex count.  Without it, as in the
    reference, the index gets a vertex-only device graph of its own (kept
    alive by the index); queries and updates take the caller's graph as usual.
    """
    if isinstance(source, str):
        with open(source, "rb") as fh:
            data = fh.read()
    else:
        data = source.read()
    d = decode_snapshot(data)
    own = g is None
    g = DynamicGraph(d["n"]) if own else as_device_graph(g)
    if g.vertex_count != d["n"]:
        from .errors import IndexGraphMismatchError
        raise IndexGraphMismatchError(f"graph has {g.vertex_count} vertices but snapshot has {d['n']}")
    cfg = d["config"]
    lm = np.ascontiguousarray(d["landmarks"].astype(np.uint32)) if cfg.k else None
    h = ctypes.c_void_p()
    N.call("dbl_index_create", g.handle, ctypes.byref(cfg.to_c()), N.ptr(lm), N.ptr(d["leaf_flags"]),
           N.ptr(d["bucket"]), None, None, 0, ctypes.byref(h))
    idx = DblIndex(h, g, cfg)
    if own:
        idx._own_graph = g
    idx.import_words(d)
    return idx


def sniff_snapshot(path: str) -> bool:
    """True if the file starts with the snapshot magic (snapshot.py:63-69)."""
    try:
        with open(path, "rb") as fh:
            return fh.read(len(MAGIC)) == MAGIC
    except OSError:
        return False
