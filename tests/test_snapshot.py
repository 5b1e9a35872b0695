"""Snapshot format parity (reference snapshot.py:76-148): the encoder,
fed the oracle's labels, must reproduce the reference's save_index bytes;
the decoder must read them back; the GPU path must write the same bytes."""
from __future__ import annotations

import io

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O
from paper_2101_09441_b200.labels import IndexConfig, LandmarkStrategy
from paper_2101_09441_b200.snapshot import SnapshotFormatError, decode_snapshot, encode_snapshot

CASES = {
    "toy": dict(cfg=IndexConfig(k=2, k_prime=2), landmarks=[4, 7], ovr={0: 0, 9: 0, 1: 1, 2: 1, 10: 1}),
    "rand_k13": dict(cfg=IndexConfig(k=13, k_prime=96, leaf_threshold=2, landmark_strategy=LandmarkStrategy.SUM,
                                     hash_seed=9)),
    "rand_k64": dict(cfg=IndexConfig()),
    "rand_k130": dict(cfg=IndexConfig(k=130, k_prime=1)),
}


def oracle_index(d, name, spec):
    g = O.OracleGraph(int(d[f"{name}_n"]), d[f"{name}_src"], d[f"{name}_dst"])
    cfg = spec["cfg"]
    if "landmarks" in spec:
        flags, bucket = g.select_leaves(0, cfg.k_prime, 0, spec["ovr"])
        return g.build(cfg.k, cfg.k_prime, landmarks=np.array(spec["landmarks"], np.uint32),
                       leaf_flags=flags, bucket=bucket)
    return g.build(cfg.k, cfg.k_prime, cfg.landmark_strategy.value, cfg.leaf_threshold, cfg.hash_seed)


@pytest.mark.parametrize("name", list(CASES))
def test_encode_matches_reference_bytes(name):
    d = golden("snapshots")
    spec = CASES[name]
    idx = oracle_index(d, name, spec)
    data = encode_snapshot(spec["cfg"], int(d[f"{name}_n"]), idx.landmarks.astype(np.uint64), idx.leaf_flags,
                           idx.bucket, idx.dl_in, idx.dl_out, idx.bl_in, idx.bl_out)
    assert data == d[f"{name}_bytes"].tobytes()


@pytest.mark.parametrize("name", list(CASES))
def test_decode_reference_bytes(name):
    d = golden("snapshots")
    spec = CASES[name]
    idx = oracle_index(d, name, spec)
    s = decode_snapshot(d[f"{name}_bytes"].tobytes())
    assert s["n"] == int(d[f"{name}_n"]) and s["config"] == spec["cfg"]
    np.testing.assert_array_equal(s["landmarks"], idx.landmarks)
    np.testing.assert_array_equal(s["leaf_flags"], idx.leaf_flags)
    m = idx.leaf_flags != 0
    np.testing.assert_array_equal(s["bucket"][m], idx.bucket[m])
    for f in ("dl_in", "dl_out", "bl_in", "bl_out"):
        np.testing.assert_array_equal(s[f], getattr(idx, f))


def test_decoder_rejects_bad_files():
    d = golden("snapshots")
    good = d["toy_bytes"].tobytes()
    with pytest.raises(SnapshotFormatError):
        decode_snapshot(b"NOTANIDX" + good[8:])
    with pytest.raises(SnapshotFormatError):
        decode_snapshot(good + b"\0")              # trailing bytes (snapshot.py:146-147)
    with pytest.raises(SnapshotFormatError):
        decode_snapshot(good[:8] + (2).to_bytes(4, "little") + good[12:])   # version
    with pytest.raises(SnapshotFormatError):
        decode_snapshot(good[:-3])
